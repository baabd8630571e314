#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 5 --warmup 3 --no-extras"
export SM_K1_VARIANT=1 SM_K1_FACTOR=2
$CMD > gpurun_out/plain_k1.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_cross_ranks -s 3 -c 1 -o gpurun_out/k1_v1f2 -f $CMD > gpurun_out/ncu_k1.log 2>&1; echo rc=$?
export SM_K1_VARIANT=0 SM_K1_FACTOR=1000000000
ncu --set full --clock-control none -k regex:k_cross_ranks -s 3 -c 1 -o gpurun_out/k1_v0finf -f $CMD > gpurun_out/ncu_k1b.log 2>&1; echo rc=$?
