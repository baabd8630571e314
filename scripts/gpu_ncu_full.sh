#!/bin/bash
# ncu --set full captures of the top kernels (each command first run plain, && ncu).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
C2="python bench.py --config 2 --steps 5 --warmup 3 --no-extras"
C5="python bench.py --config 5 --steps 3 --warmup 3 --no-extras"
$C2 > gpurun_out/plain_full_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 3 -c 1 -o gpurun_out/${TAG}_c2_k_tasks -f $C2 > gpurun_out/ncu_full_c2_k2.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_cross_ranks -s 3 -c 1 -o gpurun_out/${TAG}_c2_k_cross_ranks -f $C2 > gpurun_out/ncu_full_c2_k1.log 2>&1; echo ncu2 rc=$?
$C5 > gpurun_out/plain_full_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_block_sort -s 2 -c 1 -o gpurun_out/${TAG}_c5_k_block_sort -f $C5 > gpurun_out/ncu_full_c5_k3.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 40 -c 1 -o gpurun_out/${TAG}_c5_k_tasks -f $C5 > gpurun_out/ncu_full_c5_k2.log 2>&1; echo ncu4 rc=$?
