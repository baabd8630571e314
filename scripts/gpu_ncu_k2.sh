#!/bin/bash
# ncu --set full of K2 on C2 and C3 (plain run first).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01b}
for c in ${CONFIGS:-2 3}; do
CMD="python bench.py --config $c --steps 5 --warmup 3 --no-extras"
$CMD > gpurun_out/plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_tasks} -s 3 -c 1 -o gpurun_out/${TAG}_c${c}_k2 -f $CMD > gpurun_out/ncu_${TAG}_c$c.log 2>&1; echo ncu c$c rc=$?
done
