#!/bin/bash
# ncu --set full of k_tasks4 (C5, two rounds per pass) and of the 4-way partition kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k4
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-extras --sort-ways 4"
$CMD > gpurun_out/k4/plain.log 2>&1 || { echo plain failed; tail gpurun_out/k4/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_tasks4 -s 2 -c 1 -o gpurun_out/k4/k_tasks4 -f $CMD > gpurun_out/k4/ncu_k4.log 2>&1; echo k4 rc=$?
ncu --set full --clock-control none -k regex:k4_ranks -s 2 -c 1 -o gpurun_out/k4/k4_ranks -f $CMD > gpurun_out/k4/ncu_r.log 2>&1; echo ranks rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k4/launches.csv $CMD > /dev/null 2>&1; echo launches rc=$?
