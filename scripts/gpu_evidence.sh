#!/bin/bash
# Round evidence: bench lines (default sizes), launch lists, ncu --set full of K2 per config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/ev
TAG=${TAG:-r01}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/ev/clocks.csv 2>&1 &
SMI=$!
timeout 600 python bench.py > gpurun_out/ev/bench_default.log 2>&1; echo default rc=$?; tail -1 gpurun_out/ev/bench_default.log | cut -c1-300
for c in 1 3 4 5; do timeout 600 python bench.py --config $c > gpurun_out/ev/bench_c$c.log 2>&1; echo c$c rc=$?; done
kill $SMI
for c in ${NCU_CONFIGS:-2 1 3 4 5}; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-extras"
  $CMD > gpurun_out/ev/plain_$c.log 2>&1 || { echo plain $c failed; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/${TAG}_launches_c$c.csv $CMD > /dev/null 2>&1; echo launches c$c rc=$?
  ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 3 -c 1 -o gpurun_out/ev/${TAG}_c${c}_k_tasks -f $CMD > gpurun_out/ev/ncu_full_c$c.log 2>&1; echo full c$c rc=$?
done
