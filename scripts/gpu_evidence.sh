#!/bin/bash
# Round evidence: bench lines (default sizes), launch lists, ncu --set full of K2 per config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/ev
TAG=${TAG:-r02}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/ev/clocks.csv 2>&1 &
SMI=$!
timeout 600 python bench.py > gpurun_out/ev/bench_default.log 2>&1; echo default rc=$?; tail -1 gpurun_out/ev/bench_default.log | cut -c1-300
for c in 1 3 4 5 6; do timeout 600 python bench.py --config $c --no-per-config > gpurun_out/ev/bench_c$c.log 2>&1; echo c$c rc=$?; done
timeout 600 python bench.py --merge-path --no-per-config > gpurun_out/ev/bench_c2_mergepath.log 2>&1; echo mp rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_reference.log 2>&1; echo ref rc=$?
kill $SMI
TAG=$TAG
for c in ${NCU_CONFIGS:-2 1 3 4 5 6}; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-extras"
  $CMD > gpurun_out/ev/plain_$c.log 2>&1 || { echo plain $c failed; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/${TAG}_launches_c$c.csv $CMD > /dev/null 2>&1; echo launches c$c rc=$?
  ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 3 -c 1 -o gpurun_out/ev/${TAG}_c${c}_k_tasks -f $CMD > gpurun_out/ev/ncu_full_c$c.log 2>&1; echo full c$c rc=$?
done
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-extras"
ncu --set full --clock-control none --import-source on -k regex:k_cross_ranks -s 3 -c 1 -o gpurun_out/ev/${TAG}_c2_k_cross_ranks -f $CMD > gpurun_out/ev/ncu_k1.log 2>&1; echo k1 rc=$?
CMD="python bench.py --config 5 --steps 3 --warmup 3 --no-extras"
ncu --set full --clock-control none --import-source on -k regex:k_block_sort -s 1 -c 1 -o gpurun_out/ev/${TAG}_c5_k_block_sort -f $CMD > gpurun_out/ev/ncu_k3.log 2>&1; echo k3 rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/ev/pytest_gpu.log
# summaries on the box (gpurun merges back <= 64 MiB of gpurun_out/): the
# committed profiles/ files, the logs, and only the C2 K2 report
python scripts/make_profiles.py $TAG > gpurun_out/ev/make_profiles.log 2>&1; echo make_profiles rc=$?
mkdir -p gpurun_out/prof && cp profiles/* gpurun_out/prof/
find gpurun_out/ev -name '*.ncu-rep' ! -name "${TAG}_c2_k_tasks.ncu-rep" ! -name "${TAG}_c5_k_block_sort.ncu-rep" -delete
du -sh gpurun_out
