#!/bin/bash
# Two-rounds-per-pass sort: parity tests, then C5 bench lines with 4 and 2 ways.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_sort4.py -x -q -p no:cacheprovider ${PYTEST_EXTRA} > gpurun_out/s4/pytest_sort4.log 2>&1; echo sort4 rc=$?; tail -3 gpurun_out/s4/pytest_sort4.log
for w in 4 2; do
  timeout 300 python bench.py --config 5 --no-per-config --steps 10 --warmup 3 --sort-ways $w > gpurun_out/s4/bench_c5_w$w.log 2>&1; echo c5 w$w rc=$?
  tail -1 gpurun_out/s4/bench_c5_w$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['avg_launch_ms'], d['roofline']['k_cross_ranks_ms_per_step'], d['roofline'].get('k_block_sort_avg_ms'))"
done
if [ -n "$MORE_TESTS" ]; then timeout 1200 python -m pytest $MORE_TESTS -x -q -p no:cacheprovider > gpurun_out/s4/pytest_more.log 2>&1; echo more rc=$?; tail -3 gpurun_out/s4/pytest_more.log; fi
