#!/bin/bash
# One GPU session: parity tests, bench lines per config, launch list of the default bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for c in 2 3 4 5 1; do
  timeout 400 python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1; echo bench c$c rc=$?
  tail -1 gpurun_out/bench_c$c.log | cut -c1-400
done
python bench.py --config 2 --steps 20 --warmup 3 --no-extras > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --config 2 --steps 20 --warmup 3 --no-extras > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
