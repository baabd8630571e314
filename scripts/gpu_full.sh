#!/bin/bash
# GPU tests, then the default bench line (with per_config) and the sort headline.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/full_pytest.log
python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/full_bench.json
python bench.py --config 5 --steps 10 --warmup 3 --no-per-config > gpurun_out/full_bench_c5.json 2> gpurun_out/full_bench_c5.err; echo "bench5 rc=$?"
