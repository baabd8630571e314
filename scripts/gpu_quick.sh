timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
for c in 2 3 4 5 1; do timeout 300 python bench.py --config $c --steps 200 --warmup 5 --cpu-seconds 1 --e2e-steps 3 > gpurun_out/bench_c$c.log 2>&1; echo bench c$c rc=$?; done
