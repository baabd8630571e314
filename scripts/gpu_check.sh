#!/bin/bash
# Quick GPU iteration: parity tests (short first), then one bench line per config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_merge.py -m gpu -q -x --timeout 120 -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo quick rc=$?
tail -3 gpurun_out/pytest_quick.log
if [ "${FULL:-1}" = "1" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
fi
for c in ${CONFIGS:-2 3 4 5 1}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-500} --warmup 5 --cpu-seconds 1 --e2e-steps 3 > gpurun_out/bench_c$c.log 2>&1; echo bench c$c rc=$?
  tail -1 gpurun_out/bench_c$c.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d.get('roofline',{})
  print($c, 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['achieved_hbm_gbs'], 'frac %.3f'%d['achieved_hbm_frac'], 'K2 %.0f frac %.3f k1ms %.4f k2ms %.4f k3 %s'%(r['achieved'],r['frac'],r['k_cross_ranks_avg_ms'],r['avg_launch_ms'],r['k_block_sort_avg_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('parse fail', e)
"
done
