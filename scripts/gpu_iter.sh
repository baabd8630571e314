#!/bin/bash
# Iteration: quick parity, bench lines for CONFIGS, optional ncu of K2 on NCU_CFG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 300 python -m pytest tests/test_gpu_merge.py tests/test_gpu_sort.py -m gpu -q -x --timeout 120 -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo quick rc=$?; tail -1 gpurun_out/pytest_quick.log
for c in ${CONFIGS:-2 5 3}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-300} --warmup 5 --cpu-seconds 0.2 --e2e-steps 2 > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d.get('roofline',{})
  print($c, 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['achieved_hbm_gbs'], 'frac %.3f'%d['achieved_hbm_frac'], 'K2 %.0f frac %.3f k1ms %.4f k2ms %.4f k3 %s'%(r['achieved'],r['frac'],r['k_cross_ranks_ms_per_step'],r['avg_launch_ms'],r['k_block_sort_avg_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('parse fail', e)
"
done
if [ -n "$NCU_CFG" ]; then
CMD="python bench.py --config $NCU_CFG --steps 5 --warmup 3 --no-extras"
$CMD > gpurun_out/plain_ncu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_tasks} -s ${SKIP:-3} -c 1 -o gpurun_out/${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo ncu rc=$?
fi
