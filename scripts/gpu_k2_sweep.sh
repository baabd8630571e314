#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in ${VARIANTS:-0 1 2 3 4 5}; do
  SM_K2_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_merge.py -q -x -m gpu -k "ragged and i32 or boundaries or reduced" -p no:cacheprovider > /tmp/t_$v.log 2>&1; echo "v=$v tests rc=$?" 
  SM_K2_VARIANT=$v timeout 120 python bench.py --config 2 --steps 300 --warmup 5 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v=$v', 'step %.4f ms'%d['ms_per_step'], 'K2 %.0f GB/s frac %.3f'%(r['achieved'], r['frac']), 'k1 %.4f'%r['k_cross_ranks_ms_per_step'])
"
done
