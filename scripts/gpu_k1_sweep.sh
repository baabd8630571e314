#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 1 5 6 7 8; do for c in 2 5 3; do
  SM_K1_VARIANT=$v timeout 120 python bench.py --config $c --steps 100 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v=$v c=$c', 'k1/step %.4f ms'%r['k_cross_ranks_ms_per_step'], 'step %.4f'%d['ms_per_step'])
"
done; done
