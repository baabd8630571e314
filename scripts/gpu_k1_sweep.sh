#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_merge.py -m gpu -q -x --timeout 120 -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo quick rc=$?
for v in 0 1 2 3; do for f in 2 4 16 1000000000; do for c in 2 5; do
  SM_K1_VARIANT=$v SM_K1_FACTOR=$f timeout 120 python bench.py --config $c --steps 100 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v=$v f=$f c=$c', 'k1 %.4f ms'%r['k_cross_ranks_avg_ms'], 'step %.4f'%d['ms_per_step'])
"
done; done; done
