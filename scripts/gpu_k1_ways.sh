#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for w in 2 4 8; do
  cp gpurun_tmp_w$w.so paper_1202_6575_b200/lib/libstablemerge.so
  for c in 2 5 3 1; do
    timeout 120 python bench.py --config $c --steps 200 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ways=$w c=$c', 'step %.4f ms'%d['ms_per_step'])
"
  done
done
