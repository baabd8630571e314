#!/bin/bash
# Per-variant: bench configs (CONFIGS) + custom merge shapes (SHAPES, "kt n m payload dist;...").
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_1202_6575_b200/lib/libstablemerge.so /tmp/orig.so
for f in gpurun_tmp_*.so; do
  cp $f paper_1202_6575_b200/lib/libstablemerge.so
  for c in ${CONFIGS:-2}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-200} --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$f c=$c', 'step %.4f ms'%d['ms_per_step'])
"
  done
  IFS=';' read -ra SH <<< "${SHAPES:-}"
  for sh in "${SH[@]}"; do
    echo -n "$f "; timeout 120 python scripts/time_merge.py $sh 2>&1 | tail -1
  done
done
cp /tmp/orig.so paper_1202_6575_b200/lib/libstablemerge.so
