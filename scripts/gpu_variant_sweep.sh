#!/bin/bash
# Bench prebuilt library variants (gpurun_tmp_<name>.so) on CONFIGS.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_1202_6575_b200/lib/libstablemerge.so /tmp/orig.so
for f in gpurun_tmp_*.so; do
  cp $f paper_1202_6575_b200/lib/libstablemerge.so
  for c in ${CONFIGS:-2 5}; do
    timeout 120 python bench.py --config $c --steps ${STEPS:-300} --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$f c=$c', 'step %.4f ms'%d['ms_per_step'])
"
  done
done
cp /tmp/orig.so paper_1202_6575_b200/lib/libstablemerge.so
