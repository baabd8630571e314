#!/bin/bash
# e2e (host buffers through the C ABI) of prebuilt variants gpurun_tmp_<name>.so on CONFIGS.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_1202_6575_b200/lib/libstablemerge.so /tmp/orig.so
for f in gpurun_tmp_*.so; do
  cp $f paper_1202_6575_b200/lib/libstablemerge.so
  for c in ${CONFIGS:-2}; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --cpu-seconds 0.2 --e2e-steps ${E2E:-20} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('$f c=$c', 'step %.4f ms'%d['ms_per_step'], 'e2e %.3e %s (%.2f ms/step)'%(e['value'], e['unit'], d['config'].get('elements', 0) and 0 or 0))
" 2>&1
  done
done
cp /tmp/orig.so paper_1202_6575_b200/lib/libstablemerge.so
