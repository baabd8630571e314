#!/bin/bash
# Per-kernel live times (sm_profile_*) of prebuilt library variants
# (gpurun_tmp_<name>.so) on CONFIGS.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_1202_6575_b200/lib/libstablemerge.so /tmp/orig.so
for f in gpurun_tmp_*.so; do
  cp $f paper_1202_6575_b200/lib/libstablemerge.so
  for c in ${CONFIGS:-2 5}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --cpu-seconds 0.5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f c=$c', 'step %.4f ms'%d['ms_per_step'], 'K2 avg %.4f ms/launch, %.4f ms/step; K1 %.4f ms/step; K3 %s' % (
  r['avg_launch_ms'], r['k_tasks_ms_per_step'], r['k_cross_ranks_ms_per_step'], r['k_block_sort_avg_ms']), d.get('clocks'))
"
  done
done
cp /tmp/orig.so paper_1202_6575_b200/lib/libstablemerge.so
