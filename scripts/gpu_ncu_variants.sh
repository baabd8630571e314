#!/bin/bash
# ncu --set full of K2 for each prebuilt variant gpurun_tmp_<name>.so on CONFIGS
# (plain run first).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp paper_1202_6575_b200/lib/libstablemerge.so /tmp/orig.so
for f in gpurun_tmp_*.so; do
  v=$(basename $f .so | sed 's/gpurun_tmp_//')
  cp $f paper_1202_6575_b200/lib/libstablemerge.so
  for c in ${CONFIGS:-4}; do
    CMD="python bench.py --config $c --steps 5 --warmup 3 --no-extras"
    $CMD > gpurun_out/plain_${v}_$c.log 2>&1 && \
    ncu --set full --clock-control none -k regex:${KERN:-k_tasks} -s 3 -c 1 -o gpurun_out/var_${v}_c${c} -f $CMD > gpurun_out/ncu_var_${v}_c$c.log 2>&1; echo ncu $v c$c rc=$?
  done
done
cp /tmp/orig.so paper_1202_6575_b200/lib/libstablemerge.so
