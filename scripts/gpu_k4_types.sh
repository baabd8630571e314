#!/bin/bash
# k_tasks4 shapes per slot size: sort times by key type for every variant under lib/variants, ways 4 and 2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k4t
for v in paper_1202_6575_b200/lib/variants/*.so; do
  echo "== $v"
  for spec in "u32 268435456 1 bounded:1048576" "u32 268435456 0 full" "f32 268435456 1 full" "i64 134217728 0 full" "i64 134217728 1 full" "f64 134217728 1 full" "u32 16777216 1 full" "i64 16777216 0 full"; do
    for w in 4 2; do SM_LIB_PATH=$v timeout 120 python scripts/time_sort.py $spec $w; done
  done
done 2>&1 | tee gpurun_out/k4t/times.log
