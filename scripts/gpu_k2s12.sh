#!/bin/bash
# K2 shapes for 12-byte slots (8-byte keys + payload): random-key merges, C3 / C4, per library variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k2s12
for v in paper_1202_6575_b200/lib/libstablemerge.so paper_1202_6575_b200/lib/variants/*.so; do
  echo "== $v"
  for spec in "i64 67108864 67108864 1" "f64 33554432 33554432 1" "u64 67108864 67108864 1 bounded:1000" "i64 2097152 2097152 1"; do
    SM_LIB_PATH=$v timeout 120 python scripts/time_merge.py $spec
  done
  SM_LIB_PATH=$v timeout 120 python scripts/time_sort.py i64 67108864 1 full 0
  SM_LIB_PATH=$v timeout 200 python scripts/ab_time.py --configs 3,4
done 2>&1 | tee gpurun_out/k2s12/times.log
