#!/bin/bash
# K2 shapes for 8-byte slots: large merges, C1 / B1, and a sort with one round per pass, per library variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k2s8
for v in paper_1202_6575_b200/lib/libstablemerge.so paper_1202_6575_b200/lib/variants/*.so; do
  echo "== $v"
  for spec in "u32 67108864 67108864 1" "i64 67108864 67108864 0" "f32 33554432 33554432 1" "u32 134217728 1048576 1" "u32 4194304 4194304 1"; do
    SM_LIB_PATH=$v timeout 120 python scripts/time_merge.py $spec
  done
  SM_LIB_PATH=$v timeout 120 python scripts/time_sort.py u32 67108864 1 full 2
  SM_LIB_PATH=$v timeout 200 python scripts/ab_time.py --configs 1,6
done 2>&1 | tee gpurun_out/k2s8/times.log
