#!/bin/bash
# K3H tile size: C5 A/B, then sort times by key type for every variant under lib/variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k3t
bash scripts/gpu_ab.sh 5
for v in paper_1202_6575_b200/lib/libstablemerge.so paper_1202_6575_b200/lib/variants/*.so; do
  echo "== $v"
  for spec in "u32 268435456 0 full" "f32 268435456 1 full" "i64 134217728 1 full" "u32 33554432 1 full"; do
    SM_LIB_PATH=$v timeout 120 python scripts/time_sort.py $spec 0
  done
done 2>&1 | tee gpurun_out/k3t/times.log
