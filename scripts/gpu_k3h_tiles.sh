#!/bin/bash
# K3H tile sizes: sort times by key type for the default library and every variant under lib/variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k3t
for v in paper_1202_6575_b200/lib/libstablemerge.so paper_1202_6575_b200/lib/variants/*.so; do
  echo "== $v"
  for spec in "i64 134217728 0 full" "i64 134217728 1 full" "f64 134217728 1 full" "u64 67108864 1 full"; do
    SM_LIB_PATH=$v timeout 120 python scripts/time_sort.py $spec 0
  done
done 2>&1 | tee gpurun_out/k3t/times.log
