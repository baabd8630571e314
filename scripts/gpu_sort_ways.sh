cd "${GRAFT_REPO_ROOT:-/root/repo}"
for spec in "u32 268435456 1 bounded:1048576" "u32 268435456 0 full" "i32 268435456 1 full" "f32 268435456 1 full" "u64 134217728 0 full" "i64 134217728 1 full" "f64 134217728 1 full" "u32 16777216 1 full" "u32 2000000 1 full"; do
  for w in 4 2; do timeout 120 python scripts/time_sort.py $spec $w; done
done
