#!/bin/bash
# Merge throughput against size (i32 keys-only and u32+payload, full-range keys).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for e in 16 18 20 22 24 26 28; do
  n=$((1 << (e - 1)))
  python scripts/time_merge.py i32 $n $n 0 full 2>&1 | tail -1
  python scripts/time_merge.py u32 $n $n 1 full 2>&1 | tail -1
done
