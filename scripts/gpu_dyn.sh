#!/bin/bash
# Dynamic task assignment iteration: parity (merge, sort, batched, quick), A/B of variants, K2 timeline.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_merge.py tests/test_gpu_sort.py tests/test_gpu_batched.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_dyn.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/pytest_dyn.log
bash scripts/gpu_ab.sh ${CFGS:-1,2,3,4,5} 2>&1 | grep '"tag"'
SM_LIB_PATH=paper_1202_6575_b200/lib/variants/libstablemerge_ts_dyn.so python scripts/k2_timeline.py --configs 2,1,3,4
