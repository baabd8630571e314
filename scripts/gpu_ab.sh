#!/bin/bash
# A/B run on the GPU box: the default build's GPU tests, then ab_time.py for
# the default library and every variant under paper_1202_6575_b200/lib/variants.
#   bash scripts/gpu_ab.sh [configs] [pytest-args]
CFGS=${1:-1,2,3,4,5}
mkdir -p gpurun_out
if [ -n "$2" ]; then python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log; fi
python scripts/ab_time.py --configs $CFGS --tag default 2>&1 | tee gpurun_out/ab_default.log
for v in paper_1202_6575_b200/lib/variants/*.so; do
  [ -e "$v" ] || continue
  SM_LIB_PATH=$v python scripts/ab_time.py --configs $CFGS 2>&1 | tee gpurun_out/ab_$(basename $v .so).log
done
