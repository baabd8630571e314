#!/bin/bash
# gpu_ab.sh, then an ncu capture of one kernel: bash scripts/gpu_ab_ncu.sh <configs> <pytest -k> <ncu cfg> <kernel regex> <tag>
bash scripts/gpu_ab.sh "$1" "$2"
python bench.py --config $3 --steps 2 --warmup 3 --no-extras > gpurun_out/$5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o gpurun_out/$5 python bench.py --config $3 --steps 2 --warmup 3 --no-extras > gpurun_out/$5_ncu.log 2>&1
echo ncu rc=$?
