python bench.py --config 2 --steps 3 --warmup 3 --no-extras > gpurun_out/r2b_plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 3 -c 1 -o gpurun_out/r2b_k2_c2_src python bench.py --config 2 --steps 3 --warmup 3 --no-extras > gpurun_out/r2b_ncu_k2.log 2>&1
echo done
