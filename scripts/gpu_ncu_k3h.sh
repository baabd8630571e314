python bench.py --config 5 --steps 2 --warmup 3 --no-extras > gpurun_out/r2g_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_block_sort_hbm -s 1 -c 1 -o gpurun_out/r2g_k3h_c5_src python bench.py --config 5 --steps 2 --warmup 3 --no-extras > gpurun_out/r2g_ncu_k3h.log 2>&1
echo done
