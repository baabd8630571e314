set -x
python bench.py --config 2 --steps 3 --warmup 3 --no-extras > gpurun_out/r2_plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tasks -s 3 -c 1 -o gpurun_out/r2_k2_c2_src python bench.py --config 2 --steps 3 --warmup 3 --no-extras > gpurun_out/r2_ncu_k2.log 2>&1
python bench.py --config 5 --steps 2 --warmup 3 --no-extras > gpurun_out/r2_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_block_sort -s 1 -c 1 -o gpurun_out/r2_k3_c5_src python bench.py --config 5 --steps 2 --warmup 3 --no-extras > gpurun_out/r2_ncu_k3.log 2>&1
for c in 1 2 3 4 5; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2_base_c$c.json 2>gpurun_out/r2_base_c$c.err; done
