mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd_levels -s 0 -c 1 -o gpurun_out/prof_bwd $B > gpurun_out/ncu_bwd.log 2>&1
