mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fwd_levels -s 0 -c 1 -o gpurun_out/prof_fwd $B > gpurun_out/ncu_fwd.log 2>&1
