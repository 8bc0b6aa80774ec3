mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fwd_levels -s 0 -c 1 -o gpurun_out/prof_fwd $B > gpurun_out/ncu_fwd.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dA -s 6 -c 1 -o gpurun_out/prof_dA $B > gpurun_out/ncu_dA.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dU -s 0 -c 1 -o gpurun_out/prof_dU $B > gpurun_out/ncu_dU.log 2>&1
