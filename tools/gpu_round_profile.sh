# Bench line + launch list + ncu --set full captures of the three tensor kernels (C2 B=1024)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks > gpurun_out/bench_ncu.log 2>&1
for k in k_fwd_levels k_bwd_levels k_gemm_dU_tc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
done
