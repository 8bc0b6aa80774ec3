set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks"
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
timeout 200 python tools/probe_clocks.py --steps 200 --batch 1 > gpurun_out/probe_b1.json 2>&1
for k in k_cell_fwd_tc k_gemm_dA_tc k_gemm_dU_tc k_cell_bwd_pw; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
done
