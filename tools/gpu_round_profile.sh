# Round profile: tests, smoke, bench line (+Table 1), C3/C4/C5 lines, launch list,
# ncu --set full of the tensor kernels (C2 B=1024) and of the narrow kernels (C4 B=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
F="--no-cpu-baseline --no-e2e --no-table1"
timeout 300 python bench.py --config c3 $F > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 $F > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c5 --no-sweep --no-batch1 $F > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1 > gpurun_out/bench_ncu.log 2>&1
for k in k_fwd_levels k_bwd_levels k_gemm_dU_tc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python bench.py $B > gpurun_out/ncu_$k.log 2>&1
done
for k in k_fwd_narrow k_bwd_narrow; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_c4b1_$k python bench.py --config c4 --batch 1 $B > gpurun_out/ncu_c4b1_$k.log 2>&1
done
