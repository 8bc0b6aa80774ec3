# Round profile: tests, smoke, bench line (+Table 1), C3/C4/C5 lines, precision / SST lines,
# launch list, ncu --set full of the tensor kernels (C2 B=1024) and of the narrow kernels (C4 B=1).
# Outputs in gpurun_out/rp/.
O=gpurun_out/rp; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
F="--no-cpu-baseline --no-e2e --no-table1"
timeout 300 python bench.py --config c3 $F > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c4 $F > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c5 --no-sweep --no-batch1 $F > $O/bench_c5.json 2> $O/bench_c5.err
G="$F --no-sweep --no-batch1"
timeout 300 python bench.py --prec tf32 $G > $O/bench_tf32.json 2> $O/bench_tf32.err
timeout 300 python bench.py --prec fp32 $G > $O/bench_fp32.json 2> $O/bench_fp32.err
timeout 300 python bench.py --model sst --config c3 --prec fp32 $G > $O/bench_sst.json 2> $O/bench_sst.err
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1 > $O/bench_ncu.log 2>&1
for k in ${KERNELS:-k_fwd_levels k_bwd_levels k_gemm_dU_tc}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/prof_$k python bench.py $B > $O/ncu_$k.log 2>&1
done
if [ -z "$NO_NARROW" ]; then
for k in k_fwd_narrow k_bwd_narrow; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/prof_c4b1_$k python bench.py --config c4 --batch 1 $B > $O/ncu_c4b1_$k.log 2>&1
done
fi
ls -la $O
