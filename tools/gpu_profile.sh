# Profile pass: headline bench line, ncu launch list (serialised, cold), ncu --set full of the
# three tcgen05 kernels at C2 B=1024 (one launch each). Outputs in gpurun_out/prof/.
mkdir -p gpurun_out/prof
O=gpurun_out/prof
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1 > $O/bench_ncu.log 2>&1
for k in ${KERNELS:-k_fwd_levels k_bwd_levels k_gemm_dU_tc}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/prof_$k python bench.py $B > $O/ncu_$k.log 2>&1
done
ls -la $O
