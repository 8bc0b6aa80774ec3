# ncu launch lists (per-kernel serialised durations) of short bench runs: CONFIGS (default c3 c4)
mkdir -p gpurun_out/ll
B="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1"
for c in ${CONFIGS:-c3 c4}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/launches_$c.csv python bench.py --config $c $B > gpurun_out/ll/bench_ncu_$c.log 2>&1
python tools/ncu_summary.py gpurun_out/ll/$c --launches gpurun_out/ll/launches_$c.csv > /dev/null 2>&1
done
