# latency-bound configs: bench lines + per-level traces (fwd and bwd) for C3 / C4
mkdir -p gpurun_out/lat
O=gpurun_out/lat
F="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-table1"
for c in c3 c4; do timeout 300 python bench.py --config $c $F > $O/bench_$c.json 2> $O/bench_$c.err; done
FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config c4 --batch 1024 > $O/trace_bwd_c4.txt 2>&1
FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config c3 --batch 1024 --levels 30 > $O/trace_bwd_c3.txt 2>&1
FOLD_DBG_FWD=1 timeout 300 python tools/trace_fwd.py --config c3 --batch 1024 > $O/trace_fwd_c3.txt 2>&1
FOLD_DBG_FWD=1 timeout 300 python tools/trace_fwd.py --config c4 --batch 1024 > $O/trace_fwd_c4.txt 2>&1
