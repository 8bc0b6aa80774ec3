# GPU suite (optionally a subset via PYTEST_K) + C2 / C3 / C4 bench lines (short)
mkdir -p gpurun_out/q
O=gpurun_out/q
if [ -n "$PYTEST_K" ]; then
(timeout 1500 python -m pytest tests -m gpu -q -x -k "$PYTEST_K"; echo "exit $?") > $O/pytest.log 2>&1
elif [ -z "$NO_TESTS" ]; then
(timeout 1500 python -m pytest tests -m gpu -q -x; echo "exit $?") > $O/pytest.log 2>&1
fi
tail -n 3 $O/pytest.log
F="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 --no-sweep --no-batch1"
for c in ${CONFIGS:-c2 c3 c4}; do timeout 300 python bench.py --config $c $F $BENCH_ARGS > $O/bench_$c.json 2> $O/bench_$c.err; python - <<PY
import json
d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value']/1e6,2), 'Mn/s', round(d['ms_per_step'],3),'ms', {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, 'clk', d['clocks']['sm_mhz'] if d.get('clocks') else None)
PY
done
