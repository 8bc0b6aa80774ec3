# sweep of the pipelined scheduler's grid cap (bench --sched-bg-blocks) on CONFIGS
O=gpurun_out/sbg; mkdir -p $O
F="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 --no-sweep --no-batch1"
for rep in 1 2; do
for c in ${CONFIGS:-c2 c4 c5}; do
for nb in ${NBS:-0 4 8 16 32}; do
  timeout 300 python bench.py --config $c $F --sched-bg-blocks $nb > $O/${c}_$nb.json 2> $O/${c}_$nb.err
  python - <<PY
import json
d=json.loads(open('$O/${c}_$nb.json').read().strip().splitlines()[-1])
print('$rep $c nb=$nb', round(d['value']/1e6,2), 'Mn/s', round(d['ms_per_step'],3),'ms', {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.05}, 'clk', d['clocks']['sm_mhz'] if d.get('clocks') else None)
PY
done; done; done
