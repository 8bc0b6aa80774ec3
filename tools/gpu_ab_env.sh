# A/B of environment settings on bench lines (short runs): VARIANTS="name:ENV=.. ENV2=..;name2:..."
O=gpurun_out/ab; mkdir -p $O
F="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 --no-sweep --no-batch1"
IFS=';' read -ra VS <<< "$VARIANTS"
for rep in 1 2; do
for v in "${VS[@]}"; do
  name=${v%%:*}; envs=${v#*:}
  for c in ${CONFIGS:-c2}; do
    env $envs timeout 300 python bench.py --config $c $F $BENCH_ARGS > $O/${name}_$c.json 2> $O/${name}_$c.err
    python - <<PY
import json
d=json.loads(open('$O/${name}_$c.json').read().strip().splitlines()[-1])
print('$rep $name $c', round(d['value']/1e6,2), 'Mn/s', round(d['ms_per_step'],3),'ms', {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.05}, 'clk', d['clocks']['sm_mhz'] if d.get('clocks') else None)
PY
  done
done
done
