# sweep one bench argument: ARG=--reserve-sms VALS="0 8 16" CONFIGS="c3 c2:256" (config[:batch])
O=gpurun_out/sweep; mkdir -p $O
F="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 --no-sweep --no-batch1"
for rep in 1 2; do
for cb in ${CONFIGS:-c3}; do
c=${cb%%:*}; b=""; [ "$cb" != "$c" ] && b="--batch ${cb#*:}"
for v in $VALS; do
  n=$(echo "${cb}_${ARG}_$v" | tr -d ' -' | tr ':' '_')
  timeout 300 python bench.py --config $c $b $F $ARG $v > $O/$n.json 2> $O/$n.err
  python - <<PY
import json
d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1])
print('$rep $cb $ARG=$v', round(d['value']/1e6,2), 'Mn/s', round(d['ms_per_step'],3),'ms', {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.02}, 'clk', d['clocks']['sm_mhz'] if d.get('clocks') else None)
PY
done; done; done
