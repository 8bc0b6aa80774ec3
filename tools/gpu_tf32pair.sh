O=gpurun_out/tfp; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -k "tf32 or fp32 or sst or mo or dp" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -3 $O/pytest.log
F="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 --no-sweep --no-batch1"
for v in 0 1; do for args in "--prec fp32" "--prec tf32" "--model sst --config c3 --prec fp32" "--model mo --prec fp32" "--model mo --prec tf32"; do
  FOLD_TF32_PAIR=$v timeout 300 python bench.py $F $args > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('pair=$v', '$args', round(d['value']/1e6,2), 'Mn/s', round(d['ms_per_step'],2), 'ms', {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>0.2})"
done; done
