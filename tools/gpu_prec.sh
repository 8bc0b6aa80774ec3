# C2 B=1024 bench lines per precision mode (+ the SIMT FP32 A/B), logs in gpurun_out/
mkdir -p gpurun_out
F="--steps 5 --warmup 3 --no-sweep --no-table1 --no-cpu-baseline --no-batch1"
for p in tf32 fp32; do
timeout 600 python bench.py --prec $p $F > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err
done
FOLD_FP32_SIMT=1 timeout 900 python bench.py --prec fp32 $F --no-e2e > gpurun_out/bench_fp32_simt.json 2> gpurun_out/bench_fp32_simt.err
for p in tf32 fp32 fp32_simt; do echo $p; tail -c 400 gpurun_out/bench_$p.err; python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$p.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['roofline']['frac'])
"; done
