mkdir -p gpurun_out
FOLD_DBG_FWD=1 timeout 300 python tools/trace_fwd.py --config c5 --batch 4096 --levels 24 > gpurun_out/trace_c5.txt 2>&1
FOLD_DBG_FWD=1 timeout 300 python tools/trace_fwd.py --config c2 --batch 1024 --levels 8 > gpurun_out/trace_c2.txt 2>&1
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
timeout 300 python bench.py --config c2 --batch 64 --prec fp32 $F > gpurun_out/bench_fp32_c2b64.json 2>&1
timeout 300 python bench.py --config c2 --batch 1 --prec fp32 $F > gpurun_out/bench_fp32_c2b1.json 2>&1
timeout 300 python bench.py --config c1 --prec fp32 $F > gpurun_out/bench_fp32_c1.json 2>&1
timeout 300 python bench.py --config c1 $F > gpurun_out/bench_c1.json 2>&1
