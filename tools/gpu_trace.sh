mkdir -p gpurun_out
FOLD_DBG_FWD=1 timeout 120 python tools/trace_fwd.py --config c2 --batch 1024 --levels 8 > gpurun_out/trace_c2.txt 2>&1
FOLD_DBG_FWD=1 timeout 120 python tools/trace_fwd.py --config c4 --batch 1 --levels 4 > gpurun_out/trace_c4b1.txt 2>&1
