mkdir -p gpurun_out
FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config c4 --batch 1024 > gpurun_out/trace_bwd_c4.txt 2>&1
FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config c2 --batch 1024 > gpurun_out/trace_bwd_c2.txt 2>&1
FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config c3 --batch 1024 --levels 30 > gpurun_out/trace_bwd_c3.txt 2>&1
