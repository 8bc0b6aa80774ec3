mkdir -p gpurun_out
FOLD_DBG_SCHED=1 timeout 300 python tools/trace_sched.py c2:1024 c2:256 c2:16 c2:1 c4:1 c5:8192 > gpurun_out/trace_sched.txt 2>&1
