mkdir -p gpurun_out
timeout 300 python tools/debug_narrow.py > gpurun_out/dbg_default.txt 2>&1
FOLD_BWD_NARROW_MAX=0 timeout 300 python tools/debug_narrow.py > gpurun_out/dbg_off.txt 2>&1
