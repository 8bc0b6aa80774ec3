mkdir -p gpurun_out
FOLD_DBG_FWD=2 timeout 120 python tools/trace_narrow.py --config c4 --batch 1 > gpurun_out/trace_nw_c4b1.txt 2>&1
FOLD_FWD_NARROW_MAX=100000000 timeout 900 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_narrow_all.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_all.log
