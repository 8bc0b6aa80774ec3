mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_narrow_default.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_default.log
FOLD_FWD_NARROW_MAX=100000000 FOLD_BWD_NARROW_MAX=100000000 timeout 900 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_narrow_all.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_all.log
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
timeout 300 python bench.py --config c4 --batch 1 $F > gpurun_out/nw_c4b1.json 2>&1
timeout 300 python bench.py --config c2 --batch 1 $F > gpurun_out/nw_c2b1.json 2>&1
timeout 300 python bench.py --config c2 $F > gpurun_out/nw_c2.json 2>&1
