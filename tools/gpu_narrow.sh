mkdir -p gpurun_out
timeout 300 python tools/debug_narrow.py > gpurun_out/dbg_default.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_narrow_default.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_default.log
FOLD_FWD_NARROW_MAX=100000000 FOLD_BWD_NARROW_MAX=100000000 timeout 900 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_narrow_all.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_all.log
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1"
timeout 300 python bench.py --config c4 $F > gpurun_out/nw_c4.json 2>&1
timeout 300 python bench.py --config c2 $F > gpurun_out/nw_c2.json 2>&1
timeout 300 python bench.py --config c3 $F > gpurun_out/nw_c3.json 2>&1
for t in 32 64 128; do
FOLD_BWD_NARROW_MAX=$t timeout 300 python bench.py --config c4 --batch 64 $F --no-sweep > gpurun_out/nw_c4b64_t$t.json 2>&1
FOLD_BWD_NARROW_MAX=$t timeout 300 python bench.py --config c5 --batch 64 $F --no-sweep > gpurun_out/nw_c5b64_t$t.json 2>&1
done
