mkdir -p gpurun_out
timeout 300 python tools/debug_narrow.py > gpurun_out/dbg_default.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
FOLD_FWD_NARROW_MAX=100000000 FOLD_BWD_NARROW_MAX=100000000 timeout 900 python -m pytest tests/test_gpu_manual.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_narrow_all.log 2>&1; echo "exit $?" >> gpurun_out/pytest_narrow_all.log
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for t in 32 64 128; do
for cb in "c2 16" "c2 64" "c4 1" "c4 16" "c4 64" "c3 1024" "c5 64"; do set -- $cb
FOLD_FWD_NARROW_MAX=$t timeout 300 python bench.py --config $1 --batch $2 $F > gpurun_out/nwf_$1_$2_t$t.json 2>&1
done; done
