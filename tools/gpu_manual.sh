# manual-batching tests + full suite + bench with Table 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_manual.py -x -q > gpurun_out/pytest_manual.log 2>&1; echo "exit $?" >> gpurun_out/pytest_manual.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --no-table1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-table1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
