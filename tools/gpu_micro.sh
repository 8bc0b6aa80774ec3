mkdir -p gpurun_out
./tools/micro/hop_latency > gpurun_out/hop_latency.json 2>&1
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
timeout 300 python bench.py --config c4 --batch 1 $F > gpurun_out/bench_c4b1.json 2>&1
timeout 300 python bench.py --config c3 --batch 1024 --pipeline off $F > gpurun_out/bench_c3_nopipe.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
