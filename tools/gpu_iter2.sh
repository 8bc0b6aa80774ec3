mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
F="--no-cpu-baseline --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do timeout 300 python bench.py $F > gpurun_out/bench_c2_$i.json 2>&1; done
