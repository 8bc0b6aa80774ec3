# iteration check: GPU tests, C2 bench (short), C3/C4 benches, C4 B=1, C2 B=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
F="--no-cpu-baseline --no-e2e --no-table1"
timeout 300 python bench.py $F --no-batch1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c3 $F > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 $F > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c4 --batch 1 $F --no-sweep --no-batch1 > gpurun_out/bench_c4b1.json 2>&1
timeout 300 python bench.py --config c2 --batch 1 $F --no-sweep --no-batch1 > gpurun_out/bench_c2b1.json 2>&1
