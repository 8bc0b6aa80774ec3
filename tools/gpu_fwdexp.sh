mkdir -p gpurun_out
for v in 0; do FOLD_DBG_FWD=$v timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$v.log;
FOLD_DBG_FWD=$v timeout 200 python tools/probe_clocks.py --steps 60 > gpurun_out/probe_$v.json 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-sweep --no-batch1 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --no-sweep --no-batch1 > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
