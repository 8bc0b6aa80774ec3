# full GPU suite (or PYTEST_K subset) + one bench line; logs under gpurun_out/
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nproc > gpurun_out/nproc.txt
if [ -n "$PYTEST_K" ]; then
(timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" --durations=15; echo "exit $?") > gpurun_out/pytest_gpu.log 2>&1
else
(timeout 1500 python -m pytest tests -m gpu -q --durations=15; echo "exit $?") > gpurun_out/pytest_gpu.log 2>&1
fi
tail -n 30 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
(timeout 400 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS}; echo "exit $?") > gpurun_out/bench.log 2>&1
tail -c 300 gpurun_out/bench.log
fi
