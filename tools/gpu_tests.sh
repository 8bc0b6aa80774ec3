mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
timeout 900 python -m pytest tests -m gpu -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
else
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
fi
