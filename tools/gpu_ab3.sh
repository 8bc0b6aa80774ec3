mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sgd.py -q > gpurun_out/pytest_sgd.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sgd.log
bash tools/gpu_ab2.sh
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
