# full GPU suite on the current library, then an A/B of bench lines vs a variant library
O=gpurun_out/chk; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -3 $O/pytest.log
bash tools/gpu_ab_env.sh
