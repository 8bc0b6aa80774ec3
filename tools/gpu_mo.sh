O=gpurun_out/mo; mkdir -p $O
FOLD_DEBUG_SYNC=${SYNC:-0} timeout 1200 python -m pytest tests/test_gpu_mo.py -x -q ${PYK:+-k "$PYK"} > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -40 $O/pytest.log
