O=gpurun_out/mo; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mo.py -q > $O/pytest_nosync.log 2>&1; echo "exit $?" >> $O/pytest_nosync.log; tail -2 $O/pytest_nosync.log
for p in fp32 tf32; do
timeout 600 python bench.py --model mo --prec $p --steps 5 --warmup 3 > $O/bench_mo_$p.json 2> $O/bench_mo_$p.err
tail -c 2500 $O/bench_mo_$p.json; tail -3 $O/bench_mo_$p.err
done
