# data-parallel paths on the one GPU a gpurun call has: the dp tests (2 gloo ranks sharing
# cuda:0) and 2-rank bench runs (c2 dense exchange, c3 sparse dE exchange, c5 strong record)
O=gpurun_out/dp; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dp.py -q > $O/pytest_dp.log 2>&1; echo "exit $?" >> $O/pytest_dp.log; tail -3 $O/pytest_dp.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
F="--gpus 2 --backend gloo --steps 2 --warmup 1 --no-table1 --no-cpu-baseline --no-sweep --no-batch1"
timeout 600 $R --master-port 29521 bench.py $F --config c3 > $O/mr_c3.json 2> $O/mr_c3.err; echo "exit $?" >> $O/mr_c3.err
timeout 600 $R --master-port 29522 bench.py $F --config c2 --batch 128 > $O/mr_c2.json 2> $O/mr_c2.err; echo "exit $?" >> $O/mr_c2.err
for f in mr_c3 mr_c2; do tail -2 $O/$f.err; python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['config'].get('exchange'), d.get('c5_strong',{}) and d['c5_strong'].get('step'))"; done
