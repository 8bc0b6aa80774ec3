mkdir -p gpurun_out
F="--no-cpu-baseline --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do
timeout 300 python bench.py $F --pipeline on > gpurun_out/pipe_on_$i.json 2>&1
timeout 300 python bench.py $F --pipeline off > gpurun_out/pipe_off_$i.json 2>&1
done
for cb in "c2 1" "c2 64" "c4 256" "c3 1024" "c5 8192"; do set -- $cb
timeout 300 python bench.py --config $1 --batch $2 $F --pipeline on > gpurun_out/pipe_on_$1_$2.json 2>&1
timeout 300 python bench.py --config $1 --batch $2 $F --pipeline off > gpurun_out/pipe_off_$1_$2.json 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
