mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2 3; do
(cd ab_base && timeout 300 python bench.py $F > ../gpurun_out/ab_base_$i.json 2>&1)
timeout 300 python bench.py $F > gpurun_out/ab_new_$i.json 2>&1
done
(cd ab_base && timeout 300 python bench.py --config c5 --batch 2048 $F > ../gpurun_out/ab_base_c5.json 2>&1)
timeout 300 python bench.py --config c5 --batch 2048 $F > gpurun_out/ab_new_c5.json 2>&1
timeout 300 python bench.py --config c4 $F > gpurun_out/ab_new_c4.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
