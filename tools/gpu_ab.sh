# A/B: committed HEAD copy (ab_base/) vs working tree, C2 bench alternated; plus tests
mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do
(cd ab_base && timeout 300 python bench.py $F > ../gpurun_out/ab_base_$i.json 2>&1)
timeout 300 python bench.py $F > gpurun_out/ab_new_$i.json 2>&1
done
timeout 300 python bench.py --config c4 --batch 1 $F > gpurun_out/ab_new_c4b1.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
