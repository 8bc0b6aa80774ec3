# three-way A/B: ab_base (HEAD), ab_a (variant A build), working tree (variant B)
mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do
(cd ab_base && timeout 300 python bench.py $F > ../gpurun_out/ab_base_$i.json 2>&1)
(cd ab_a && timeout 300 python bench.py $F > ../gpurun_out/ab_a_$i.json 2>&1)
timeout 300 python bench.py $F > gpurun_out/ab_new_$i.json 2>&1
done
