# A/B against ab_base/ (a build of the previous commit): C2 x3 alternating, C3, C4
mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2 3; do
(cd ab_base && timeout 300 python bench.py $F > ../gpurun_out/ab_base_$i.json 2>&1)
timeout 300 python bench.py $F > gpurun_out/ab_new_$i.json 2>&1
done
for c in c3 c4; do
(cd ab_base && timeout 300 python bench.py --config $c $F > ../gpurun_out/ab_base_$c.json 2>&1)
timeout 300 python bench.py --config $c $F > gpurun_out/ab_new_$c.json 2>&1
done
