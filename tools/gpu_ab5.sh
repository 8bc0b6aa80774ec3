# three-way A/B on C2 x2, C3, C4: ab_base (HEAD), ab_a, working tree
mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for c in c2 c2b c3 c4; do
cc=${c%b}
(cd ab_base && timeout 300 python bench.py --config $cc $F > ../gpurun_out/ab_base_$c.json 2>&1)
(cd ab_a && timeout 300 python bench.py --config $cc $F > ../gpurun_out/ab_a_$c.json 2>&1)
timeout 300 python bench.py --config $cc $F > gpurun_out/ab_new_$c.json 2>&1
done
