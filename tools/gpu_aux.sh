mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do for o in 0 1 2; do
FOLD_AUX_ORDER=$o timeout 300 python bench.py $F > gpurun_out/aux_o${o}_$i.json 2>&1
done; done
FOLD_AUX_ORDER=2 timeout 300 python bench.py --config c5 --batch 2048 $F > gpurun_out/aux_o2_c5.json 2>&1
FOLD_AUX_ORDER=0 timeout 300 python bench.py --config c5 --batch 2048 $F > gpurun_out/aux_o0_c5.json 2>&1
