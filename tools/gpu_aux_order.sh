mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do for v in 0 1 2; do FOLD_AUX_ORDER=$v timeout 300 python bench.py $F > gpurun_out/auxo${v}_$i.json 2>&1; done; done
for v in 0 2; do FOLD_AUX_ORDER=$v timeout 300 python bench.py --config c3 $F > gpurun_out/auxo${v}_c3.json 2>&1; done
