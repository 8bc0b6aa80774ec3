mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2 3; do for v in 0 1; do FOLD_AUX_PRIO=$v timeout 300 python bench.py $F > gpurun_out/diag_prio${v}_$i.json 2>&1; done; done
for v in 0 1; do FOLD_AUX_PRIO=$v timeout 300 python bench.py --config c3 $F > gpurun_out/diag_prio${v}_c3.json 2>&1; FOLD_AUX_PRIO=$v timeout 300 python bench.py --config c4 $F > gpurun_out/diag_prio${v}_c4.json 2>&1; done
