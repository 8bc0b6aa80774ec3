# diagnostics: wide-kernel mainloop speed with parts of the epilogue removed (results invalid)
mkdir -p gpurun_out
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do
timeout 300 python bench.py $F > gpurun_out/diag_base_$i.json 2>&1
for v in 2 3 4; do FOLD_DBG_BWD=$v timeout 300 python bench.py $F > gpurun_out/diag_bwd${v}_$i.json 2>&1; done
done
