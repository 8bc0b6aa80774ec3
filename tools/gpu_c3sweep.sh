mkdir -p gpurun_out/c3
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep --config c3 --pipeline off"
for f in 32 96 256; do for b in 128 384 1024; do
FOLD_FWD_NARROW_MAX=$f FOLD_BWD_NARROW_MAX=$b timeout 120 python bench.py $F > gpurun_out/c3/f${f}_b${b}.json 2>&1
done; done
for cb in "c3 64" "c3 256"; do set -- $cb
for f in 32 256; do for b in 128 1024; do
FOLD_FWD_NARROW_MAX=$f FOLD_BWD_NARROW_MAX=$b timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep --config $1 --batch $2 --pipeline off > gpurun_out/c3/${1}_${2}_f${f}_b${b}.json 2>&1
done; done; done
