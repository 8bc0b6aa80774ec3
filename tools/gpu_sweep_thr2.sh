# backward narrow threshold re-sweep (forward threshold at its default)
mkdir -p gpurun_out/thr2
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for t in 32 64 128 256; do
for cfg in "c3 1024" "c3 64" "c2 16" "c2 64" "c4 16" "c4 64" "c5 64"; do
set -- $cfg
FOLD_BWD_NARROW_MAX=$t timeout 120 python bench.py --config $1 --batch $2 $F > gpurun_out/thr2/${1}_b${2}_t$t.json 2>&1
done
done
