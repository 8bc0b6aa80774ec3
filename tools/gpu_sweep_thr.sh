mkdir -p gpurun_out/thr
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for t in 0 16 32 64 128; do
for cfg in "c3 1024" "c2 16" "c2 64" "c4 4" "c4 16" "c5 64"; do
set -- $cfg
FOLD_FWD_NARROW_MAX=$t FOLD_BWD_NARROW_MAX=$t timeout 120 python bench.py --config $1 --batch $2 $F > gpurun_out/thr/${1}_b${2}_t$t.json 2>&1
done
done
