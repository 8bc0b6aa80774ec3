mkdir -p gpurun_out/nb
F="--no-cpu-baseline --no-e2e --no-table1 --no-batch1 --no-sweep"
for t in "50 100" "100 200" "200 400" "400 800"; do
set -- $t
for cfg in "c2 16" "c2 64" "c2 256" "c2 1024" "c3 1024" "c5 64" "c4 64"; do
set -- $t $cfg
FOLD_FWD_NARROW_BELOW=$1 FOLD_BWD_NARROW_BELOW=$2 timeout 120 python bench.py --config $3 --batch $4 $F > gpurun_out/nb/${3}_b${4}_f$1_b$2.json 2>&1
done
done
