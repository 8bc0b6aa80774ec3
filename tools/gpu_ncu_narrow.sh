# ncu --set full of the persistent fwd/bwd kernels on the latency-bound configs (C3 B=1024, C4 B=1)
mkdir -p gpurun_out
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1"
for cfg in "c3 1024" "c4 1"; do
set -- $cfg
for k in k_fwd_levels k_bwd_levels; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${1}_b${2}_$k python bench.py --config $1 --batch $2 $B > gpurun_out/ncu_${1}_$k.log 2>&1
done
done
