mkdir -p gpurun_out
B="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-batch1 --no-sweep --no-clocks --no-table1 --pipeline off"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd_levels -s 1 -c 1 -o gpurun_out/prof_c5_fwd python bench.py --config c5 --batch 2048 $B > gpurun_out/ncu_c5.log 2>&1
