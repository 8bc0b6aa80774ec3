mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 2 -c 1 -o gpurun_out/prof_sched_c2b1 python tools/sched_time.py c2:1 > gpurun_out/ncu_sched.log 2>&1
