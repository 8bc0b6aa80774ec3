mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_schedule.py -x -q > gpurun_out/pytest_sched.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sched.log
timeout 200 python tools/probe_clocks.py --steps 100 > gpurun_out/probe.json 2>&1
timeout 200 python tools/probe_clocks.py --steps 100 --batch 1 > gpurun_out/probe_b1.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sched.csv python tools/probe_clocks.py --steps 2 --batch 1024 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sched1.csv python tools/probe_clocks.py --steps 2 --batch 1 > /dev/null 2>&1
