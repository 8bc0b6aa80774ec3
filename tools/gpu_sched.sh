mkdir -p gpurun_out
C="c4:1 c2:1 c2:4 c2:16 c2:64 c3:64 c3:256 c2:256 c2:1024"
python tools/sched_time.py $C > gpurun_out/sched_times.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_manual.py -q > gpurun_out/pytest_sched.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sched.log
F="--no-cpu-baseline --no-table1 --no-batch1"
timeout 300 python bench.py $F > gpurun_out/bench_c2.json 2>&1
