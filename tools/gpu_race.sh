mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
(timeout 300 python tools/db_race.py --batch 1024 --reps 40; echo "exit $?") > gpurun_out/race_b1024.log 2>&1
(timeout 300 python tools/db_race.py --batch 256 --reps 60; echo "exit $?") > gpurun_out/race_b256.log 2>&1
(timeout 300 python tools/db_race.py --config c3 --batch 1024 --reps 30; echo "exit $?") > gpurun_out/race_c3.log 2>&1
(timeout 900 python -m pytest tests -m gpu -q -x; echo "exit $?") > gpurun_out/pytest_gpu.log 2>&1
(timeout 300 python bench.py --steps 20 --warmup 5; echo "exit $?") > gpurun_out/bench.log 2>&1
for f in gpurun_out/race_*.log gpurun_out/pytest_gpu.log; do echo "== $f"; tail -n 3 $f; done
tail -c 600 gpurun_out/bench.log
