# quick GPU check: parity tests + smoke + probe timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 200 python tools/probe_clocks.py --steps 100 > gpurun_out/probe.json 2>&1
timeout 200 python tools/probe_clocks.py --steps 100 --batch 1 > gpurun_out/probe_b1.json 2>&1
