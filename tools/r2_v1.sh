#!/bin/bash
# round 2 (re-entry): verify HEAD on one B200: smoke, all GPU tests (timed), bench, per-launch sweep times
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/v1_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1; echo smoke=$? >> gpurun_out/v1_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/v1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/v1_pytest.log
timeout 600 python bench.py > gpurun_out/v1_bench.json 2> gpurun_out/v1_bench.err; echo bench=$? >> gpurun_out/v1_bench.err
python tools/sweep_times.py C2 1024 6 > gpurun_out/v1_times.json 2>&1
