#!/bin/bash
# warp-local phase exchanges: A/B on C2 per-launch times + GPU parity
mkdir -p gpurun_out
QF_JIT_WARPSYNC=0 QF_WARP_RUNS=0 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/w1_off.json 2>&1
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/w1_on.json 2>&1
QF_WARP_RUNS=0 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/w1_runsoff.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/w1_pytest.log
