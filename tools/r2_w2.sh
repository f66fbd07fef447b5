#!/bin/bash
# window tile search: A/B on C2 per-launch times, then GPU parity
mkdir -p gpurun_out
QF_SWEEP_SEARCH=0 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/w2_off.json 2>&1
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/w2_on.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w2_pytest.log 2>&1; echo pytest=$? >> gpurun_out/w2_pytest.log
