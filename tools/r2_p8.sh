#!/bin/bash
# phase-level window search (QF_PHASE_SEARCH=1): fewer phases (exchanges) in the heavy sweeps
mkdir -p gpurun_out
timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p8_base.json 2>&1
QF_PHASE_SEARCH=1 timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p8_on.json 2>&1
QF_PHASE_SEARCH=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p8_pytest.log 2>&1; echo pytest=$? >> gpurun_out/p8_pytest.log
