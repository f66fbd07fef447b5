#!/bin/bash
# stab tables from shared memory: parity + timing (C2 B=1024), C5 and C3 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/p6_parity.log 2>&1; echo rc=$? >> gpurun_out/p6_parity.log
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p6_c2.json 2>&1
