#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -k "virtual or device_entry or nccl" -x -q > gpurun_out/s4_tests.log 2>&1
python tools/sweep_times.py C2 1024 8 > gpurun_out/s4_times_defer.json 2>&1
QF_JIT_NOPACK=1 python tools/sweep_times.py C2 1024 8 > gpurun_out/s4_times_nopack.json 2>&1
python tools/sweep_times.py C2 256 8 > gpurun_out/s4_times_b256.json 2>&1
