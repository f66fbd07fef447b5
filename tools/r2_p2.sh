#!/bin/bash
# perf: 3 adjoint CTAs per SM (register cap 85, tap staging 8 slots), C2 B=1024
mkdir -p gpurun_out
QF_JIT_MINB_BWD=3 QF_JIT_TAPSTAGE=8 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p2_mb3_s8.json 2>&1
QF_JIT_TAPSTAGE=8 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p2_s8.json 2>&1
QF_JIT_MINB_FWD=3 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p2_fmb3.json 2>&1
