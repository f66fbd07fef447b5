#!/bin/bash
# occupancy probes on the capped, swizzle-searched sweeps: 3 CTAs/SM for the adjoint / forward sweeps
mkdir -p gpurun_out
timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/o1_base.json 2>&1
QF_JIT_MINB_BWD=3 QF_JIT_TAPSTAGE=8 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/o1_b3.json 2>&1
QF_JIT_MINB_FWD=3 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/o1_f3.json 2>&1
QF_MAX_SWEEP_OPS=60 QF_JIT_MINB_BWD=3 QF_JIT_TAPSTAGE=8 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/o1_b3c60.json 2>&1
