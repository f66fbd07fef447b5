#!/bin/bash
# NVRTC / ptxas option A/B on C2 (QF_JIT_OPTS; each variant is a different cache entry)
mkdir -p gpurun_out
timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/x1_base.json 2>&1
QF_JIT_OPTS="--extra-device-vectorization" timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/x1_edv.json 2>&1
QF_JIT_OPTS="-Xptxas --allow-expensive-optimizations=true" timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/x1_aeo.json 2>&1
QF_JIT_OPTS="--maxrregcount=128" timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/x1_r128.json 2>&1
QF_JIT_OPTS="-Xptxas -O2" timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/x1_o2.json 2>&1
