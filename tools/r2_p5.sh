#!/bin/bash
# ncu of the heavy forward sweep fwd0 (C2, batch 64)
mkdir -p gpurun_out
QF_JIT_NOILV=1 python tools/c2_once.py C2 64 > /dev/null 2>&1
QF_JIT_NOILV=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 22 --launch-count 1 \
    -o gpurun_out/p5_fwd0 python tools/c2_once.py C2 64 > gpurun_out/p5_ncu.log 2>&1
