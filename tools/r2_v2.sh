#!/bin/bash
# C4 adjoint-vs-shift probe across n (engine only), and a full ncu of C2's bwd0 at batch 64
mkdir -p gpurun_out
timeout 900 python tools/dbg_adjoint_shift.py 1 20 c128 12 16 20 24 26 28 30 > gpurun_out/v2_dbg_c128.log 2>&1
timeout 300 python tools/dbg_adjoint_shift.py 1 20 c64 20 30 > gpurun_out/v2_dbg_c64.log 2>&1
QF_JIT_DUMP=gpurun_out/jitdump python tools/c2_once.py C2 64 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 31 --launch-count 1 \
    -o gpurun_out/v2_bwd0 python tools/c2_once.py C2 64 > gpurun_out/v2_ncu_bwd0.log 2>&1
