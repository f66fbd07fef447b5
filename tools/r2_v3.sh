#!/bin/bash
# localise the n=30 adjoint defect: H|psi> JIT vs generic, sweeps JIT vs AOT, n=29, TFIM
mkdir -p gpurun_out
timeout 300 python tools/dbg_adjoint_shift.py 1 20 c128 29 30 > gpurun_out/v3_default.log 2>&1
QF_JIT_HPSI=0 timeout 300 python tools/dbg_adjoint_shift.py 1 20 c128 30 > gpurun_out/v3_nohpsijit.log 2>&1
QF_JIT=0 timeout 600 python tools/dbg_adjoint_shift.py 1 20 c128 30 > gpurun_out/v3_aot.log 2>&1
timeout 300 python tools/dbg_adjoint_shift.py 1 0 c128 30 > gpurun_out/v3_tfim.log 2>&1
timeout 300 python tools/dbg_adjoint_shift.py 2 0 c64 30 > gpurun_out/v3_tfim_d2_c64.log 2>&1
