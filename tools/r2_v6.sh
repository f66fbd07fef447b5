#!/bin/bash
# n >= 29 fix: adjoint vs engine shift, C4 full-size fixtures
mkdir -p gpurun_out
timeout 600 python tools/dbg_adjoint_shift.py 1 0 c128 29 30 > gpurun_out/v6_dbg.log 2>&1
timeout 600 python tools/dbg_adjoint_shift.py 1 0 c64 30 >> gpurun_out/v6_dbg.log 2>&1
timeout 600 python tools/dbg_adjoint_shift.py 1 20 c128 30 >> gpurun_out/v6_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k c4 -x -q -s > gpurun_out/v6_c4.log 2>&1
