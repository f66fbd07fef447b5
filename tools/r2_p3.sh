#!/bin/bash
# interleaved psi/lambda exchange + split tap accumulators: parity, then A/B timings (C2 B=1024)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not c3 and not c4 and not n30" -x -q > gpurun_out/p3_parity.log 2>&1; echo rc=$? >> gpurun_out/p3_parity.log
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p3_new.json 2>&1
QF_JIT_NOILV=1 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p3_noilv.json 2>&1
QF_JIT_TAPACC1=1 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p3_tapacc1.json 2>&1
