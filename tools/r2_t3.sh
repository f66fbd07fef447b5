#!/bin/bash
# specialised H|psi> partner tiles: TMA bulk copy double-buffered (default) vs direct register loads
mkdir -p gpurun_out
for v in 0 1; do
  QF_JIT_HPSI_TMA=$v timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/t3_C2_$v.json 2>&1
  QF_JIT_HPSI_TMA=$v timeout 900 python tools/sweep_times.py C3 64 2 > gpurun_out/t3_C3_$v.json 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t3_pytest.log 2>&1; echo pytest=$? >> gpurun_out/t3_pytest.log
