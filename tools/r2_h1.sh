#!/bin/bash
# generic H|psi> at 2048-amplitude tiles (C5, complex128): 16 amplitudes x 128 threads vs 8 x 256
mkdir -p gpurun_out
for v in 0 1; do
  QF_HPSI_NA8=$v timeout 600 python tools/sweep_times.py C5 4096 4 > gpurun_out/h1_$v.json 2>&1
done
QF_HPSI_NA8=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or stress or config" > gpurun_out/h1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/h1_pytest.log
