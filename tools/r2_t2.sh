#!/bin/bash
# TMA partner tiles for the staged (compute-heavy) H|psi> path too: C5 / C4, GPU parity
mkdir -p gpurun_out
for v in 0 1; do
  QF_HPSI_TMA=$v timeout 900 python tools/sweep_times.py C5 4096 4 > gpurun_out/t2_C5_$v.json 2>&1
done
QF_HPSI_TMA=1 timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu > gpurun_out/t2_C4_1.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1; echo pytest=$? >> gpurun_out/t2_pytest.log
