#!/bin/bash
# generic H|psi> partner tiles: TMA bulk copy + mbarrier (default) vs per-thread cp.async (QF_HPSI_TMA=0)
mkdir -p gpurun_out
for v in 0 1; do
  QF_HPSI_TMA=$v timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu > gpurun_out/t1_C4_$v.json 2>/dev/null
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/t1_pytest.log
