#!/bin/bash
# sweep-level window search on top of the phase search (QF_SWEEP_SEARCH=1): C2 per-launch, C2/C3/C5 bench, parity
mkdir -p gpurun_out
timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p10_base.json 2>&1
QF_SWEEP_SEARCH=1 timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p10_on.json 2>&1
for cfg in C3 C5; do
  for v in 0 1; do
    QF_SWEEP_SEARCH=$v timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/p10_${cfg}_$v.json 2>/dev/null
  done
done
QF_SWEEP_SEARCH=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p10_pytest.log 2>&1; echo pytest=$? >> gpurun_out/p10_pytest.log
