#!/bin/bash
# phase search default-on: C2/C3/C5 bench vs QF_PHASE_SEARCH=0, GPU parity
mkdir -p gpurun_out
for v in 0 1; do
  for cfg in C2 C3 C5; do
    QF_PHASE_SEARCH=$v timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/p9_${cfg}_$v.json 2> gpurun_out/p9_${cfg}_$v.err
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p9_pytest.log 2>&1; echo pytest=$? >> gpurun_out/p9_pytest.log
