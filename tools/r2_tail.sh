#!/bin/bash
# light tail phases handed to the next sweep (QF_TAIL_MAX)
mkdir -p gpurun_out
for t in -1 2 3; do
  QF_TAIL_MAX=$t timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/tail_C2_$t.json 2>&1
  for cfg in C3 C5; do
    QF_TAIL_MAX=$t timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/tail_${cfg}_$t.json 2>/dev/null
  done
done
QF_TAIL_MAX=2 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tail_pytest.log 2>&1; echo pytest=$? >> gpurun_out/tail_pytest.log
