#!/bin/bash
# sweep objective: gates per phase (QF_SWEEP_OBJ=ratio) vs gates (default)
mkdir -p gpurun_out
for v in items ratio_fwd; do
  QF_SWEEP_OBJ=$v timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p12_C2_$v.json 2>&1
  for cfg in C3 C5; do
    QF_SWEEP_OBJ=$v timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/p12_${cfg}_$v.json 2>/dev/null
  done
done
