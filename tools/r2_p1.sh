#!/bin/bash
# perf: cap on ops per sweep (splits the heavy triangle sweeps; icache / balance), C2 B=1024
mkdir -p gpurun_out
for m in 0 200 120 80; do
  if [ $m = 0 ]; then env=""; else env="QF_MAX_SWEEP_OPS=$m"; fi
  env $env timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p1_max$m.json 2>&1
done
