#!/bin/bash
# C1 (n = 10, one tile per state): fewer register bits -> more threads per state
mkdir -p gpurun_out
for g in "13,5,12,4" "13,3,12,3" "13,2,12,2" "13,4,12,3" "13,3,12,2"; do
  QF_GEOM_C64=$g timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu > gpurun_out/c1g_$g.json 2>/dev/null
done
