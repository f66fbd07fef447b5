#!/bin/bash
# C5 (complex128) sweep geometry with the searches on
mkdir -p gpurun_out
for g in "12,4,11,3" "12,3,11,3" "11,3,11,3" "12,4,12,3" "13,4,11,3" "12,4,11,2"; do
  QF_GEOM_C128=$g timeout 900 python tools/sweep_times.py C5 4096 4 > gpurun_out/c5g_$g.json 2>&1
done
