#!/bin/bash
# adjoint tiles of 2^11 at 4 CTAs/SM (16 warps as 4 independent CTAs) vs 2^12 at 2
mkdir -p gpurun_out
for g in "13,5,12,4:2" "13,5,11,4:4" "13,5,11,4:3"; do
  geo=${g%%:*}; mb=${g##*:}
  QF_GEOM_C64=$geo QF_JIT_MINB_BWD=$mb timeout 900 python tools/sweep_times.py C2 1024 4 > "gpurun_out/g4_${geo}_$mb.json" 2>&1
done
