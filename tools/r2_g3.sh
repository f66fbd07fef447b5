#!/bin/bash
# forward occupancy: 16 amplitudes per thread at 3-4 CTAs/SM (searches on)
mkdir -p gpurun_out
for g in "13,5,12,4:2" "12,4,12,4:4" "12,4,12,4:3" "13,4,12,4:2" "12,3,12,4:4"; do
  geo=${g%%:*}; mf=${g##*:}
  QF_GEOM_C64=$geo QF_JIT_MINB_FWD=$mf timeout 900 python tools/sweep_times.py C2 1024 4 > "gpurun_out/g3_${geo}_$mf.json" 2>&1
done
