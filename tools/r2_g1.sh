#!/bin/bash
# adjoint geometry with 8 register amplitudes per thread (R = 3): occupancy vs exchanges
mkdir -p gpurun_out
for g in "13,5,12,4:2" "13,5,11,3:3" "13,5,11,3:4" "13,5,12,3:1" "13,4,12,4:2"; do
  geo=${g%%:*}; mb=${g##*:}
  QF_GEOM_C64=$geo QF_JIT_MINB_BWD=$mb timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/g1_${geo}_$mb.json 2>&1
done
