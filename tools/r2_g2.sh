#!/bin/bash
# tile geometry (kf,Rf,kb,Rb) with the tile + phase searches on
mkdir -p gpurun_out
for g in "13,5,12,4:2:2" "14,5,12,4:1:2" "13,5,13,4:2:1" "13,4,12,4:2:2" "12,4,12,4:2:2" "14,6,12,4:1:2"; do
  geo=${g%%:*}; rest=${g#*:}; mf=${rest%%:*}; mb=${rest##*:}
  QF_GEOM_C64=$geo QF_JIT_MINB_FWD=$mf QF_JIT_MINB_BWD=$mb timeout 900 python tools/sweep_times.py C2 1024 4 > "gpurun_out/g2_${geo}_${mf}_${mb}.json" 2>&1
done
