#!/bin/bash
# n=30 JIT adjoint defect: bisect over the generator's toggles (TFIM, D=1, c128)
mkdir -p gpurun_out
for t in NONE QF_JIT_NODEFER QF_JIT_NORATIO QF_JIT_NOSTAB QF_JIT_NOHOIST QF_JIT_NOLAZY; do
  if [ $t = NONE ]; then env=""; else env="$t=1"; fi
  echo "== $t" >> gpurun_out/v4.log
  env $env timeout 300 python tools/dbg_adjoint_shift.py 1 0 c128 30 >> gpurun_out/v4.log 2>&1
done
for t in QF_JIT_DIRECT QF_JIT_FUSE; do
  echo "== $t=0" >> gpurun_out/v4.log
  env $t=0 timeout 300 python tools/dbg_adjoint_shift.py 1 0 c128 30 >> gpurun_out/v4.log 2>&1
done
