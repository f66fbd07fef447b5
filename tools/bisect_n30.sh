#!/bin/bash
# development: the n=30 closed-form gradient test under codegen toggles
for E in "X=1" "QF_JIT_HPSI=0" "QF_JIT_NOHOIST=1" "QF_JIT_NORATIO=1" "QF_JIT_NOSTAB=1" "QF_JIT_NOLAZY=1" "QF_JIT=0"; do
  env $E timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "closed_form and 30" > gpurun_out/bis.log 2>&1
  echo "$E rc=$? $(grep -o 'AssertionError: (np.float64([0-9.e+-]*)' gpurun_out/bis.log | head -1)"
done
