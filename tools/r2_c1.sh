#!/bin/bash
# sweep-size cap (QF_MAX_SWEEP_OPS, default 120 now) vs no cap on C2/C3/C5, cold-compile time, GPU parity
mkdir -p gpurun_out
export QF_JIT_CACHE=/tmp/qf_cap_cache_$$
for cap in 120 0; do
  rm -rf $QF_JIT_CACHE
  s=$(date +%s.%N)
  QF_MAX_SWEEP_OPS=$cap timeout 900 python -c "
import sys; sys.path.insert(0, '.')
import bench
from paper_2602_14167_b200 import engine
ctx = engine.default_context(0)
ops, P = bench.hea_template(20, 8)
p = engine.Program(ctx, 20, ops, P, 'c64')
print('jit', p.jit_status())
" > gpurun_out/c1_cold_$cap.log 2>&1
  e=$(date +%s.%N); python -c "print('cold program create s', $e - $s)" >> gpurun_out/c1_cold_$cap.log
  for cfg in C2 C3 C5; do
    QF_MAX_SWEEP_OPS=$cap timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/c1_${cfg}_$cap.json 2> gpurun_out/c1_${cfg}_$cap.err
  done
done
rm -rf $QF_JIT_CACHE
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c1_pytest.log
