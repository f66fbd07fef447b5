#!/bin/bash
# with both searches on: sweep-size cap 120 (default) vs 200 vs none; C2 per-launch + C3/C5 bench + cold compile
mkdir -p gpurun_out
for cap in 120 200 0; do
  export QF_JIT_CACHE=/tmp/qf_p11_$cap
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
" > gpurun_out/p11_cold_$cap.log 2>&1
  e=$(date +%s.%N); python -c "print('cold program create s', $e - $s)" >> gpurun_out/p11_cold_$cap.log
  QF_MAX_SWEEP_OPS=$cap timeout 900 python tools/sweep_times.py C2 1024 4 > gpurun_out/p11_C2_$cap.json 2>&1
  for cfg in C3 C5; do
    QF_MAX_SWEEP_OPS=$cap timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/p11_${cfg}_$cap.json 2>/dev/null
  done
  rm -rf $QF_JIT_CACHE
done
