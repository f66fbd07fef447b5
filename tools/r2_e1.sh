#!/bin/bash
# hetrd fused-sweep unroll (columns in flight per thread): MIPT Table IV entropy time, eigen-solver tests
mkdir -p gpurun_out
for u in 4 8 2; do
  QF_HETRD_UNROLL=$u QF_MIPT_TIMING=1 timeout 600 python tools/bench_mipt.py > gpurun_out/e1_$u.json 2>&1
done
QF_HETRD_UNROLL=8 timeout 600 python -m pytest tests/test_gpu_traj.py -x -q -k "eigvals or mipt" > gpurun_out/e1_pytest.log 2>&1; echo rc=$? >> gpurun_out/e1_pytest.log
