#!/bin/bash
# Round profile of the C2 headline: bench line, ncu launch list of the same command,
# full captures of the first adjoint sweep of the second evaluation (launch index
# = sweeps per evaluation + forward sweeps, from the plan) and of H|psi> at batch 1024.
python bench.py --steps 3 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err; echo BENCH $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/prof_ncu_launch.log 2>&1; echo LAUNCH $?
python tools/c2_once.py C2 1024 > /dev/null; echo ONCE $?
SKIP=$(python -c "
import sys; sys.path.insert(0, '.')
import bench
from paper_2602_14167_b200 import engine
ops, P = bench.hea_template(20, 8)
d = engine.describe_plan(20, ops, P, 'c64')['passes']
f, b = len(d['fwd']['sweeps']), len(d['bwd']['sweeps'])
print(f + b + f)")
echo SKIP $SKIP
ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip $SKIP --launch-count 1 \
    -o gpurun_out/prof_bwd0 python tools/c2_once.py C2 1024 > gpurun_out/prof_ncu_bwd0.log 2>&1; echo BWD0 $?
ncu --set full --import-source on --clock-control none -k regex:qf_hpsi --launch-skip 1 --launch-count 1 \
    -o gpurun_out/prof_hpsi python tools/c2_once.py C2 1024 > gpurun_out/prof_ncu_hpsi.log 2>&1; echo HPSI $?
