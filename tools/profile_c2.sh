#!/bin/bash
# Round profile of the C2 headline: bench line, ncu launch list of the same command,
# full captures of the first adjoint sweep (second evaluation: 24 sweeps per
# evaluation, 10 forward, so launch 24 + 10 = 34) and of H|psi> at batch 1024.
python bench.py --steps 3 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err; echo BENCH $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/prof_ncu_launch.log 2>&1; echo LAUNCH $?
python tools/c2_once.py C2 1024 > /dev/null; echo ONCE $?
ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 34 --launch-count 1 \
    -o gpurun_out/prof_bwd0 python tools/c2_once.py C2 1024 > gpurun_out/prof_ncu_bwd0.log 2>&1; echo BWD0 $?
ncu --set full --import-source on --clock-control none -k regex:qf_hpsi --launch-skip 1 --launch-count 1 \
    -o gpurun_out/prof_hpsi python tools/c2_once.py C2 1024 > gpurun_out/prof_ncu_hpsi.log 2>&1; echo HPSI $?
