#!/bin/bash
# dram traffic / FMA-pipe metrics of the dominant kernel of C3 (first adjoint sweep, batch 64),
# C4 (H|psi>, batch 1) and C5 (H|psi>, batch 4096), second evaluation (first one compiles)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
python tools/c2_once.py C3 64 > /dev/null
ncu --metrics $M --clock-control none -k regex:qf_sweep --launch-skip $(python -c "
import sys; sys.path.insert(0,'.')
import bench; from paper_2602_14167_b200 import engine
c=bench.CONFIGS['C3']; ops,P=bench.hea_template(c['n'],c['layers'])
d=engine.describe_plan(c['n'],ops,P,c['prec']); f=len(d['passes']['fwd']['sweeps']); b=len(d['passes']['bwd']['sweeps'])
print(2*f+b)") --launch-count 1 --csv --log-file gpurun_out/ncu_c3.csv python tools/c2_once.py C3 64 > gpurun_out/ncu_c3.log 2>&1; echo C3 $?
python tools/c2_once.py C4 1 > /dev/null
ncu --metrics $M --clock-control none -k regex:hpsi --launch-skip 1 --launch-count 1 --csv --log-file gpurun_out/ncu_c4.csv python tools/c2_once.py C4 1 > gpurun_out/ncu_c4.log 2>&1; echo C4 $?
python tools/c2_once.py C5 4096 > /dev/null
ncu --metrics $M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:hpsi --launch-skip 1 --launch-count 1 --csv --log-file gpurun_out/ncu_c5.csv python tools/c2_once.py C5 4096 > gpurun_out/ncu_c5.log 2>&1; echo C5 $?
