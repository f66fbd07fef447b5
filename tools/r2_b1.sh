#!/bin/bash
# lane order for bank-conflict-free exchanges: A/B on C2 per-launch times, bank conflicts of bwd0, parity
mkdir -p gpurun_out
QF_LANE_ORDER=0 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/b1_off.json 2>&1
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/b1_on.json 2>&1
for v in 0 1; do
  QF_LANE_ORDER=$v timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:qf_sweep -c 22 --csv \
    python tools/c2_once.py C2 64 > gpurun_out/b1_ncu_$v.csv 2> gpurun_out/b1_ncu_$v.err
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/b1_pytest.log
