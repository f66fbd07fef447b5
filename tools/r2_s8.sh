#!/bin/bash
# per-sweep swizzle search (QF_JIT_FOLDSWZ=1: XOR-fold default): A/B on C2 per-launch times, bank conflicts of bwd0, parity
mkdir -p gpurun_out
QF_JIT_FOLDSWZ=1 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/s1_off.json 2>&1
timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/s1_on.json 2>&1
for v in 1 0; do
  QF_JIT_FOLDSWZ=$v timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:qf_sweep -c 24 --csv \
    python tools/c2_once.py C2 64 > gpurun_out/s1_ncu_$v.csv 2> gpurun_out/s1_ncu_$v.err
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s1_pytest.log
for v in 1 0; do QF_JIT_FOLDSWZ=$v timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu > gpurun_out/s1_C5_$v.json 2>/dev/null; done
