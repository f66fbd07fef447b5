#!/bin/bash
mkdir -p gpurun_out
python tools/sweep_times.py C2 1024 6 > gpurun_out/s5_t_sust.json 2>&1
QF_PAUSE_S=0.5 python tools/sweep_times.py C2 1024 6 > gpurun_out/s5_t_pause.json 2>&1
QF_PAUSE_S=0.5 QF_JIT_NOPACK=1 python tools/sweep_times.py C2 1024 6 > gpurun_out/s5_t_pause_nopack.json 2>&1
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/s5_smi_q.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s5_parity.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
