#!/bin/bash
mkdir -p gpurun_out
QF_CARVEOUT=0 QF_GRAPHS=0 QF_DEV_BWD_PAUSE_US=200000 python tools/sweep_times.py C2 1024 4 > gpurun_out/s7_t_bwdpause.json 2>&1
QF_CARVEOUT=0 QF_GRAPHS=0 python tools/sweep_times.py C2 1024 4 > gpurun_out/s7_t_ref.json 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 20 > gpurun_out/s7_smi_trace.csv &
SMI=$!
QF_CARVEOUT=0 python tools/sweep_times.py C2 1024 10 > gpurun_out/s7_t_trace.json 2>&1
kill $SMI
