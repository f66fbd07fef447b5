#!/bin/bash
mkdir -p gpurun_out
python tools/sweep_times.py C2 1024 6 > gpurun_out/s6_t_carve.json 2>&1
QF_CARVEOUT=0 python tools/sweep_times.py C2 1024 6 > gpurun_out/s6_t_nocarve.json 2>&1
QF_GRAPHS=0 python tools/sweep_times.py C2 1024 6 > gpurun_out/s6_t_nographs.json 2>&1
python tools/c2_once.py C2 1024 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__maximum_warps_per_active_cycle_pct --clock-control none -k regex:qf_sweep --launch-skip 22 --launch-count 22 --csv \
    --log-file gpurun_out/s6_launch.csv python tools/c2_once.py C2 1024 > gpurun_out/s6_ncu.log 2>&1
ncu --cache-control none --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:qf_sweep --launch-skip 22 --launch-count 22 --csv \
    --log-file gpurun_out/s6_launch_nocache.csv python tools/c2_once.py C2 1024 > gpurun_out/s6_ncu2.log 2>&1
