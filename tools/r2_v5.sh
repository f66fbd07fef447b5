#!/bin/bash
mkdir -p gpurun_out
QF_GRAPHS=0 timeout 600 python tools/dbg_bwd_sweeps.py 30 1 c64 > gpurun_out/v5_n30.log 2>&1
