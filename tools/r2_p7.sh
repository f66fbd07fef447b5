#!/bin/bash
mkdir -p gpurun_out
QF_JIT_NOPACK=1 timeout 600 python tools/sweep_times.py C2 1024 6 > gpurun_out/p7_nopack.json 2>&1
