#!/bin/bash
# timing probes: where the adjoint sweep time goes (results of probe runs are wrong by design)
mkdir -p gpurun_out
QF_JIT_NOILV=1 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/p4_base.json 2>&1
QF_JIT_NOILV=1 QF_JIT_PROBE_NOFLUSH=1 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/p4_noflush.json 2>&1
QF_JIT_NOILV=1 QF_JIT_PROBE_NOSTS=1 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/p4_nosts.json 2>&1
QF_JIT_NOILV=1 QF_JIT_PROBE_NOSTS=1 QF_JIT_PROBE_NOFLUSH=1 timeout 600 python tools/sweep_times.py C2 1024 4 > gpurun_out/p4_both.json 2>&1
