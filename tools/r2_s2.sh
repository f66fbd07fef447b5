#!/bin/bash
# round 2, GPU session 2: peaks v2, parity after the deferred-relabel change, A/B of defer / packed FP32
mkdir -p gpurun_out
./tools/micro/peaks_bin 1.5 > gpurun_out/s2_peaks.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not c3 and not c4" -x -q > gpurun_out/s2_parity.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s2_bench_defer.json 2>&1
QF_JIT_NODEFER=1 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s2_bench_nodefer.json 2>&1
QF_JIT_NOPACK=1 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s2_bench_nopack.json 2>&1
