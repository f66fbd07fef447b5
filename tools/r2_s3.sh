#!/bin/bash
# round 2, GPU session 3: sharding tests, C3 full size, per-sweep launch lists (packed vs scalar FP32)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_fullsize.py -k "virtual or device_entry or nccl or c3" -x -q -s > gpurun_out/s3_tests.log 2>&1
python tools/c2_once.py C2 1024 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qf_ --launch-skip 23 --launch-count 23 --csv \
    --log-file gpurun_out/s3_launch_defer.csv python tools/c2_once.py C2 1024 > gpurun_out/s3_ncu1.log 2>&1
QF_JIT_NOPACK=1 python tools/c2_once.py C2 64 > /dev/null 2>&1
QF_JIT_NOPACK=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qf_ --launch-skip 23 --launch-count 23 --csv \
    --log-file gpurun_out/s3_launch_nopack.csv python tools/c2_once.py C2 1024 > gpurun_out/s3_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 32 --launch-count 2 \
    -o gpurun_out/s3_bwd01 python tools/c2_once.py C2 256 > gpurun_out/s3_ncu3.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s3_bench.json 2>&1
