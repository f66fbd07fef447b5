#!/bin/bash
# round 2, GPU session 1: peaks, baseline C2 bench, full-size parity (C2, C5), L2 batch probe
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s1_smi.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/peaks.cu -o /tmp/peaks && /tmp/peaks 2.0 > gpurun_out/s1_peaks.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/s1_bench_c2.json 2> gpurun_out/s1_bench_c2.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "c2 or c5" -x -q -s > gpurun_out/s1_fullsize.log 2>&1
for b in 4 8 32 128; do
  python bench.py --batch $b --steps 5 --warmup 3 --no-cpu > gpurun_out/s1_batch_$b.json 2>&1
done
