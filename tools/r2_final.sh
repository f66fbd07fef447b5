#!/bin/bash
# Round-2 end verification of HEAD on one B200: smoke, GPU tests, C++ drop-in,
# bench (ours + reference arm), torchrun single-rank bench, ncu launch list and
# full captures of the dominant sweep and of H|psi>, MIPT / noise benches.
mkdir -p gpurun_out
bash tools/verify_round.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/f_torchrun.log 2>&1; echo torchrun=$? >> gpurun_out/f_torchrun.log
bash tools/profile_c2.sh > gpurun_out/prof_steps.log 2>&1
timeout 600 python tools/bench_mipt.py > gpurun_out/f_mipt.json 2>&1
timeout 600 python tools/bench_noise.py > gpurun_out/f_noise.jsonl 2>&1
for cfg in C1 C3 C4 C5; do timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/f_bench_$cfg.json 2> gpurun_out/f_bench_$cfg.err; done
