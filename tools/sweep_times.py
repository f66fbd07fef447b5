#!/usr/bin/env python
"""Per-launch device times of one bench config in a sustained run (timing level
2: CUDA events around every sweep / H|psi> launch on the engine stream), next to
the un-instrumented step time, NVML clocks and power.  Development tool.

  python tools/sweep_times.py [C2] [batch] [steps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = dict(bench.CONFIGS[cfg_name])
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["batch"]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
pause = float(os.environ.get("QF_PAUSE_S", "0"))  # idle GPU time between evaluations (power/thermal probe)
import torch  # noqa: E402

ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian(cfg_name, cfg)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, cfg["prec"])
obs = h.observable(ctx)
dev = torch.device("cuda", 0)
th = torch.tensor(bench.thetas_for(cfg_name, B, P), device=dev)
E = torch.zeros(B, dtype=torch.float64, device=dev)
G = torch.zeros((B, P), dtype=torch.float64, device=dev)
ext = torch.cuda.ExternalStream(ctx.stream, device=dev)


def run(k):
    for _ in range(k):
        with torch.cuda.stream(ext):
            engine.energy_grad_batch_device(ctx, prog, obs, th, E, G)
        if pause:
            torch.cuda.synchronize()
            time.sleep(pause)
    torch.cuda.synchronize()


clk = bench.ClockSampler(0)
run(3)
t0 = time.perf_counter()
run(steps)
plain = (time.perf_counter() - t0) / steps * 1e3
clk.start()
ctx.reset_stats()
ctx.set_timing(2)
run(steps)
lt = ctx.launch_times()
ctx.set_timing(0)
c = clk.stop()
out = {"config": cfg_name, "batch": B, "pause_s": pause, "plain_ms_per_step": plain, "clocks": c,
       "env": {k: v for k, v in os.environ.items() if k.startswith("QF_")},
       "launch_ms": {str(k): round(v[0] / v[1], 4) for k, v in sorted(lt.items())}}
tot = sum(v[0] / v[1] for v in lt.values())
out["sum_launch_ms"] = tot
print(json.dumps(out))
