"""development: C2 per-eval throughput vs batch size (one context, host buffers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

cfg = bench.CONFIGS["C2"]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian("C2", cfg)
th = bench.thetas_for("C2", 1024, P)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, "c64")
obs = h.observable(ctx)
engine.energy_grad_batch(ctx, prog, obs, th)
for B in [64, 128, 256, 512, 1024]:
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        engine.energy_grad_batch(ctx, prog, obs, th[:B])
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    print(f"B={B:5d} {best*1000:8.1f} ms  {B/best:7.0f} evals/s", flush=True)
