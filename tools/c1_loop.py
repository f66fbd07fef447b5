"""development: C1 per-call wall time in a tight loop (launch-bound regime)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

mode = os.environ.get("C1_MODE", "plain")
if mode != "plain":
    import torch
    if mode in ("cuda", "device"):
        torch.zeros(1, device="cuda")
    if mode == "device":
        torch.cuda.set_device(0)
cfg = bench.CONFIGS["C1"]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian("C1", cfg)
th = bench.thetas_for("C1", cfg["batch"], P)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, cfg["prec"])
obs = h.observable(ctx)
for _ in range(20):
    engine.energy_grad_batch(ctx, prog, obs, th)
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(200):
        engine.energy_grad_batch(ctx, prog, obs, th)
    dt = (time.perf_counter() - t0) / 200
    ctx.reset_stats()
    engine.energy_grad_batch(ctx, prog, obs, th)
    print(f"mode={mode} QF_GRAPHS={os.environ.get('QF_GRAPHS', '1')} {dt*1e6:.1f} us/call  {cfg['batch']/dt:.0f} evals/s  "
          f"launches/call={ctx.stats()[0]}", flush=True)
ctx.set_timing(True)
ctx.reset_stats()
t0 = time.perf_counter()
for _ in range(50):
    engine.energy_grad_batch(ctx, prog, obs, th)
dt = (time.perf_counter() - t0) / 50
st = ctx.stats()
print("timed: wall/call", round(dt * 1e6, 1), "us; gpu class ms per call", [round(x / 50 * 1000, 1) for x in st[2]], "us")
