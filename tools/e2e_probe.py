"""development: C2 B=1024 host-buffer evals/s with / without torch imported and
with / without the nvidia-smi sampler thread (bench.py measurement overhead)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
if "torch" in mode:
    import torch  # noqa: F401
    if "nocuda" not in mode:
        torch.zeros(1, device="cuda")
cfg = bench.CONFIGS["C2"]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian("C2", cfg)
th = bench.thetas_for("C2", 1024, P)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, "c64")
obs = h.observable(ctx)
for _ in range(3):
    engine.energy_grad_batch(ctx, prog, obs, th)
sampler = None
if "smi" in mode:
    sampler = bench.ClockSampler(0)
    sampler.start()
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    engine.energy_grad_batch(ctx, prog, obs, th)
    ts.append(time.perf_counter() - t0)
if sampler:
    sampler.stop()
print(mode, " ".join(f"{1024 / t:.0f}" for t in ts), flush=True)
