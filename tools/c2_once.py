#!/usr/bin/env python
"""Two host-buffer evaluations of a bench config at a given batch (profiling
driver: the first call JIT-compiles, ncu --launch-skip 22 skips it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = bench.CONFIGS[cfg_name]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian(cfg_name, cfg)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, cfg["prec"])
obs = h.observable(ctx)
th = bench.thetas_for(cfg_name, B, P)
for _ in range(2):
    e, g = engine.energy_grad_batch(ctx, prog, obs, th)
print("E0", e[0], "sweeps", prog.info() if hasattr(prog, "info") else "")
