#!/usr/bin/env python
"""Development check: n = 20 MIPT entropies (own eigen-solver) against the numpy
oracle for a few trajectories of the Table IV configuration."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

ctx = engine.default_context(0)
n, D, p, T, seed = 20, 40, 0.1, int(sys.argv[1]) if len(sys.argv) > 1 else 3, 2026
t0 = time.perf_counter()
ref = po.mipt_haar(n, D, p, T, seed)
t1 = time.perf_counter()
for prec in ("c128", "c64"):
    got, _ = engine.mipt_haar(ctx, n, D, p, T, seed, prec)
    print(prec, "max |dS| =", np.abs(got - ref).max(), "ref", ref[:4], "got", got[:4])
print("oracle s:", t1 - t0)
