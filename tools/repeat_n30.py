"""development: repeat the n=30 product-ansatz evaluation; print G[0..3] each time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200.rng import RngStream  # noqa: E402
from test_gpu_parity import _product_ansatz, _product_energy_and_grad  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ctx = engine.default_context(0)
ops, P = _product_ansatz(n)
rng = po.Rng(4000 + n)
T = 40
codes = np.zeros((T, n), np.int8)
for t in range(T):
    for _ in range(1 + rng.uniform_below(3)):
        codes[t, rng.uniform_below(n)] = 1 + rng.uniform_below(3)
w = np.array([rng.normal() for _ in range(T)])
th = np.array([RngStream(7).split(1)[0].normal() for _ in range(P)])
Er, Gr = _product_energy_and_grad(n, th, codes, w)
prog = engine.Program(ctx, n, ops, P, "c64")
obs = engine.Observable(ctx, n, codes, w)
print("ref", Gr[:4])
for r in range(4):
    E, G = engine.energy_grad_batch(ctx, prog, obs, th[None, :])
    print(r, G[0, :4], E[0] - Er)
