"""development: closed-form product-ansatz gradient check over n (c64/c128)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200.rng import RngStream  # noqa: E402
from test_gpu_parity import _product_ansatz, _product_energy_and_grad  # noqa: E402

ctx = engine.default_context(0)
for prec in sys.argv[2:] or ["c64"]:
    for n in [int(x) for x in sys.argv[1].split(",")]:
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
        E, G = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, prec), engine.Observable(ctx, n, codes, w),
                                        th[None, :])
        err = np.abs(G[0] - Gr)
        bad = np.nonzero(err > 1e-5 * np.abs(Gr).max())[0]
        print(prec, n, "dE", abs(E[0] - Er) / max(abs(Er), 1e-30), "dG", err.max() / np.abs(Gr).max(), "bad", bad[:10],
              flush=True)
