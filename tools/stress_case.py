"""development: re-run one saved stress case (gpurun_out/stress_caseK.npz) under the current env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

d = np.load(sys.argv[1], allow_pickle=True)
n, P = int(d["n"]), int(d["P"])
ops = [tuple(o) for o in d["ops"]]
mats = d["mats"] if d["mats"].size else None
h = po.Hamil(n, d["codes"], d["wr"] + 1j * d["wi"])
th = d["th"]
E_ref, G_ref = po.energy_grad_batch(po.Ansatz(n, ops, P, mats), th, h, mode="adjoint", workers=8)
ctx = engine.Context(0)
obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
for prec in sys.argv[2:] or ["c128"]:
    prog = engine.Program(ctx, n, ops, P, prec, mats)
    E, G = engine.energy_grad_batch(ctx, prog, obs, th)
    scale = max(np.abs(E_ref).max(), np.abs(G_ref).max(), 1e-3 * np.abs(h.wr + 1j * h.wi).sum())
    print(prec, "dE", np.abs(E - E_ref).max() / scale, "dG", np.abs(G - G_ref).max() / scale, flush=True)
