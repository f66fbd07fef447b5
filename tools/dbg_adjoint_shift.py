#!/usr/bin/env python
"""Development probe: the engine's adjoint gradient against the parameter-shift
rule evaluated with the engine's own energies (2P shifted rows in one batch), for
HEA depth D on the first `terms` terms (0: the TFIM chain) of random_pauli_sum(n, 2000, RngStream(2004)).
No oracle needed, so it runs at n = 30.  Prints per-n worst relative deviation and
the worst components.

  python tools/dbg_adjoint_shift.py D terms prec n1 n2 ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2602_14167_b200 import qforge as qf  # noqa: E402
from paper_2602_14167_b200.rng import RngStream  # noqa: E402

D, terms, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
for n in map(int, sys.argv[4:]):
    if terms == 0:
        h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
    else:
        full = qf.random_pauli_sum(n, 2000 if n == 30 else terms, RngStream(2004), True)
        h = qf.PauliSum(n)
        for t in full.terms[:terms]:
            h.add(t.weight, t.codes)
    a = qf.hea_ansatz(n, D)
    P = a.n_params
    s = RngStream(1004).split(1)[0]
    th = np.array([[s.normal() for _ in range(P)]])
    E, G = qf.energy_gradient_batch(a, th, h, grads=True, precision=prec)
    rows = np.repeat(th, 2 * P, axis=0)
    for j in range(P):
        rows[2 * j, j] += np.pi / 2
        rows[2 * j + 1, j] -= np.pi / 2
    Es = []
    for c in range(0, 2 * P, 16):
        e, _ = qf.energy_gradient_batch(a, rows[c:c + 16], h, grads=False, precision=prec)
        Es.append(e)
    Es = np.concatenate(Es)
    S = (Es[0::2] - Es[1::2]) / 2
    g = G[0]
    dev = np.abs(g - S)
    print(f"n={n} D={D} terms={terms} {prec}: E={E[0]:.6e} max|g|={np.abs(S).max():.3e} "
          f"max|dg|/max|g|={dev.max() / np.abs(S).max():.3e}", flush=True)
    worst = np.argsort(-dev)[:6]
    print("   worst comps", [(int(j), f"{g[j]:.4e}", f"{S[j]:.4e}") for j in worst], flush=True)
    for per_ctx in list(a._programs.values()):
        for p in per_ctx.values():
            p.close()
