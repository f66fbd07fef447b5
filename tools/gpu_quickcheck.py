"""Quick GPU parity sweep used during development: prints, does not stop at first failure."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as po
from paper_2602_14167_b200 import engine
from paper_2602_14167_b200.rng import RngStream

ctx = engine.Context(0)

def check(name, n, ops, P, h, B=3, precs=("c128", "c64"), seed=1, mats=None):
    rng = RngStream(seed).split(B)
    thetas = np.array([[r.normal() for _ in range(P)] for r in rng]) if P else np.zeros((B, 0))
    ref = po.Ansatz(n, ops, P, mats)
    t0 = time.time()
    E_ref, G_ref = po.energy_grad_batch(ref, thetas, h, mode="adjoint" if n > 12 else "parameter_shift", workers=8)
    tr = time.time() - t0
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    for prec in precs:
        try:
            prog = engine.Program(ctx, n, ops, P, prec, mats)
            t0 = time.time()
            E, G = engine.energy_grad_batch(ctx, prog, obs, thetas)
            tg = time.time() - t0
            scale = max(np.abs(E_ref).max(), np.abs(G_ref).max() if P else 0, 1e-300)
            eE = np.abs(E - E_ref).max() / scale
            eG = np.abs(G - G_ref).max() / max(np.abs(G_ref).max(), 1e-300) if P else 0
            print(f"{name:28s} {prec}: dE={eE:.2e} dG={eG:.2e} info={prog.info()} jit={prog.jit_status()['active']} t_ref={tr:.2f}s t_gpu={tg:.3f}s E0={E[0]:.6f}/{E_ref[0]:.6f}", flush=True)
        except Exception as e:
            print(f"{name:28s} {prec}: EXC {e}", flush=True)
            traceback.print_exc()

for n in (1, 2, 3, 5, 8, 10, 13, 14, 16):
    if n >= 2:
        _, ops, P = po.hea_template(n, 2)
        check(f"hea n={n}", n, ops, P, po.tfim(n, 1.0))
        _, ops, P = po.tca_template(n, 2)
        check(f"tca n={n}", n, ops, P, po.heisenberg(n, 1.0, 1.0, 0.5))
    rs = po.random_sum(n, 20, po.Rng(5 + n), real_weights=True)
    _, ops, P = po.hea_template(max(n, 2), 1) if n >= 2 else (1, [(6, 0, -1, 0, 1.0, 0.0, -1), (7, 0, -1, 1, 1.0, 0.0, -1)], 2)
    check(f"rand20 n={n}", n, ops, P, rs)
for n in (18, 20):
    _, ops, P = po.hea_template(n, 2)
    check(f"hea n={n}", n, ops, P, po.tfim(n, 1.0), B=2)
    rs = po.random_sum(n, 30, po.Rng(77), real_weights=True)
    check(f"rand30 n={n}", n, ops, P, rs, B=2)
