#!/usr/bin/env python
"""Development probe: psi / lambda after the first i adjoint sweeps, JIT vs AOT
programs of the same template (QF_DEBUG_BWD_STOP, qf_debug_copy_state), for
HEA depth D with the TFIM chain.  Prints the first sweep whose outputs differ and
the index bits of the largest differences.   QF_GRAPHS=0 is required.

  QF_GRAPHS=0 python tools/dbg_bwd_sweeps.py n D prec
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200 import qforge as qf  # noqa: E402
from paper_2602_14167_b200.rng import RngStream  # noqa: E402

assert os.environ.get("QF_GRAPHS") == "0"
n, D, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ops, P = bench.hea_template(n, D)
h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
ctx = engine.default_context(0)
obs = h.observable(ctx)
os.environ["QF_JIT"] = "1"
pj = engine.Program(ctx, n, ops, P, prec)
os.environ["QF_JIT"] = "0"
pa = engine.Program(ctx, n, ops, P, prec)
os.environ.pop("QF_JIT")
s = RngStream(1004).split(1)[0]
th = np.array([[s.normal() for _ in range(P)]])
nb = pj.info()
print("program", nb, flush=True)
dt = torch.complex64 if prec == "c64" else torch.complex128
N = 1 << n


def grab(which):
    t = torch.empty(N, dtype=dt, device="cuda")
    engine.check(ctx.lib.qf_debug_copy_state(ctx.handle, which, ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size()))
    return t


nbwd = nb["bwd_sweeps"] if isinstance(nb, dict) and "bwd_sweeps" in nb else 8
for stop in range(0, nbwd + 1):
    os.environ["QF_DEBUG_BWD_STOP"] = str(stop)
    res = []
    for p in (pj, pa):
        engine.energy_grad_batch(ctx, p, obs, th)
        res.append((grab(0), grab(1)))
    # global phases (the adjoint's per-gate phase trick) cancel in |psi|, |lambda| and conj(lambda) psi
    def rel_phase(a, b):  # a = e^{i alpha} b up to rounding <=> this is ~constant where |b| is not tiny
        r = a * b.conj()
        m = b.abs() > 1e-3 * b.abs().max()
        ref = r[m][0] / r[m][0].abs()
        out = torch.zeros_like(b.real)
        out[m] = ((r[m] / b[m].abs() ** 2) - ref).abs()
        return out
    cmp = (("|psi|", res[0][0].abs(), res[1][0].abs()), ("|lam|", res[0][1].abs(), res[1][1].abs()),
           ("conj(lam)psi", res[0][1].conj() * res[0][0], res[1][1].conj() * res[1][0]),
           ("psi phase", rel_phase(res[0][0], res[1][0]), torch.ones_like(res[1][0].real)),
           ("lam phase", rel_phase(res[0][1], res[1][1]), torch.ones_like(res[1][1].real)))
    for name, a, b in cmp:
        d = (a - b).abs() if not name.endswith("phase") else a
        m = float(d.max())
        scale = float(b.abs().max())
        line = f"stop={stop} {name}: max|d|={m:.3e} (max|amp| {scale:.3e})"
        if m > 1e-6 * scale:
            idx = torch.nonzero(d > 0.1 * m).flatten()[:4096].cpu().numpy()
            bits_set = [int(((idx >> q) & 1).mean() * 100) for q in range(n)]
            line += f"  {len(idx)} big; % with bit q set (q=0..n-1): {bits_set}"
        print(line, flush=True)
    del res
    torch.cuda.empty_cache()
