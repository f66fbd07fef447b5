"""Randomized GPU parity stress (development): random circuits over every gate
kind with random slot bindings (shared slots, coefficients, offsets), random
constant 1q/2q unitaries, random Pauli sums (real / complex, 1..300 terms: both
the specialised and the generic H|psi> kernel), both precisions, energies and
adjoint gradients against the C oracle.  Prints failures and a summary."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

ctx = engine.Context(0)
rs = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
N_CASES = int(sys.argv[2]) if len(sys.argv) > 2 else 200
TOL = {"c128": 1e-10, "c64": 2e-5}
worst = {"c128": 0.0, "c64": 0.0}
fails = 0


def haar(d):
    z = rs.normal(size=(d, d)) + 1j * rs.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))[None, :]


t_start = time.time()
for case in range(N_CASES):
    n = int(rs.integers(2, 15))
    P = int(rs.integers(1, 12))
    ops, mats = [], []
    for _ in range(int(rs.integers(5, 70))):
        g = rs.choice(["h", "x", "y", "z", "s", "rx", "ry", "rz", "rzz", "cx", "cz", "u1", "u2", "su4"])
        q0 = int(rs.integers(0, n))
        q1 = int(rs.integers(0, n - 1))
        q1 = q1 + 1 if q1 >= q0 else q1
        if g in ("rx", "ry", "rz", "rzz"):
            two = g == "rzz"
            if rs.random() < 0.8:
                ops.append((po.GID[g], q0, q1 if two else -1, int(rs.integers(0, P)), float(rs.choice([1.0, -1.0, 0.5, 2.0])),
                            float(rs.normal()), -1))
            else:
                ops.append((po.GID[g], q0, q1 if two else -1, -1, 1.0, float(rs.normal()), -1))
        elif g in ("cx", "cz"):
            ops.append((po.GID[g], q0, q1, -1, 1.0, 0.0, -1))
        elif g in ("u1", "u2", "su4"):
            d = 2 if g == "u1" else 4
            m = np.zeros((4, 4), complex)
            m[:d, :d] = haar(d)
            mats.append(m)
            kind = po.GID["unitary"] if g != "su4" else po.GID["su4"]
            ops.append((kind, q0, q1 if d == 4 else -1, -1, 1.0, 0.0, len(mats) - 1))
        else:
            ops.append((po.GID[g], q0, -1, -1, 1.0, 0.0, -1))
    T = int(rs.choice([1, 3, 12, 40, 120, 300]))
    h = po.random_sum(n, T, po.Rng(int(rs.integers(1, 10 ** 6))), bool(rs.random() < 0.5))
    B = int(rs.integers(1, 4))
    th = rs.normal(size=(B, P))
    mv = np.array(mats) if mats else None
    try:
        E_ref, G_ref = po.energy_grad_batch(po.Ansatz(n, ops, P, mv), th, h, mode="adjoint", workers=8)
    except Exception as e:  # noqa: BLE001
        print(f"case {case}: oracle rejected: {e}", flush=True)
        continue
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    for prec in ("c128", "c64"):
        try:
            prog = engine.Program(ctx, n, ops, P, prec, mv)
            E, G = engine.energy_grad_batch(ctx, prog, obs, th)
        except Exception as e:  # noqa: BLE001
            fails += 1
            print(f"ERROR case {case} {prec}: n={n} ops={len(ops)} P={P} terms={T}: {e}", flush=True)
            np.savez(f"gpurun_out/stress_case{case}.npz", n=n, P=P, ops=np.array(ops, dtype=object),
                     mats=mv if mv is not None else np.zeros(0), codes=h.codes, wr=h.wr, wi=h.wi, th=th)
            if "CUDA" in str(e):
                sys.exit(1)  # the context is unusable after a launch failure
            continue
        scale = max(np.abs(E_ref).max(), np.abs(G_ref).max(), 1e-3 * np.abs(h.wr + 1j * h.wi).sum())
        err = max(np.abs(E - E_ref).max(), np.abs(G - G_ref).max()) / scale
        worst[prec] = max(worst[prec], err)
        if err > TOL[prec]:
            fails += 1
            print(f"FAIL case {case} {prec}: n={n} ops={len(ops)} P={P} terms={T} err={err:.3e}", flush=True)
            np.savez(f"gpurun_out/stress_case{case}.npz", n=n, P=P, ops=np.array(ops, dtype=object),
                     mats=mv if mv is not None else np.zeros(0), codes=h.codes, wr=h.wr, wi=h.wi, th=th)
print(f"cases={N_CASES} fails={fails} worst c128={worst['c128']:.2e} c64={worst['c64']:.2e} "
      f"time={time.time() - t_start:.0f}s", flush=True)
