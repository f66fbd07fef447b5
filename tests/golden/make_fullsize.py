"""Generates the full-size parity fixtures tests/golden/fullsize_C{2,3,4,5}.json
(committed) for the BASELINE configurations.

TEST INFRASTRUCTURE ONLY.  Every number comes from the C restatement of the
reference hot path (oracle/, complex128, the reference's own algorithm):

  energies       energy(ansatz, theta, H)            variational.cpp:38-43
  shift_grads    gradient(..., parameter_shift)      variational.cpp:54-81, on
                 the listed components (all of them for C5)
  adjoint_grads  the oracle's CPU adjoint gradient (new math, pinned here to the
                 parameter-shift components above before it is written)

Inputs follow SURVEY.md section 8: theta row b = RngStream(1000+cfg).split(B)[b]
.normal() x P, H = tfim(chain, 1) / heisenberg(chain, 1, 1, 0.5) /
random_pauli_sum(n, T, RngStream(2000+cfg), real weights).  The GPU box cannot
run the oracle at n = 26/30 inside the test budget, hence the fixtures.

Run from the repo root (CPU only; C4 needs ~50 GB of RAM and ~2 h on 8 cores):
    python tests/golden/make_fullsize.py C2 C5 C3 C4
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CORES = os.cpu_count() or 1
CODE = "IXYZ"


def thetas(cfg_index, rows, P):
    streams = po.Rng(1000 + cfg_index).split(rows)
    return np.array([[s.normal() for _ in range(P)] for s in streams])


def ham_digest(h):
    m = hashlib.sha256()
    m.update(np.ascontiguousarray(h.codes, np.int8).tobytes())
    m.update(np.ascontiguousarray(h.wr, np.float64).tobytes())
    m.update(np.ascontiguousarray(h.wi, np.float64).tobytes())
    return m.hexdigest()


def subset(h, T):
    return po.Hamil(h.n, h.codes[:T], h.wr[:T] + 1j * h.wi[:T])


def shift_components(a, th, h, comps, parallel):
    """parameter-shift g_j = [E(theta_j + pi/2) - E(theta_j - pi/2)] / 2 (variational.cpp:72-79),
    the 2*len(comps) energies spread over `parallel` Python threads (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(j):
        tp = th.copy(); tp[j] += np.pi / 2
        tm = th.copy(); tm[j] -= np.pi / 2
        return (po.energy(a, tp, h) - po.energy(a, tm, h)) / 2.0

    with ThreadPoolExecutor(parallel) as ex:
        return np.array(list(ex.map(one, comps)))


def entry(cfg, n, layers, ham_name, h, th, E, G_adj, comps, G_shift, notes, t0):
    if G_adj is not None and len(comps):
        gs = np.abs(G_adj).max()
        dev = np.abs(G_adj[:, comps] - G_shift).max() / max(gs, 1e-300) if G_shift.size else 0.0
        assert dev < 1e-9, f"oracle adjoint disagrees with parameter shift: {dev}"
    return {"config": cfg, "n": n, "layers": layers, "ansatz": "hea", "hamiltonian": ham_name,
            "n_terms": int(len(h.wr)), "ham_sha256": ham_digest(h),
            "thetas": th.tolist(), "energies": list(map(float, E)),
            "adjoint_grads": None if G_adj is None else G_adj.tolist(),
            "shift_components": list(map(int, comps)),
            "shift_grads": None if G_shift is None else G_shift.tolist(),
            "notes": notes, "oracle_seconds": round(time.time() - t0, 1)}


def make_c2():
    t0 = time.time()
    n, ops, P = po.hea_template(20, 8)
    h = po.tfim(20, 1.0)
    th = thetas(2, 4, P)
    a = po.Ansatz(n, ops, P)
    po.lib().qo_set_inner_threads(1)
    E, G = po.energy_grad_batch(a, th, h, mode="adjoint", workers=min(CORES, 4))
    comps = list(range(0, P, P // 16))[:16]
    GS = np.array([shift_components(a, th[b], h, comps, CORES) for b in range(len(th))])
    return [entry("C2", n, 8, "tfim", h, th, E, G, comps, GS,
                  "rows 0-3 of the bench batch; full adjoint gradient pinned by 16 parameter-shift components", t0)]


def make_c5():
    t0 = time.time()
    n, ops, P = po.hea_template(16, 8)
    h = po.random_sum(16, 1000, po.Rng(2005), True)
    th = thetas(5, 8, P)
    a = po.Ansatz(n, ops, P)
    po.lib().qo_set_inner_threads(1)
    E, G = po.energy_grad_batch(a, th, h, mode="parameter_shift", workers=CORES)
    _, GA = po.energy_grad_batch(a, th, h, mode="adjoint", workers=CORES)
    comps = list(range(P))
    return [entry("C5", n, 8, "random1000", h, th, E, GA, comps, G,
                  "rows 0-7 of the bench batch; the full parameter-shift gradient (the reference algorithm)", t0)]


def make_c3():
    out = []
    po.lib().qo_set_inner_threads(CORES)
    h = po.heisenberg(26, 1.0, 1.0, 0.5)
    # depth 10 (the config): energies of bench rows 0-1
    t0 = time.time()
    n, ops, P = po.hea_template(26, 10)
    th = thetas(3, 2, P)
    a = po.Ansatz(n, ops, P)
    E = np.array([po.energy(a, th[b], h) for b in range(len(th))])
    out.append(entry("C3", n, 10, "xxz", h, th, E, None, [], None,
                     "energies at the full config (n=26, depth 10) through run(c, guard 40)", t0))
    # depth 2: full adjoint gradient pinned by 8 parameter-shift components
    t0 = time.time()
    n, ops, P = po.hea_template(26, 2)
    th = thetas(3, 1, P)
    a = po.Ansatz(n, ops, P)
    E, G = po.energy_grad_batch(a, th, h, mode="adjoint", workers=1)
    comps = list(range(0, P, P // 8))[:8]
    GS = np.array([shift_components(a, th[0], h, comps, 2)])
    out.append(entry("C3", n, 2, "xxz", h, th, E, G, comps, GS,
                     "gradient at reduced depth 2 (n=26): adjoint pinned by 8 parameter-shift components", t0))
    return out


def make_c4():
    """n = 30 at the config depth 8, on the first 20 of the 2000 terms: the energy
    and the full adjoint gradient (psi, lambda, scratch = 48 GiB of host RAM),
    pinned by one parameter-shift component.  (Depth 1 was tried first: on the
    near-product state its weight-~22 Pauli expectations are ~1e-9 sums with
    heavy cancellation, ill-conditioned even in complex128.)"""
    po.lib().qo_set_inner_threads(CORES)
    hfull = po.random_sum(30, 2000, po.Rng(2004), True)
    h = subset(hfull, 20)
    t0 = time.time()
    n, ops, P = po.hea_template(30, 8)
    th = thetas(4, 1, P)
    a = po.Ansatz(n, ops, P)
    E, G = po.energy_grad_batch(a, th, h, mode="adjoint", workers=1)
    print("C4 d8 energy + adjoint", E, time.time() - t0, flush=True)
    comps = [int(np.argmax(np.abs(G[0])))]
    GS = np.array([shift_components(a, th[0], h, comps, 1)])
    e = entry("C4", n, 8, "random2000[:20]", h, th, E, G, comps, GS,
              "energy + adjoint gradient at the full config (n=30, depth 8) on the first 20 terms of the "
              "2000-term sum; the largest gradient component pinned by parameter shift", t0)
    e["full_ham_sha256"] = ham_digest(hfull)
    return [e]


def main(argv):
    makers = {"C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}
    for cfg in argv or ["C2", "C5", "C3", "C4"]:
        t0 = time.time()
        cases = makers[cfg]()
        path = os.path.join(HERE, f"fullsize_{cfg}.json")
        with open(path, "w") as f:
            json.dump(cases, f)
        print(f"wrote {path}: {len(cases)} case(s) in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
