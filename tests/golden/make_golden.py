"""Generates the golden fixtures of tests/golden/ (committed).

Sources:
  rng_known_answers.txt  -- oracle/_ref/ref_rng_driver: the reference's own
                            proj/include/qforge/rng.hpp compiled by oracle/Makefile
  vqe_fixtures.json      -- energies and parameter-shift gradients from the C
                            restatement of the reference hot path (oracle/), the
                            reference algorithm (variational.cpp:38-81) in complex128

Run from the repo root (CPU only):  python tests/golden/make_golden.py
"""
import json
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def thetas(seed, batch, P):
    streams = po.Rng(seed).split(batch)
    return np.array([[s.normal() for _ in range(P)] for s in streams])


def case(name, n, ops, P, h, th, mode="parameter_shift"):
    a = po.Ansatz(n, ops, P)
    E, G = po.energy_grad_batch(a, th, h, mode=mode, workers=os.cpu_count() or 1)
    return {"name": name, "n": n, "ops": [list(map(float, o)) for o in ops], "n_params": P,
            "codes": h.codes.tolist(), "w_re": h.wr.tolist(), "w_im": h.wi.tolist(),
            "thetas": th.tolist(), "energies": E.tolist(), "grads": G.tolist(), "grad_mode": mode}


def main():
    ref = os.path.join(ROOT, "oracle", "_ref", "rng_known_answers.txt")
    if os.path.exists(ref):
        shutil.copy(ref, os.path.join(HERE, "rng_known_answers.txt"))
    cases = []
    n, ops, P = po.hea_template(10, 4)
    cases.append(case("C1_hea10_d4_tfim_b16", n, ops, P, po.tfim(10, 1.0), thetas(1001, 16, P)))
    n, ops, P = po.tca_template(5, 2)
    r = po.Rng(3)
    cases.append(case("tca5x2_tfim1.3_seed3", n, ops, P, po.tfim(5, 1.3), np.array([[r.normal() for _ in range(P)]])))
    n, ops, P = po.hea_template(8, 3)
    cases.append(case("hea8_d3_xxz", n, ops, P, po.heisenberg(8, 1.0, 1.0, 0.5), thetas(1003, 4, P)))
    n, ops, P = po.hea_template(9, 2)
    cases.append(case("hea9_d2_random40_complexw", n, ops, P, po.random_sum(9, 40, po.Rng(2005), False),
                      thetas(1005, 3, P)))
    n, ops, P = po.tca_template(12, 2)
    cases.append(case("tca12x2_tfim_b2", n, ops, P, po.tfim(12, 1.0), thetas(1006, 2, P)))
    with open(os.path.join(HERE, "vqe_fixtures.json"), "w") as f:
        json.dump(cases, f)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
