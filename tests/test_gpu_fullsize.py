"""Full-size parity at the BASELINE configurations:
the CUDA path, driven through the drop-in Python mirror exactly as a user would
(qforge.hea_ansatz + the reference's Hamiltonian builders + energy_gradient_batch),
against committed oracle fixtures (tests/golden/fullsize_C*.json, generated on
the CPU by tests/golden/make_fullsize.py: the reference algorithm restated in C,
complex128).

Tolerances are the north-star ones, norm-wise (test_gpu_parity.py explains why):
complex64 1e-5, complex128 1e-11:
  |dE|_inf <= tol * max(|E_ref|_inf, |g_ref|_inf)      (energy-only cases: |E_ref|_inf)
  |dg|_inf <= tol * |g_ref|_inf
Every fixture also carries the reference's own parameter-shift gradient on a
subset of components (the whole gradient for C5), checked the same way."""
import json
import os

import numpy as np
import pytest

from paper_2602_14167_b200 import engine
from paper_2602_14167_b200 import qforge as qf
from paper_2602_14167_b200.rng import RngStream

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = {"c128": 1e-11, "c64": 1e-5}


def _fixture(cfg):
    path = os.path.join(HERE, "golden", f"fullsize_{cfg}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path}: run tests/golden/make_fullsize.py {cfg}")
    return json.load(open(path))


def _hamiltonian(case):
    import hashlib
    n, name = case["n"], case["hamiltonian"]
    if name == "tfim":
        h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
    elif name == "xxz":
        h = qf.heisenberg_terms(qf.build_lattice("chain", [n], [False]), 1.0, 1.0, 0.5)
    else:  # random<T>[:k]: random_pauli_sum(n, T, RngStream(2000 + cfg)), first k terms
        T = int(name[6:].split("[")[0])
        cfg_index = int(case["config"][1])
        full = qf.random_pauli_sum(n, T, RngStream(2000 + cfg_index), True)
        keep = int(name.split("[:")[1].rstrip("]")) if "[:" in name else T
        h = qf.PauliSum(n)
        for t in full.terms[:keep]:
            h.add(t.weight, t.codes)
    codes, w = h.arrays()
    m = hashlib.sha256()
    m.update(np.ascontiguousarray(codes, np.int8).tobytes())
    m.update(np.ascontiguousarray(w.real, np.float64).tobytes())
    m.update(np.ascontiguousarray(w.imag, np.float64).tobytes())
    assert m.hexdigest() == case["ham_sha256"], "Hamiltonian differs from the fixture's inputs"
    return h


def _thetas(case):
    th = np.array(case["thetas"])
    cfg_index = int(case["config"][1])
    streams = RngStream(1000 + cfg_index).split(th.shape[0])  # SURVEY.md 8 seeds
    mine = np.array([[s.normal() for _ in range(th.shape[1])] for s in streams])
    assert np.array_equal(mine, th), "theta rows differ from the fixture's inputs"
    return th


def _run(case, prec, grads):
    ansatz = qf.hea_ansatz(case["n"], case["layers"])
    h = _hamiltonian(case)
    th = _thetas(case)
    E, G = qf.energy_gradient_batch(ansatz, th, h, grads=grads, precision=prec)
    for per_ctx in list(ansatz._programs.values()):
        for p in per_ctx.values():
            p.close()
    return E, G


def _check(case, prec, E, G):
    tol = TOL[prec]
    Er = np.array(case["energies"])
    Ga = None if case["adjoint_grads"] is None else np.array(case["adjoint_grads"])
    gs = np.abs(Ga).max() if Ga is not None else 0.0
    scale = max(np.abs(Er).max(), gs)
    dE = np.abs(E - Er).max() / scale
    assert dE <= tol, (case["config"], case["layers"], prec, "energy", dE)
    out = {"dE": dE}
    if Ga is not None:
        dG = np.abs(G - Ga).max() / gs
        assert dG <= tol, (case["config"], case["layers"], prec, "adjoint gradient", dG)
        comps = case["shift_components"]
        S = np.array(case["shift_grads"])
        dS = np.abs(G[:, comps] - S).max() / gs
        assert dS <= tol, (case["config"], case["layers"], prec, "parameter-shift components", dS)
        out.update(dG=dG, dS=dS)
    print(case["config"], "layers", case["layers"], prec, {k: f"{v:.2e}" for k, v in out.items()})


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_c2_full_config(prec):
    """C2: n=20, HEA depth 8 (P=320), TFIM 39 terms; bench rows 0-3."""
    for case in _fixture("C2"):
        E, G = _run(case, prec, True)
        _check(case, prec, E, G)


def test_c5_full_config_c128():
    """C5: n=16, HEA depth 8 (P=256), random 1000-term sum, complex128; the full
    parameter-shift gradient of 8 bench rows (the reference algorithm) at 1e-11."""
    for case in _fixture("C5"):
        E, G = _run(case, "c128", True)
        _check(case, "c128", E, G)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_c3_full_config(prec):
    """C3: n=26, XXZ (75 terms): energies at depth 10 (the config), gradient at depth 2."""
    for case in _fixture("C3"):
        grads = case["adjoint_grads"] is not None
        E, G = _run(case, prec, grads)
        _check(case, prec, E, G)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_c4_full_config(prec):
    """C4: n=30 (8 GiB complex64 state): energy at depth 8 on the first 20 terms of
    the 2000-term random sum, gradient at depth 1."""
    for case in _fixture("C4"):
        grads = case["adjoint_grads"] is not None
        E, G = _run(case, prec, grads)
        _check(case, prec, E, G)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_n30_adjoint_matches_parameter_shift_of_engine_energies(prec):
    """Regression (round 2): at n >= 29 the generated sweeps indexed HBM as
    `st[g | C]` (32-bit) with C * sizeof(amplitude) >= 2^31; the compiler split
    the constant out of the address and wrapped it, corrupting the last adjoint
    sweep (tools/micro/sweep_harness.cu).  TFIM chain, HEA depth 1, n = 30: the
    adjoint gradient against the parameter-shift rule (variational.cpp:72-79) on
    the engine's own energies, on the components whose taps sit in the sweeps
    that touch the top memory bits (qubits 0-2 ry / rz) and a few others."""
    n = 30
    a = qf.hea_ansatz(n, 1)
    h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
    P = a.n_params
    s = RngStream(1004).split(1)[0]
    th = np.array([[s.normal() for _ in range(P)]])
    E, G = qf.energy_gradient_batch(a, th, h, grads=True, precision=prec)
    comps = [0, 1, 2, 12, 29, 30, 31, 32, 45, 59]
    rows = np.repeat(th, 2 * len(comps), axis=0)
    for i, j in enumerate(comps):
        rows[2 * i, j] += np.pi / 2
        rows[2 * i + 1, j] -= np.pi / 2
    Es, _ = qf.energy_gradient_batch(a, rows, h, grads=False, precision=prec)
    S = (Es[0::2] - Es[1::2]) / 2
    scale = np.abs(G[0]).max()
    d = np.abs(G[0, comps] - S).max() / scale
    assert d <= TOL[prec], (prec, d)
    for per_ctx in list(a._programs.values()):
        for p in per_ctx.values():
            p.close()
