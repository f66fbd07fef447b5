"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, the
committed golden fixtures and size-independent properties.

Tolerances (north star): complex128 <= 1e-11, complex64 <= 1e-5, relative,
norm-wise for gradients: |dg|_inf <= tol * |g_ref|_inf, |dE| <= tol * max(|E_ref|, |g_ref|_inf)
(SURVEY.md 7 explains why component-wise relative error is ill-posed)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import engine
from paper_2602_14167_b200.rng import RngStream

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-11, "c64": 1e-5}
HERE = os.path.dirname(os.path.abspath(__file__))


def thetas(seed, batch, P):
    return np.array([[s.normal() for _ in range(P)] for s in RngStream(seed).split(batch)])


def check(E, G, Er, Gr, prec):
    tol = TOL[prec]
    gs = np.abs(Gr).max() if Gr is not None and Gr.size else 0.0
    scale = max(np.abs(Er).max(), gs, 1e-300)
    assert np.abs(E - Er).max() <= tol * scale, (np.abs(E - Er).max() / scale, prec)
    if Gr is not None and Gr.size:
        assert np.abs(G - Gr).max() <= tol * max(gs, 1e-300), (np.abs(G - Gr).max() / gs, prec)


@pytest.fixture(params=["jit", "aot"])
def path(request, monkeypatch):
    monkeypatch.setenv("QF_JIT", "2" if request.param == "jit" else "0")
    return request.param


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_golden_fixtures(ctx, prec, path):
    cases = json.load(open(os.path.join(HERE, "golden", "vqe_fixtures.json")))
    for c in cases:
        ops = [tuple(int(v) if i in (0, 1, 2, 3, 6) else v for i, v in enumerate(o)) for o in c["ops"]]
        prog = engine.Program(ctx, c["n"], ops, c["n_params"], prec)
        assert prog.jit_status()["active"] == (path == "jit")
        obs = engine.Observable(ctx, c["n"], np.array(c["codes"], np.int8),
                                np.array(c["w_re"]) + 1j * np.array(c["w_im"]))
        E, G = engine.energy_grad_batch(ctx, prog, obs, np.array(c["thetas"]))
        check(E, G, np.array(c["energies"]), np.array(c["grads"]), prec)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_config_c1_full_vs_oracle_parameter_shift(ctx, prec):
    """C1: 10-qubit HEA depth 4, TFIM, batch 16 (the CPU-reference config)."""
    n, ops, P = po.hea_template(10, 4)
    h = po.tfim(10, 1.0)
    th = thetas(1001, 16, P)
    Er, Gr = po.energy_grad_batch(po.Ansatz(n, ops, P), th, h, mode="parameter_shift", workers=os.cpu_count())
    E, G = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, prec),
                                    engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi), th)
    check(E, G, Er, Gr, prec)


@pytest.mark.parametrize("n,depth,ham,batch,prec", [
    (20, 2, "tfim", 3, "c64"), (20, 2, "tfim", 2, "c128"),       # C2 family (reduced depth)
    (16, 3, "random1000", 2, "c128"),                              # C5 family (reduced depth)
    (22, 1, "xxz", 1, "c64"),                                      # C3 family (reduced size)
])
def test_config_families_vs_oracle(ctx, n, depth, ham, batch, prec):
    _, ops, P = po.hea_template(n, depth)
    if ham == "tfim":
        h = po.tfim(n, 1.0)
    elif ham == "xxz":
        h = po.heisenberg(n, 1.0, 1.0, 0.5)
    else:
        h = po.random_sum(n, int(ham[6:]), po.Rng(2005), True)
    th = thetas(1000 + n, batch, P)
    Er, Gr = po.energy_grad_batch(po.Ansatz(n, ops, P), th, h, mode="adjoint", workers=os.cpu_count())
    E, G = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, prec),
                                    engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi), th)
    check(E, G, Er, Gr, prec)


def _product_ansatz(n):
    ops, k = [], 0
    for q in range(n):
        ops.append((po.GID["ry"], q, -1, k, 1.0, 0.0, -1)); k += 1
        ops.append((po.GID["rz"], q, -1, k, 1.0, 0.0, -1)); k += 1
    return ops, k


def _product_energy_and_grad(n, th, codes, w):
    """Closed form for a product state ry(a) rz(b) |0>: <X> = sin a cos b,
    <Y> = sin a sin b, <Z> = cos a; E = sum_t w_t prod_q <P_q>."""
    a, b = th[0::2], th[1::2]
    ex = np.stack([np.ones(n), np.sin(a) * np.cos(b), np.sin(a) * np.sin(b), np.cos(a)])
    da = np.stack([np.zeros(n), np.cos(a) * np.cos(b), np.cos(a) * np.sin(b), -np.sin(a)])
    db = np.stack([np.zeros(n), -np.sin(a) * np.sin(b), np.sin(a) * np.cos(b), np.zeros(n)])
    E = 0.0
    g = np.zeros(2 * n)
    for t in range(len(w)):
        f = ex[codes[t], np.arange(n)]
        E += w[t] * np.prod(f)
        for q in range(n):
            rest = np.prod(np.delete(f, q))
            g[2 * q] += w[t] * da[codes[t][q], q] * rest
            g[2 * q + 1] += w[t] * db[codes[t][q], q] * rest
    return E, g


@pytest.mark.parametrize("n,prec", [(30, "c64"), (24, "c128")])
def test_large_state_product_closed_form(ctx, n, prec):
    """C4 scale (n = 30, 8 GiB complex64 state): closed-form energy and gradient of
    a product ansatz under a random Pauli sum with low-weight terms (size-independent
    property; the CPU oracle cannot evaluate 2^30 amplitudes in test time)."""
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
    E, G = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, prec),
                                    engine.Observable(ctx, n, codes, w), th[None, :])
    check(E, G, np.array([Er]), Gr[None, :], prec)


def test_gradient_matches_finite_differences_of_gpu_energies(ctx):
    """Self-consistency at a size the oracle cannot reach quickly (n = 26, c128)."""
    n, depth = 26, 1
    _, ops, P = po.hea_template(n, depth)
    h = po.heisenberg(n, 1.0, 1.0, 0.5)
    prog = engine.Program(ctx, n, ops, P, "c128")
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    th = thetas(1003, 1, P)[0]
    E, G = engine.energy_grad_batch(ctx, prog, obs, th[None, :])
    js = [0, 7, 25, 26, 40, P - 1]
    eps = 1e-4
    T = np.repeat(th[None, :], 2 * len(js), axis=0)
    for i, j in enumerate(js):
        T[2 * i, j] += eps
        T[2 * i + 1, j] -= eps
    Es, _ = engine.energy_grad_batch(ctx, prog, obs, T, grads=False)
    fd = (Es[0::2] - Es[1::2]) / (2 * eps)
    assert np.abs(fd - G[0, js]).max() <= 1e-7 * max(1.0, np.abs(G).max())


def test_batch_composition_chunking_and_repeat_are_bitwise_invariant(ctx):
    """parallel.hpp:9-10 (results never depend on the worker split): entry b's
    result is bitwise identical alone, in a batch, split into chunks, repeated."""
    n, ops, P = po.hea_template(16, 2)
    h = po.tfim(16, 1.0)
    th = thetas(77, 6, P)
    prog = engine.Program(ctx, n, ops, P, "c64")
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    E, G = engine.energy_grad_batch(ctx, prog, obs, th)
    E2, G2 = engine.energy_grad_batch(ctx, prog, obs, th)
    assert np.array_equal(E, E2) and np.array_equal(G, G2)
    E1, G1 = engine.energy_grad_batch(ctx, prog, obs, th[3:4])
    assert np.array_equal(E1[0], E[3]) and np.array_equal(G1[0], G[3])
    ctx.set_memory_budget(3 * (1 << 16) * 8 * 2)  # forces chunks of ~2 entries
    try:
        E3, G3 = engine.energy_grad_batch(ctx, prog, obs, th)
    finally:
        ctx.set_memory_budget(0)
    assert np.array_equal(E, E3) and np.array_equal(G, G3)


def test_jit_and_aot_kernels_agree(ctx, monkeypatch):
    n, ops, P = po.tca_template(14, 3)
    h = po.random_sum(14, 60, po.Rng(9), False)
    th = thetas(5, 3, P)
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    monkeypatch.setenv("QF_JIT", "2")
    Ej, Gj = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, "c128"), obs, th)
    monkeypatch.setenv("QF_JIT", "0")
    Ea, Ga = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, "c128"), obs, th)
    check(Ej, Gj, Ea, Ga, "c128")


def test_device_buffers_match_host_api(ctx):
    import torch
    n, ops, P = po.hea_template(12, 2)
    h = po.tfim(12, 0.8)
    th = thetas(3, 5, P)
    prog = engine.Program(ctx, n, ops, P, "c64")
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    E, G = engine.energy_grad_batch(ctx, prog, obs, th)
    dth = torch.tensor(th, device="cuda:0")
    dE = torch.zeros(5, dtype=torch.float64, device="cuda:0")
    dG = torch.zeros(5, P, dtype=torch.float64, device="cuda:0")
    s = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
    with torch.cuda.stream(s):
        engine.energy_grad_batch_device(ctx, prog, obs, dth, dE, dG)
    torch.cuda.synchronize()
    assert np.array_equal(dE.cpu().numpy(), E) and np.array_equal(dG.cpu().numpy(), G)


def test_all_gate_kinds_state_and_expectation(ctx):
    """run() and expectation_pauli over every qubit gate kind, multi-sweep
    schedule (small tiles), both precisions, vs the oracle."""
    G_ = po.GID
    rng = np.random.default_rng(3)
    u4 = np.linalg.qr(rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))[0]
    u2 = np.linalg.qr(rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2)))[0]
    m2 = np.zeros((4, 4), complex)
    m2[:2, :2] = u2
    ops = []
    for layer in range(3):
        for q in range(15):
            k = [G_["h"], G_["x"], G_["y"], G_["z"], G_["s"], G_["rx"], G_["ry"], G_["rz"]][(q + layer) % 8]
            ops.append((k, q, -1, -1, 1.0, 0.3 * q + layer, -1))
        for q in range(layer % 2, 14, 2):
            k = [G_["cx"], G_["cz"], G_["rzz"], G_["unitary"]][(q // 2 + layer) % 4]
            ops.append((k, q, q + 1, -1, 1.0, 0.7, 0 if k == G_["unitary"] else -1))
        ops.append((G_["unitary"], 4, -1, -1, 1.0, 0.0, 1))
        ops.append((G_["cx"], 14, 0, -1, 1.0, 0.0, -1))
    mats = [u4, m2]
    ref = po.run(15, ops, mats=np.array(mats))
    h = po.random_sum(15, 30, po.Rng(12), False)
    eref = po.expectation(15, ref, h)
    for prec in ("c128", "c64"):
        prog = engine.Program(ctx, 15, ops, 0, prec, mats=np.array(mats))
        psi = engine.run_state(ctx, prog, np.zeros(0), 40)
        assert np.abs(psi - ref).max() <= TOL[prec], (prec, np.abs(psi - ref).max())
        e = engine.expectation(ctx, prog, engine.Observable(ctx, 15, h.codes, h.wr + 1j * h.wi), np.zeros(0))
        assert abs(e - eref) <= TOL[prec] * max(1.0, abs(eref)), (prec, abs(e - eref))


def test_pauli_sum_to_coo_matches_oracle(ctx):
    """pauli_sum_to_coo (pauli.cpp:89-153): identical canonical triplets."""
    from paper_2602_14167_b200 import qforge as qf
    cases = [po.tfim(10, 1.3), po.heisenberg(9, 1.0, 0.5, 0.25), po.random_sum(8, 40, po.Rng(3), False),
             po.random_sum(7, 300, po.Rng(4), True),  # 300 terms: block-per-row sort path
             po.random_sum(9, 50, po.Rng(5), False),  # 33..64 groups: thread-per-row path
             po.random_sum(1, 3, po.Rng(6), False), po.random_sum(2, 9, po.Rng(7), True)]
    # exact cancellations: XX + YY vanishes on rows with equal bits, Z0 - Z1 likewise
    codes = np.zeros((6, 5), np.int8)
    codes[0, :2] = 1
    codes[1, :2] = 2
    codes[2, 0] = 3
    codes[3, 1] = 3
    codes[4, 3] = 1
    codes[5, 2:4] = [1, 3]
    cases.append(po.Hamil(5, codes, np.array([1.0, 1.0, 0.5, -0.5, 0.25, 0.25 + 0.5j])))
    for ho in cases:
        r0, c0, v0 = po.pauli_sum_to_coo(ho)
        r, c, v = engine.pauli_sum_to_coo(ctx, engine.Observable(ctx, ho.n, ho.codes, ho.wr + 1j * ho.wi))
        assert np.array_equal(r, r0) and np.array_equal(c, c0)
        assert np.abs(v - v0).max() <= 1e-12 * max(1.0, np.abs(v0).max())
    h = qf.tfim_terms(qf.build_lattice("chain", [6], [False]), 0.7)
    coo = qf.pauli_sum_to_coo(h)
    codes, w = h.arrays()
    P = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1, -1])]
    dense = np.zeros((64, 64), complex)
    for t in range(len(w)):
        m = np.eye(1)
        for cc in codes[t]:
            m = np.kron(m, P[cc])
        dense += w[t] * m
    assert np.abs(coo.to_dense() - dense).max() < 1e-12
    with pytest.raises(ValueError, match="memory guard"):
        qf.pauli_sum_to_coo(qf.tfim_terms(qf.build_lattice("chain", [27], [False]), 1.0))
    empty = qf.PauliSum(3)
    assert qf.pauli_sum_to_coo(empty).nnz() == 0


def test_randomized_stress_regressions(ctx):
    """Cases found by tools/stress_parity.py: stress_case6 (c128 adjoint kernel whose
    static tables pushed static + dynamic shared memory past the 48 KB default)
    and stress_case138 (deep su4-rich circuit, the c64 worst case: float32
    arithmetic itself, the generic kernels agree)."""
    import os
    here = os.path.join(os.path.dirname(__file__), "cases")
    for name, prec in [("stress_case6.npz", "c128"), ("stress_case6.npz", "c64"),
                       ("stress_case138.npz", "c128"), ("stress_case138.npz", "c64")]:
        tol = TOL[prec]
        d = np.load(os.path.join(here, name), allow_pickle=True)
        n, P = int(d["n"]), int(d["P"])
        ops = [tuple(o) for o in d["ops"]]
        mats = d["mats"] if d["mats"].size else None
        h = po.Hamil(n, d["codes"], d["wr"] + 1j * d["wi"])
        E_ref, G_ref = po.energy_grad_batch(po.Ansatz(n, ops, P, mats), d["th"], h, mode="adjoint")
        obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
        E, G = engine.energy_grad_batch(ctx, engine.Program(ctx, n, ops, P, prec, mats), obs, d["th"])
        # normwise relative error against ||H||_1 = sum |w_k| (>= ||H|| >= |E|, and
        # |dE/dtheta_j| <= 2 |coef_j| ||H||): these random Hamiltonians can vanish on
        # the state (E, G ~ 1e-17), where an error relative to |E| is undefined
        scale = np.abs(h.wr + 1j * h.wi).sum() * max(1.0, max(abs(o[4]) for o in ops))
        err = max(np.abs(E - E_ref).max(), np.abs(G - G_ref).max()) / scale
        assert err <= tol, (name, prec, err)
