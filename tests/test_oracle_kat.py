"""Pins the CPU oracle (oracle/, the C restatement of the reference hot path)
against every known answer the reference's own tests hold for this path
(SURVEY.md 8c).  Test names cite the reference test they port
(paths relative to /root/reference/proj).  CPU only."""
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po

H = po.GID


# ---------------------------------------------------------------- dense helpers (tests/helpers.hpp)
PAULI = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1, -1])]


def pauli_sum_dense(h):
    n = h.n
    out = np.zeros((1 << n, 1 << n), complex)
    for t in range(len(h.wr)):
        m = np.eye(1)
        for c in h.codes[t]:
            m = np.kron(m, PAULI[c])
        out += complex(h.wr[t], h.wi[t]) * m
    return out


def lift(op, wires, n):
    """helpers.hpp:66-86: dense n-qubit lift, wires[0] most significant."""
    dim = 1 << n
    w = len(wires)
    out = np.zeros((dim, dim), complex)
    for row in range(dim):
        lrow = 0
        for k in range(w):
            lrow = (lrow << 1) | ((row >> (n - 1 - wires[k])) & 1)
        for lcol in range(1 << w):
            if op[lrow, lcol] == 0:
                continue
            col = row
            for k in range(w):
                bit = (lcol >> (w - 1 - k)) & 1
                pos = n - 1 - wires[k]
                col = (col & ~(1 << pos)) | (bit << pos)
            out[col, row] += op[lcol, lrow]
    return out


def gate_dense(kind, theta):
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    isq = 1 / math.sqrt(2)
    return {H["h"]: np.array([[isq, isq], [isq, -isq]]), H["s"]: np.diag([1, 1j]),
            H["rx"]: np.array([[c, -1j * s], [-1j * s, c]]), H["ry"]: np.array([[c, -s], [s, c]]),
            H["rz"]: np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta)]),
            H["rzz"]: np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta), np.exp(0.5j * theta),
                               np.exp(-0.5j * theta)]),
            H["cx"]: np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]])}[kind]


def random_circuit(n, depth, rng):
    """test_circuit.cpp:15-33 (same RNG draw order)."""
    ops = []
    for layer in range(depth):
        for q in range(n):
            r = rng.uniform_below(5)
            if r == 0:
                ops.append((H["h"], q, -1, -1, 1.0, 0.0, -1))
            elif r in (1, 2, 3):
                ops.append(({1: H["rx"], 2: H["ry"], 3: H["rz"]}[r], q, -1, -1, 1.0, rng.uniform() * 6.28, -1))
            else:
                ops.append((H["s"], q, -1, -1, 1.0, 0.0, -1))
        for q in range(layer % 2, n - 1, 2):
            if rng.uniform() < 0.5:
                ops.append((H["cx"], q, q + 1, -1, 1.0, 0.0, -1))
            else:
                ops.append((H["rzz"], q, q + 1, -1, 1.0, rng.uniform() * 6.28, -1))
    return ops


# ---------------------------------------------------------------- RNG (rng.hpp)
def test_rng_matches_reference_header_golden():
    """tests/golden/rng_known_answers.txt was produced by the reference's own
    rng.hpp (oracle/_ref/ref_rng_driver)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "rng_known_answers.txt")
    lines = [l.split() for l in open(path)]
    r3 = po.Rng(3)
    r7 = po.Rng(7)
    kids = po.Rng(0).split(8)
    r11 = po.Rng(11)
    r13 = po.Rng(13)
    rps_codes, rps_w = [], []
    for l in lines:
        tag = l[0]
        if tag == "normal3":
            assert r3.normal() == float(l[1])
        elif tag == "u64_7":
            assert r7.next_u64() == int(l[1])
        elif tag == "split0":
            assert kids[int(l[1])].normal() == float(l[2])
        elif tag == "below5":
            assert r11.uniform_below(5) == int(l[1])
        elif tag == "uniform":
            assert r11.uniform() == float(l[1])
        elif tag == "rps_codes":
            rps_codes.append([int(x) for x in l[1:]])
        elif tag == "rps_w":
            rps_w.append(complex(float(l[1]), float(l[2])))
    h = po.random_sum(5, 4, r13, real_weights=False)
    assert h.codes.tolist() == rps_codes
    assert [complex(a, b) for a, b in zip(h.wr, h.wi)] == rps_w


def test_rng_survey_values():
    """SURVEY.md 8c 'Measured this session' table."""
    r = po.Rng(3)
    assert [r.normal() for _ in range(4)] == [-1.1682818837958107, -0.82785524824902013,
                                              -1.6428854116943845, 0.48790908971558378]
    assert po.Rng(0).split(8)[1].normal() == 1.6213865529772808
    assert po.Rng(7).next_u64() == 9065798422547270908


# ---------------------------------------------------------------- test_variational.cpp
def test_chain_ansatz_layout_and_zero_energy():
    """test_variational.cpp:33-53: TCA(4,3) at theta=0 on TFIM(4,1) = -4; counts h=4 rx=12 rzz=9."""
    n, ops, P = po.tca_template(4, 3)
    assert P == 3 * (2 * 4 - 1)
    kinds = [o[0] for o in ops]
    assert kinds.count(H["h"]) == 4 and kinds.count(H["rx"]) == 12 and kinds.count(H["rzz"]) == 9
    e = po.energy(po.Ansatz(n, ops, P), np.zeros(P), po.tfim(4, 1.0))
    assert e == pytest.approx(-4.0, rel=1e-10)


def test_identity_ansatz_on_zero_state():
    """test_variational.cpp:56-63: empty 2-site circuit picks the -zz element: -1."""
    assert po.energy(po.Ansatz(2, [], 0), np.zeros(0), po.tfim(2, 1.0)) == pytest.approx(-1.0, rel=1e-10)


def test_injected_ground_state():
    """test_variational.cpp:64-77: initial_state = exact ground -> -sqrt(5)."""
    h = po.tfim(2, 1.0)
    w, v = np.linalg.eigh(pauli_sum_dense(h))
    e = po.energy(po.Ansatz(2, [], 0, init=v[:, 0]), np.zeros(0), h)
    assert e == pytest.approx(-math.sqrt(5.0), rel=1e-10)


def test_pure_pipeline_and_dense_agreement():
    """test_variational.cpp:78-89: repeated energy bit-identical; PauliSum vs matrix 1e-12."""
    n, ops, P = po.tca_template(5, 2)
    r = po.Rng(3)
    th = np.array([r.normal() for _ in range(P)])
    h = po.tfim(5, 1.3)
    a = po.Ansatz(n, ops, P)
    e1, e2 = po.energy(a, th, h), po.energy(a, th, h)
    assert e1 == e2
    psi = po.run(n, ops, th)
    e3 = np.vdot(psi, pauli_sum_dense(h) @ psi).real
    assert e1 == pytest.approx(e3, rel=1e-12)


def test_variational_bound():
    """test_variational.cpp:90-100."""
    h = po.tfim(5, 1.0)
    ground = np.linalg.eigvalsh(pauli_sum_dense(h)).min()
    n, ops, P = po.tca_template(5, 2)
    a = po.Ansatz(n, ops, P)
    r = po.Rng(8)
    for _ in range(10):
        th = np.array([r.normal() for _ in range(P)])
        assert po.energy(a, th, h) >= ground - 1e-9


def _single_rx():
    return po.Ansatz(1, [(H["rx"], 0, -1, 0, 1.0, 0.0, -1)], 1)


def _z1():
    return po.Hamil(1, [[3]], [1.0])


def test_single_rotation_derivative():
    """test_variational.cpp:104-116: d<Z>/dtheta = -sin(pi/3); FD within 1e-6."""
    g = po.gradient(_single_rx(), [math.pi / 3], _z1(), "parameter_shift")
    assert g[0] == pytest.approx(-math.sin(math.pi / 3), rel=1e-10)
    gf = po.gradient(_single_rx(), [math.pi / 3], _z1(), "finite_diff")
    assert gf[0] == pytest.approx(g[0], rel=1e-6)
    ga = po.gradient(_single_rx(), [math.pi / 3], _z1(), "adjoint")
    assert ga[0] == pytest.approx(g[0], rel=1e-12)


def test_stationary_at_minimum():
    """test_variational.cpp:117-126."""
    assert abs(po.gradient(_single_rx(), [math.pi], _z1(), "parameter_shift")[0]) < 1e-8


def test_shift_vs_fd_and_worker_invariance():
    """test_variational.cpp:127-138: TCA(6,2), TFIM g=0.8, seed 5."""
    n, ops, P = po.tca_template(6, 2)
    a = po.Ansatz(n, ops, P)
    h = po.tfim(6, 0.8)
    r = po.Rng(5)
    th = np.array([r.normal() for _ in range(P)])
    gs = po.gradient(a, th, h, "parameter_shift")
    gf = po.gradient(a, th, h, "finite_diff")
    assert np.abs(gs - gf).max() < 1e-6
    g4 = po.gradient(a, th, h, "parameter_shift", workers=4)
    assert np.array_equal(gs, g4)


def test_shift_rule_refuses_compound_generators():
    """test_variational.cpp:139-153: a parameter feeding su4 is not shift-eligible."""
    m = np.eye(4, dtype=complex)
    a = po.Ansatz(2, [(H["su4"], 0, 1, 0, 1.0, 0.0, 0), (H["rx"], 0, -1, -1, 1.0, 0.0, -1)], 1, mats=[m])
    with pytest.raises(ValueError):
        po.gradient(a, [0.0], po.tfim(2, 1.0), "parameter_shift")
    po.gradient(a, [0.0], po.tfim(2, 1.0), "finite_diff")


def test_adjoint_equals_parameter_shift():
    """New math (the reference has no adjoint): exact agreement with the shift rule."""
    for tmpl, hm in ((po.hea_template(6, 2), po.heisenberg(6, 1.0, 1.0, 0.5)),
                     (po.tca_template(7, 2), po.tfim(7, 0.9)),
                     (po.hea_template(5, 2), po.random_sum(5, 12, po.Rng(4), False))):
        n, ops, P = tmpl
        a = po.Ansatz(n, ops, P)
        r = po.Rng(21)
        th = np.array([r.normal() for _ in range(P)])
        gs = po.gradient(a, th, hm, "parameter_shift")
        ga = po.gradient(a, th, hm, "adjoint")
        assert np.abs(gs - ga).max() <= 1e-12 * max(1.0, np.abs(gs).max())


def test_adam_first_step_and_fixed_point():
    """test_variational.cpp:156-190."""
    import ctypes
    L = po.lib()
    L.qo_adam_step.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.POINTER(ctypes.c_int)] + \
        [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.c_int] + [ctypes.c_double] * 4
    d = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    m, v, th = np.zeros(2), np.zeros(2), np.zeros(2)
    t = ctypes.c_int(0)
    L.qo_adam_step(d(m), d(v), ctypes.byref(t), d(th), d(np.array([0.3, -7.0])), 2, 0.05, 0.9, 0.999, 1e-8)
    assert th[0] == pytest.approx(-0.05, rel=1e-6) and th[1] == pytest.approx(0.05, rel=1e-6)
    m, v, th = np.zeros(3), np.zeros(3), np.array([1.0, -2.0, 0.5])
    t = ctypes.c_int(0)
    L.qo_adam_step(d(m), d(v), ctypes.byref(t), d(th), d(np.zeros(3)), 3, 0.1, 0.9, 0.999, 1e-8)
    assert np.abs(th - [1.0, -2.0, 0.5]).max() < 1e-12


def test_vqe_two_site_reaches_ground():
    """test_variational.cpp:194-209: n=2, 8 seeds x 300 steps -> -sqrt(5) +- 1e-3."""
    n, ops, P = po.tca_template(2, 2)
    r = po.Rng(7)
    batch = np.array([[0.1 * r.normal() for _ in range(P)] for _ in range(8)])
    tr, fin, best, bi = po.vqe_run(po.Ansatz(n, ops, P), batch, po.tfim(2, 1.0), 300, 0.02)
    assert best == pytest.approx(-math.sqrt(5.0), rel=1e-3)
    assert bi >= 0 and tr[bi, -1] == best


def test_vqe_zero_rate_and_worker_invariance():
    """test_variational.cpp:210-232."""
    n, ops, P = po.tca_template(3, 1)
    a = po.Ansatz(n, ops, P)
    h = po.tfim(3, 1.0)
    t0 = np.full((1, P), 0.3)
    _, _, best, _ = po.vqe_run(a, t0, h, 1, 0.0)
    assert best == pytest.approx(po.energy(a, t0[0], h), rel=1e-12)
    r = po.Rng(9)
    batch = np.array([[r.normal() for _ in range(P)] for _ in range(3)])
    tr1 = po.vqe_run(a, batch, h, 10, 0.02, workers=1)[0]
    tr3 = po.vqe_run(a, batch, h, 10, 0.02, workers=3)[0]
    assert np.array_equal(tr1, tr3)


# ---------------------------------------------------------------- test_circuit.cpp
def test_basic_gates():
    """test_circuit.cpp:37-58: H|0>, Bell ZZ = XX = 1, rx(pi)|0> = -i|1>."""
    psi = po.run(1, [(H["h"], 0, -1, -1, 1, 0, -1)])
    assert np.allclose(psi, [1 / math.sqrt(2)] * 2, atol=1e-12)
    bell = [(H["h"], 0, -1, -1, 1, 0, -1), (H["cx"], 0, 1, -1, 1, 0, -1)]
    psi = po.run(2, bell)
    assert po.expectation(2, psi, po.Hamil(2, [[3, 3]], [1.0])).real == pytest.approx(1.0)
    assert po.expectation(2, psi, po.Hamil(2, [[1, 1]], [1.0])).real == pytest.approx(1.0)
    psi = po.run(1, [(H["rx"], 0, -1, -1, 1, math.pi, -1)])
    assert abs(psi[0]) < 1e-12 and abs(psi[1] - (-1j)) < 1e-12


def test_random_circuits_match_dense_lift():
    """test_circuit.cpp:59-72: 10 random circuits (n 3..5) vs Kronecker lift, 1e-10."""
    rng = po.Rng(31)
    for _ in range(10):
        n = 3 + rng.uniform_below(3)
        ops = random_circuit(n, 4, rng)
        psi = po.run(n, ops)
        ref = np.zeros(1 << n, complex)
        ref[0] = 1
        for o in ops:
            wires = [o[1]] if o[2] < 0 else [o[1], o[2]]
            ref = lift(gate_dense(o[0], o[5]), wires, n) @ ref
        assert np.abs(psi - ref).max() < 1e-10


def test_norm_preserved_and_memory_guard():
    """test_circuit.cpp:73-80."""
    ops = random_circuit(6, 40, po.Rng(77))
    assert abs(np.linalg.norm(po.run(6, ops)) - 1.0) < 1e-10
    with pytest.raises(ValueError, match="memory guard"):
        po.run(30, [], guard_log2=24)


def test_expectation_vs_dense_sandwich():
    """test_circuit.cpp:83-118: Z on |0>, Ising ground -sqrt(5), 20 random complex sums."""
    assert po.expectation(1, np.array([1, 0], complex), po.Hamil(1, [[3]], [1.0])).real == pytest.approx(1.0)
    h = po.Hamil(2, [[3, 3], [1, 0], [0, 1]], [-1.0, -1.0, -1.0])
    w, v = np.linalg.eigh(pauli_sum_dense(h))
    assert po.expectation(2, v[:, 0].copy(), h).real == pytest.approx(-math.sqrt(5.0))
    rng = po.Rng(13)
    for _ in range(20):
        n = 1 + rng.uniform_below(8)
        hh = po.random_sum(n, 4, rng, real_weights=False)
        psi = np.array([complex(rng.normal(), rng.normal()) for _ in range(1 << n)])
        psi /= np.linalg.norm(psi)
        want = np.vdot(psi, pauli_sum_dense(hh) @ psi)
        assert abs(po.expectation(n, psi, hh) - want) < 1e-10


def test_rzz_lowering_equivalent():
    """test_circuit.cpp:302-314: rzz == cx rz cx up to a global phase."""
    direct = po.run(2, [(H["h"], 0, -1, -1, 1, 0, -1), (H["h"], 1, -1, -1, 1, 0, -1),
                        (H["rzz"], 0, 1, -1, 1, 0.9, -1)])
    lowered = po.run(2, [(H["h"], 0, -1, -1, 1, 0, -1), (H["h"], 1, -1, -1, 1, 0, -1),
                         (H["cx"], 0, 1, -1, 1, 0, -1), (H["rz"], 1, -1, -1, 1, 0.9, -1),
                         (H["cx"], 0, 1, -1, 1, 0, -1)])
    ratio = lowered[0] / direct[0]
    assert np.abs(direct * ratio - lowered).max() < 1e-12


# ---------------------------------------------------------------- test_hamiltonian.cpp
def test_model_builders():
    """test_hamiltonian.cpp:115-148."""
    h = po.tfim(3, 0.7)
    assert len(h.wr) == 5
    assert sorted(h.wr.tolist()) == sorted([-1.0, -1.0, -0.7, -0.7, -0.7])
    assert len(po.heisenberg(2, 1, 1, 1).wr) == 3
    h10 = po.tfim(10, 1.0)
    assert len(h10.wr) == 19
    assert po.heisenberg(26, 1.0, 1.0, 0.5).codes.shape == (75, 26)
    # periodic chain: (0, n-1) joins the first shell (lattice.cpp:29-48, 89-122)
    assert len(po.tfim(5, 1.0, pbc=True).wr) == 10


def test_oracle_coo_matches_dense():
    """test_hamiltonian.cpp:18-50: COO lowering equals the dense Kronecker sum."""
    for ho in (po.tfim(5, 0.7), po.heisenberg(4, 1.0, 1.0, 1.0), po.random_sum(5, 12, po.Rng(8), False)):
        r, c, v = po.pauli_sum_to_coo(ho)
        m = np.zeros((1 << ho.n, 1 << ho.n), complex)
        np.add.at(m, (r, c), v)
        assert np.abs(m - pauli_sum_dense(ho)).max() < 1e-12
        assert np.all(np.diff(r) >= 0)
        same = r[1:] == r[:-1]
        assert np.all(c[1:][same] > c[:-1][same])
        assert np.all(v != 0)


def test_trajectory_restatements_properties():
    """Oracle restatements of the trajectory callers (oracle/pyoracle.py): haar_su4
    is unitary with det 1 (circuit.cpp:472-489); MIPT with p = 1 or depth 0 has
    zero half-chain entropy, a Bell pair has one bit; shadows of |+++> in the X
    basis are all zeros and Z-basis samples of |0..0> are all zeros
    (test_shadows.cpp:101-118)."""
    import numpy as np
    for s in range(5):
        u = po.haar_su4(po.Rng(s))
        assert np.abs(u.conj().T @ u - np.eye(4)).max() < 1e-12
        assert abs(np.linalg.det(u) - 1.0) < 1e-12
    assert np.abs(po.mipt_haar(6, 4, 1.0, 3, 9)).max() < 1e-12
    assert np.abs(po.mipt_haar(6, 0, 0.5, 2, 9)).max() < 1e-12
    bell = np.zeros(4, complex)
    bell[0] = bell[3] = np.sqrt(0.5)
    assert abs(po.subsystem_entropy_half(bell, 2) - 1.0) < 1e-12
    plus = np.full(8, np.sqrt(1 / 8), complex)
    assert not po.shadow_snapshots(plus, 3, [[1, 1, 1]] * 10, np.linspace(0, 0.99, 10)).any()
    zero = np.zeros(8, complex)
    zero[0] = 1
    assert not po.shadow_snapshots(zero, 3, [[3, 3, 3]] * 10, np.linspace(0, 0.99, 10)).any()
