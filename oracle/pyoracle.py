"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/liboracle.so, the CPU
restatement of the reference hot path (see qforge_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product (paper_2602_14167_b200)
never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liboracle.so")

GATES = ["h", "x", "y", "z", "s", "rx", "ry", "rz", "rzz", "cx", "cz", "su4", "csum",
         "subspace_ry", "subspace_rz", "unitary"]
GID = {g: i for i, g in enumerate(GATES)}


class QoOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("slot", ctypes.c_int32), ("coef", ctypes.c_double), ("offset", ctypes.c_double),
                ("mat", ctypes.c_int32), ("pad", ctypes.c_int32)]


class QoRng(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("stream", ctypes.c_uint64), ("counter", ctypes.c_uint64),
                ("have_spare", ctypes.c_int32), ("pad", ctypes.c_int32), ("spare", ctypes.c_double)]


class QoAnsatz(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("n_params", ctypes.c_int), ("n_ops", ctypes.c_int),
                ("ops", ctypes.POINTER(QoOp)), ("mats", ctypes.c_void_p), ("init", ctypes.c_void_p),
                ("guard_log2", ctypes.c_int)]


class QoHamil(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("n_terms", ctypes.c_int), ("w_re", ctypes.POINTER(ctypes.c_double)),
                ("w_im", ctypes.POINTER(ctypes.c_double)), ("codes", ctypes.POINTER(ctypes.c_int8))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB)
        D = ctypes.POINTER(ctypes.c_double)
        L.qo_last_error.restype = ctypes.c_char_p
        L.qo_rng_next_u64.restype = ctypes.c_uint64
        L.qo_rng_uniform.restype = ctypes.c_double
        L.qo_rng_uniform_below.restype = ctypes.c_uint64
        L.qo_rng_uniform_below.argtypes = [ctypes.POINTER(QoRng), ctypes.c_uint64]
        L.qo_rng_normal.restype = ctypes.c_double
        L.qo_rng_init.argtypes = [ctypes.POINTER(QoRng), ctypes.c_uint64, ctypes.c_uint64]
        L.qo_rng_split_child.argtypes = [ctypes.POINTER(QoRng), ctypes.c_uint64, ctypes.POINTER(QoRng)]
        L.qo_energy.argtypes = [ctypes.POINTER(QoAnsatz), D, ctypes.POINTER(QoHamil), D]
        L.qo_gradient.argtypes = [ctypes.POINTER(QoAnsatz), D, ctypes.POINTER(QoHamil), ctypes.c_int,
                                  ctypes.c_double, ctypes.c_int, D]
        L.qo_energy_grad_batch.argtypes = [ctypes.POINTER(QoAnsatz), ctypes.c_int, D, ctypes.POINTER(QoHamil),
                                           ctypes.c_int, ctypes.c_int, D, D]
        L.qo_vqe_run.argtypes = [ctypes.POINTER(QoAnsatz), ctypes.c_int, D, ctypes.POINTER(QoHamil),
                                 ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, D, D, D,
                                 ctypes.POINTER(ctypes.c_int)]
        L.qo_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(QoOp), ctypes.c_void_p, D,
                             ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.qo_expectation_pauli.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, D, D,
                                           ctypes.POINTER(ctypes.c_int8), ctypes.c_void_p]
        L.qo_tfim_terms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, D, D,
                                    ctypes.POINTER(ctypes.c_int8)]
        L.qo_heisenberg_terms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, D, D, ctypes.POINTER(ctypes.c_int8)]
        L.qo_random_pauli_sum.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(QoRng), ctypes.c_int,
                                          D, D, ctypes.POINTER(ctypes.c_int8)]
        L.qo_chain_edges.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc):
    if rc != 0:
        raise ValueError(lib().qo_last_error().decode())


class Rng:
    def __init__(self, seed=0, stream=0):
        self.s = QoRng()
        lib().qo_rng_init(ctypes.byref(self.s), seed, stream)

    def next_u64(self):
        return lib().qo_rng_next_u64(ctypes.byref(self.s))

    def uniform(self):
        return lib().qo_rng_uniform(ctypes.byref(self.s))

    def uniform_below(self, b):
        return lib().qo_rng_uniform_below(ctypes.byref(self.s), b)

    def normal(self):
        return lib().qo_rng_normal(ctypes.byref(self.s))

    def split(self, n):
        out = []
        for i in range(n):
            r = Rng.__new__(Rng)
            r.s = QoRng()
            lib().qo_rng_split_child(ctypes.byref(self.s), i, ctypes.byref(r.s))
            out.append(r)
        return out


# ------------------------------------------------------------------ templates
def tca_template(n, layers):
    """tfim_chain_ansatz, variational.cpp:18-36, as an explicit slot template."""
    ops = [(GID["h"], q, -1, -1, 1.0, 0.0, -1) for q in range(n)]
    k = 0
    for _ in range(layers):
        for i in range(n):
            ops.append((GID["rx"], i, -1, k, 1.0, 0.0, -1)); k += 1
        for i in range(n - 1):
            ops.append((GID["rzz"], i, i + 1, k, 1.0, 0.0, -1)); k += 1
    return n, ops, k


def hea_template(n, layers):
    """SURVEY.md 8 HEA: ry all, rz all, cx ladder, per layer."""
    ops, k = [], 0
    for _ in range(layers):
        for q in range(n):
            ops.append((GID["ry"], q, -1, k, 1.0, 0.0, -1)); k += 1
        for q in range(n):
            ops.append((GID["rz"], q, -1, k, 1.0, 0.0, -1)); k += 1
        for q in range(n - 1):
            ops.append((GID["cx"], q, q + 1, -1, 1.0, 0.0, -1))
    return n, ops, k


class Ansatz:
    def __init__(self, n, ops, n_params, mats=None, init=None, guard_log2=40):
        self.n, self.n_params = n, n_params
        self._ops = (QoOp * max(1, len(ops)))()
        for i, o in enumerate(ops):
            self._ops[i] = QoOp(int(o[0]), int(o[1]), int(o[2]), int(o[3]), float(o[4]), float(o[5]), int(o[6]), 0)
        self._mats = None if mats is None else np.ascontiguousarray(np.asarray(mats, np.complex128).reshape(-1, 16))
        self._init = None if init is None else np.ascontiguousarray(np.asarray(init, np.complex128))
        self.s = QoAnsatz(n, n_params, len(ops), self._ops,
                          self._mats.ctypes.data if self._mats is not None else None,
                          self._init.ctypes.data if self._init is not None else None, guard_log2)


class Hamil:
    def __init__(self, n, codes, w):
        self.n = n
        self.codes = np.ascontiguousarray(np.asarray(codes, np.int8).reshape(-1, n))
        w = np.asarray(w, np.complex128).reshape(-1)
        self.wr = np.ascontiguousarray(w.real)
        self.wi = np.ascontiguousarray(w.imag)
        self.s = QoHamil(n, len(w), _d(self.wr), _d(self.wi),
                         self.codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))


def tfim(n, g, pbc=False):
    T = 3 * n + 2
    wr, wi = np.zeros(T), np.zeros(T)
    codes = np.zeros((T, n), np.int8)
    t = lib().qo_tfim_terms(n, int(pbc), g, _d(wr), _d(wi), codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
    _check(0 if t >= 0 else -1)
    return Hamil(n, codes[:t], wr[:t] + 1j * wi[:t])


def heisenberg(n, jx, jy, jz, pbc=False):
    T = 3 * (n + 1)
    wr, wi = np.zeros(T), np.zeros(T)
    codes = np.zeros((T, n), np.int8)
    t = lib().qo_heisenberg_terms(n, int(pbc), jx, jy, jz, _d(wr), _d(wi),
                                  codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
    _check(0 if t >= 0 else -1)
    return Hamil(n, codes[:t], wr[:t] + 1j * wi[:t])


def random_sum(n, terms, rng: Rng, real_weights=True):
    wr, wi = np.zeros(terms), np.zeros(terms)
    codes = np.zeros((terms, n), np.int8)
    lib().qo_random_pauli_sum(n, terms, ctypes.byref(rng.s), int(real_weights), _d(wr), _d(wi),
                              codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
    return Hamil(n, codes, wr + 1j * wi)


# ------------------------------------------------------------------ engine
def run(n, ops, theta=None, mats=None, init=None, guard_log2=40):
    a = Ansatz(n, ops, 0 if theta is None else len(theta), mats, init)
    th = np.ascontiguousarray(np.zeros(1) if theta is None or len(theta) == 0 else np.asarray(theta, np.float64))
    out = np.zeros(1 << n, np.complex128)
    _check(lib().qo_run(n, len(ops), a._ops, a.s.mats, _d(th), a.s.init, guard_log2, out.ctypes.data))
    return out


def expectation(n, psi, h: Hamil):
    psi = np.ascontiguousarray(psi, np.complex128)
    out = np.zeros(1, np.complex128)
    _check(lib().qo_expectation_pauli(n, psi.ctypes.data, len(h.wr), _d(h.wr), _d(h.wi),
                                      h.codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), out.ctypes.data))
    return complex(out[0])


MODES = {"parameter_shift": 0, "finite_diff": 1, "adjoint": 2}


def pauli_sum_to_coo(h: Hamil):
    L = lib()
    L.qo_pauli_sum_to_coo.restype = ctypes.c_longlong
    L.qo_pauli_sum_to_coo.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int8),
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
    c8 = h.codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))
    nnz = L.qo_pauli_sum_to_coo(h.n, len(h.wr), _d(h.wr), _d(h.wi), c8, None, None, None, 0)
    rows = np.zeros(nnz, np.int64)
    cols = np.zeros(nnz, np.int64)
    vals = np.zeros(nnz, np.complex128)
    L.qo_pauli_sum_to_coo(h.n, len(h.wr), _d(h.wr), _d(h.wi), c8, rows.ctypes.data, cols.ctypes.data,
                          vals.ctypes.data, nnz)
    return rows, cols, vals


def energy(a: Ansatz, theta, h: Hamil):
    th = np.ascontiguousarray(np.asarray(theta, np.float64).reshape(-1)) if a.n_params else np.zeros(1)
    e = np.zeros(1)
    _check(lib().qo_energy(ctypes.byref(a.s), _d(th), ctypes.byref(h.s), _d(e)))
    return float(e[0])


def gradient(a: Ansatz, theta, h: Hamil, mode="parameter_shift", fd_step=1e-5, workers=1):
    th = np.ascontiguousarray(np.asarray(theta, np.float64).reshape(-1))
    g = np.zeros(max(1, a.n_params))
    _check(lib().qo_gradient(ctypes.byref(a.s), _d(th), ctypes.byref(h.s), MODES[mode], fd_step, workers, _d(g)))
    return g[: a.n_params]


def energy_grad_batch(a: Ansatz, thetas, h: Hamil, mode="parameter_shift", workers=1, grads=True):
    th = np.ascontiguousarray(np.asarray(thetas, np.float64).reshape(-1, a.n_params))
    B = th.shape[0]
    E = np.zeros(B)
    G = np.zeros((B, a.n_params)) if grads else None
    _check(lib().qo_energy_grad_batch(ctypes.byref(a.s), B, _d(th), ctypes.byref(h.s), MODES[mode], workers,
                                      _d(E), _d(G) if grads else None))
    return E, G


def vqe_run(a: Ansatz, theta0, h: Hamil, steps, lr, mode="parameter_shift", workers=1):
    th = np.ascontiguousarray(np.asarray(theta0, np.float64).reshape(-1, a.n_params))
    B = th.shape[0]
    traces = np.zeros((B, steps + 1))
    fin = np.zeros((B, a.n_params))
    be = np.zeros(1)
    bi = ctypes.c_int()
    _check(lib().qo_vqe_run(ctypes.byref(a.s), B, _d(th), ctypes.byref(h.s), steps, lr, MODES[mode], workers,
                            _d(traces), _d(fin), _d(be), ctypes.byref(bi)))
    return traces, fin, float(be[0]), bi.value


# ------------------------------------------------------------------ trajectories
# TEST INFRASTRUCTURE ONLY: numpy restatement of the MIPT-Haar experiment
# (reference proj/src/experiments.cpp:210-250) for parity tests at small n.
def haar_su4(rng: Rng) -> np.ndarray:
    """circuit.cpp:472-489: QR of a complex Gaussian 4x4, R-diagonal phases moved
    into Q, Q *= det(Q)^(-1/4).  cplx(rng.normal(), rng.normal()) draws the
    imaginary part first (gcc argument order, pinned with the RNG fixtures)."""
    g = np.zeros((4, 4), complex)
    for r in range(4):
        for c in range(4):
            im = rng.normal()
            re = rng.normal()
            g[r, c] = re + 1j * im
    q, rr = np.linalg.qr(g)
    d = np.diag(rr)
    ph = np.where(np.abs(d) > 0, d / np.where(np.abs(d) > 0, np.abs(d), 1), 1.0)
    q = q * ph[None, :]
    q = q * np.exp(-1j * np.angle(np.linalg.det(q)) / 4.0)
    return q


def apply_2q(psi: np.ndarray, n: int, u: np.ndarray, a: int, b: int) -> np.ndarray:
    """apply_local_unitary(psi, u, {a, b}) with wire a the most significant local bit."""
    t = psi.reshape([2] * n)
    t = np.moveaxis(t, [a, b], [0, 1]).reshape(4, -1)
    t = (u @ t).reshape([2, 2] + [2] * (n - 2))
    return np.moveaxis(t, [0, 1], [a, b]).reshape(-1)


def measure_collapse(psi: np.ndarray, n: int, wire: int, u: float) -> np.ndarray:
    """circuit.cpp:391-429 for d = 2 with the uniform already drawn."""
    t = psi.reshape([2] * n)
    sel = [slice(None)] * n
    probs = []
    for o in range(2):
        sel[wire] = o
        probs.append(float(np.sum(np.abs(t[tuple(sel)]) ** 2)))
    outcome, acc = 1, 0.0
    for o in range(2):
        acc += probs[o]
        if u < acc:
            outcome = o
            break
    out = np.zeros_like(t)
    sel[wire] = outcome
    out[tuple(sel)] = t[tuple(sel)] / np.sqrt(probs[outcome])
    return out.reshape(-1)


def subsystem_entropy_half(psi: np.ndarray, n: int) -> float:
    """circuit.cpp:431-470 with keep = {0 .. n/2 - 1} (the leading wires)."""
    k = n // 2
    s = np.linalg.svd(psi.reshape(1 << k, 1 << (n - k)), compute_uv=False)
    ent = 0.0
    for v in s:
        p = min(max(v * v, 0.0), 1.0)
        if p > 1e-15:
            ent -= p * np.log2(p)
    return max(ent, 0.0)


def mipt_haar(n: int, depth: int, p: float, trajectories: int, seed: int):
    """exp_mipt_haar (experiments.cpp:210-250): per-trajectory half-chain entropies."""
    streams = Rng(seed).split(trajectories)
    ents = []
    for tr in range(trajectories):
        rs = streams[tr]
        psi = np.zeros(1 << n, complex)
        psi[0] = 1.0
        for layer in range(depth):
            for i in range(layer % 2, n - 1, 2):
                psi = apply_2q(psi, n, haar_su4(rs), i, i + 1)
            for q in range(n):
                if rs.uniform() < p:
                    psi = measure_collapse(psi, n, q, rs.uniform())
        ents.append(subsystem_entropy_half(psi, n))
    return np.array(ents)


# classical shadows (reference proj/src/shadows.cpp:24-85, experiments.cpp:252-274)
_S = np.sqrt(0.5)
BASIS_ROTATION = {1: np.array([[_S, _S], [_S, -_S]], complex), 2: np.array([[_S, -1j * _S], [_S, 1j * _S]]),
                  3: np.eye(2, dtype=complex)}


def shadow_snapshots(psi: np.ndarray, n: int, bases, us) -> np.ndarray:
    """shadow_snapshots with the per-snapshot uniforms already drawn: rotate, then
    the first index whose running sum of |a_i|^2 exceeds u (last index if none)."""
    out = np.zeros((len(bases), n), np.int8)
    for r, (row, u) in enumerate(zip(bases, us)):
        t = psi.reshape([2] * n)
        for q, code in enumerate(row):
            if code != 3:
                t = np.moveaxis(np.tensordot(BASIS_ROTATION[int(code)], t, axes=([1], [q])), 0, q)
        acc = np.cumsum(np.abs(t.reshape(-1)) ** 2)
        idx = int(np.searchsorted(acc, u, side="right"))
        idx = min(idx, (1 << n) - 1)
        out[r] = [(idx >> (n - 1 - q)) & 1 for q in range(n)]
    return out


def shadow_gen_inputs(n: int, m: int, depth: int, seed: int):
    """exp_shadow_gen randomness: ry angles (streams[0]), bases (streams[1]),
    per-snapshot uniforms (streams[2].split(m)); returns (ops, bases, us)."""
    streams = Rng(seed).split(3)
    ops = []
    for _ in range(depth):
        for q in range(n):
            ops.append((GID["ry"], q, -1, -1, 1.0, 2.0 * 3.14159265358979323846 * streams[0].uniform(), -1))
        for q in range(n - 1):
            ops.append((GID["cx"], q, q + 1, -1, 1.0, 0.0, -1))
    bases = [[1 + streams[1].uniform_below(3) for _ in range(n)] for _ in range(m)]
    us = [s.uniform() for s in streams[2].split(m)]
    return ops, np.array(bases, np.int8), np.array(us)


# noise trajectories (reference proj/src/noise.cpp:162-197)
def _gate_matrix_np(kind, offset):
    """circuit.cpp:202-302 for the constant gates used by the noise tests."""
    g = GATES[kind]
    c, s = np.cos(offset / 2), np.sin(offset / 2)
    h = np.sqrt(0.5)
    table = {
        "h": np.array([[h, h], [h, -h]], complex), "x": np.array([[0, 1], [1, 0]], complex),
        "y": np.array([[0, -1j], [1j, 0]]), "z": np.diag([1.0 + 0j, -1]), "s": np.diag([1.0 + 0j, 1j]),
        "rx": np.array([[c, -1j * s], [-1j * s, c]]), "ry": np.array([[c, -s], [s, c]], complex),
        "rz": np.diag([np.exp(-0.5j * offset), np.exp(0.5j * offset)]),
        "rzz": np.diag([np.exp(-0.5j * offset), np.exp(0.5j * offset), np.exp(0.5j * offset), np.exp(-0.5j * offset)]),
        "cx": np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], complex),
        "cz": np.diag([1.0 + 0j, 1, 1, -1]),
    }
    return table[g]


def _apply_np(psi, n, m, wires):
    if len(wires) == 1:
        t = np.moveaxis(np.tensordot(m, psi.reshape([2] * n), axes=([1], [wires[0]])), 0, wires[0])
        return t.reshape(-1)
    return apply_2q(psi, n, m, wires[0], wires[1])


def mc_trajectory(n, ops, op_channels, channels, u_row):
    """One trajectory with its uniforms already drawn: (state, log_prob)."""
    psi = np.zeros(1 << n, complex)
    psi[0] = 1.0
    logp, app = 0.0, 0
    for j, op in enumerate(ops):
        kind, q0, q1 = op[0], op[1], op[2]
        wires = [q0] if q1 < 0 else [q0, q1]
        psi = _apply_np(psi, n, _gate_matrix_np(kind, op[5]), wires)
        for ch in op_channels[j]:
            branches = [_apply_np(psi, n, np.asarray(k, complex), wires) for k in channels[ch]]
            probs = [float(np.sum(np.abs(b) ** 2)) for b in branches]
            acc = sum(probs)
            uu = u_row[app] * acc
            app += 1
            pick, run = len(probs) - 1, 0.0
            for i, p in enumerate(probs):
                run += p
                if uu < run:
                    pick = i
                    break
            psi = branches[pick] / np.sqrt(probs[pick])
            logp += np.log(probs[pick] / acc) + np.log(acc)
    return psi, logp


def density_matrix_expect_z0(n, ops, op_channels, channels):
    """Exact <Z_0> of the channel-averaged state (density_matrix_run, noise.cpp:199-240)."""
    rho = np.zeros((1 << n, 1 << n), complex)
    rho[0, 0] = 1.0
    for j, op in enumerate(ops):
        wires = [op[1]] if op[2] < 0 else [op[1], op[2]]

        def conj(r, m):
            cols = np.stack([_apply_np(r[:, c], n, m, wires) for c in range(1 << n)], axis=1)
            rows = np.stack([_apply_np(cols[i, :].conj(), n, m, wires).conj() for i in range(1 << n)], axis=0)
            return rows
        rho = conj(rho, _gate_matrix_np(op[0], op[5]))
        for ch in op_channels[j]:
            rho = sum(conj(rho, np.asarray(k, complex)) for k in channels[ch])
    z0 = np.array([1.0 if ((i >> (n - 1)) & 1) == 0 else -1.0 for i in range(1 << n)])
    return float(np.real(np.sum(np.diag(rho) * z0)))
