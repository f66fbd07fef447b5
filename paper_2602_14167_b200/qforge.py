"""Python mirror of the reference qforge hot-path API, backed by the B200 engine.

Same names, argument meaning and error behaviour as the reference C++ headers
(paths relative to /root/reference/proj):

  include/qforge/circuit.hpp      Gate, GateInstruction, StateVector, Circuit,
                                  apply_local_unitary, gate_matrix, run,
                                  expectation_pauli
  include/qforge/pauli.hpp        PauliTerm, PauliSum, tfim_terms, heisenberg_terms
  include/qforge/lattice.hpp      build_lattice (chain: the only geometry on the path)
  include/qforge/variational.hpp  AnsatzSpec, tfim_chain_ansatz, energy, GradMode,
                                  gradient, AdamState, adam_step, VqeResult, vqe_run

require() failures raise ValueError (std::invalid_argument in the reference).
All state-vector work runs in libqforge_b200.so on the GPU; there is no CPU
path.  Differences, all additive: GradMode.adjoint, energy_gradient_batch, the
`precision` switch (the reference is complex128 only; default here is c128),
and hea_ansatz (the synthetic hardware-efficient ansatz of BASELINE.json).
"""
from __future__ import annotations

import enum
import json
import weakref
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from . import engine as _eng

# ---------------------------------------------------------------- precision
_precision = "c128"


def set_precision(p: str) -> None:
    """'c128' (reference numerics, default) or 'c64' (complex64 fast path)."""
    global _precision
    if p not in ("c64", "c128"):
        raise ValueError("precision must be 'c64' or 'c128'")
    _precision = p


def get_precision() -> str:
    return _precision


def _require(cond: bool, msg: str) -> None:  # common.hpp:24-26
    if not cond:
        raise ValueError(msg)


# ---------------------------------------------------------------- circuits
class Gate(enum.IntEnum):  # circuit.hpp:14-23
    h = 0
    x = 1
    y = 2
    z = 3
    s = 4
    rx = 5
    ry = 6
    rz = 7
    rzz = 8
    cx = 9
    cz = 10
    su4 = 11
    csum = 12
    subspace_ry = 13
    subspace_rz = 14
    unitary = 15


def gate_name(g: Gate) -> str:
    return Gate(g).name


@dataclass
class GateInstruction:  # circuit.hpp:27-32
    name: Gate
    wires: list
    params: list = field(default_factory=list)
    matrix: Optional[np.ndarray] = None


_PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_PY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_PZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
_I2 = np.eye(2, dtype=np.complex128)


def _su4_matrix(theta: Sequence[float]) -> np.ndarray:
    """exp(-i/2 sum_k theta_k P_k), two-qubit Pauli words in lexicographic code
    order without (0,0) (circuit.cpp:254-272)."""
    from scipy.linalg import expm

    single = [_I2, _PX, _PY, _PZ]
    gen = np.zeros((4, 4), dtype=np.complex128)
    k = 0
    for a in range(4):
        for b in range(4):
            if a == 0 and b == 0:
                continue
            gen += theta[k] * np.kron(single[a], single[b])
            k += 1
    return expm(-0.5j * gen)


def gate_matrix(instr: GateInstruction, d: int = 2) -> np.ndarray:
    """Dense matrix of one instruction (circuit.cpp:202-302, qubit gates)."""
    g = Gate(instr.name)
    if g in (Gate.csum, Gate.subspace_ry, Gate.subspace_rz):
        raise ValueError("gate_matrix: qudit gates are not supported on the qubit device path")
    _require(d == 2, "gate_matrix: qubit-only gate in a qudit circuit")
    isq = 1.0 / math.sqrt(2.0)
    if g == Gate.h:
        return np.array([[isq, isq], [isq, -isq]], dtype=np.complex128)
    if g == Gate.x:
        return _PX.copy()
    if g == Gate.y:
        return _PY.copy()
    if g == Gate.z:
        return _PZ.copy()
    if g == Gate.s:
        return np.array([[1, 0], [0, 1j]], dtype=np.complex128)
    if g in (Gate.rx, Gate.ry, Gate.rz, Gate.rzz):
        t = instr.params[0]
        c, s = math.cos(0.5 * t), math.sin(0.5 * t)
        if g == Gate.rx:
            return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
        if g == Gate.ry:
            return np.array([[c, -s], [s, c]], dtype=np.complex128)
        em = complex(math.cos(-0.5 * t), math.sin(-0.5 * t))
        ep = complex(math.cos(0.5 * t), math.sin(0.5 * t))
        if g == Gate.rz:
            return np.diag([em, ep]).astype(np.complex128)
        return np.diag([em, ep, ep, em]).astype(np.complex128)
    if g == Gate.cx:
        m = np.zeros((4, 4), dtype=np.complex128)
        m[0, 0] = m[1, 1] = m[2, 3] = m[3, 2] = 1
        return m
    if g == Gate.cz:
        return np.diag([1, 1, 1, -1]).astype(np.complex128)
    if g == Gate.su4:
        _require(len(instr.params) == 15, "su4: needs 15 parameters")
        return _su4_matrix(instr.params)
    return np.asarray(instr.matrix, dtype=np.complex128)


class StateVector:  # circuit.hpp:36-44
    def __init__(self, n: int = 0, d: int = 2, amps: Optional[np.ndarray] = None):
        self.n, self.d = n, d
        self.amps = amps if amps is not None else np.zeros(0, dtype=np.complex128)

    @staticmethod
    def zero_state(n: int, d: int = 2) -> "StateVector":
        a = np.zeros(d ** n, dtype=np.complex128)
        a[0] = 1.0
        return StateVector(n, d, a)

    def dim(self) -> int:
        return int(self.amps.size)

    def norm(self) -> float:
        return float(np.linalg.norm(self.amps))


class Circuit:  # circuit.hpp:51-83
    def __init__(self, n: int = 0, d: int = 2):
        self.n, self.d = n, d
        self.ops: list[GateInstruction] = []
        self.initial_state: Optional[np.ndarray] = None

    def gate(self, g, wires, params=()) -> "Circuit":  # circuit.cpp:178-186
        wires = [int(w) for w in wires]
        for w in wires:
            _require(0 <= w < self.n, "Circuit: wire out of range")
        for a in range(len(wires)):
            for b in range(a + 1, len(wires)):
                _require(wires[a] != wires[b], "Circuit: duplicate wires")
        params = list(params)
        for p in params:
            _require(_isfinite(p), "Circuit: non-finite parameter")
        self.ops.append(GateInstruction(Gate(g), wires, params))
        return self

    def h(self, w): return self.gate(Gate.h, [w])
    def x(self, w): return self.gate(Gate.x, [w])
    def y(self, w): return self.gate(Gate.y, [w])
    def z(self, w): return self.gate(Gate.z, [w])
    def s(self, w): return self.gate(Gate.s, [w])
    def rx(self, w, t): return self.gate(Gate.rx, [w], [t])
    def ry(self, w, t): return self.gate(Gate.ry, [w], [t])
    def rz(self, w, t): return self.gate(Gate.rz, [w], [t])
    def rzz(self, a, b, t): return self.gate(Gate.rzz, [a, b], [t])
    def cx(self, c, t): return self.gate(Gate.cx, [c, t])
    def cz(self, a, b): return self.gate(Gate.cz, [a, b])

    def su4(self, a, b, theta):  # circuit.cpp:188-191
        _require(len(theta) == 15, "su4: needs 15 parameters")
        return self.gate(Gate.su4, [a, b], theta)

    def unitary(self, wires, u):  # circuit.cpp:193-200
        u = np.asarray(u, dtype=np.complex128)
        _require(np.abs(u.conj().T @ u - np.eye(u.shape[0])).max() < 1e-10,
                 "unitary: matrix is not unitary")
        self.gate(Gate.unitary, wires, [])
        self.ops[-1].matrix = u
        return self

    def to_json(self) -> str:  # circuit.cpp:524-547: {"d","n","ops":[{"name","params","wires"[,"im","re","rows"]}]}
        ops = []
        for op in self.ops:
            o = {"name": gate_name(op.name), "wires": [int(w) for w in op.wires],
                 "params": [float(p) for p in op.params]}
            if op.name == Gate.unitary:
                m = np.asarray(op.matrix, dtype=np.complex128)
                o["rows"] = int(m.shape[0])
                o["re"] = [float(v) for v in m.real.reshape(-1)]
                o["im"] = [float(v) for v in m.imag.reshape(-1)]
            ops.append(o)
        return _dump({"n": int(self.n), "d": int(self.d), "ops": ops})

    @staticmethod
    def from_json(text: str) -> "Circuit":  # circuit.cpp:549-571
        j = json.loads(text)
        c = Circuit(j["n"], j.get("d", 2))
        for o in j["ops"]:
            g = Gate[o["name"]] if o["name"] in Gate.__members__ else None
            _require(g is not None, "unknown gate name: " + str(o["name"]))
            if g == Gate.unitary:
                rows = int(o["rows"])
                m = (np.array(o["re"], dtype=float) + 1j * np.array(o["im"], dtype=float))[: rows * rows]
                c.unitary(o["wires"], m.reshape(rows, rows))
            else:
                c.gate(g, o["wires"], o["params"])
        return c


def _dump(obj) -> str:
    """nlohmann::json::dump() layout: compact separators, keys sorted."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def _isfinite(p) -> bool:
    try:
        return math.isfinite(float(p))
    except TypeError:
        return True


def _circuit_ops(c: Circuit, slot_of=None):
    """Circuit -> (qf ops, constant matrices).  slot_of(op_index) -> (slot, coef, offset)."""
    ops, mats = [], []
    for i, op in enumerate(c.ops):
        g = Gate(op.name)
        q0 = op.wires[0]
        q1 = op.wires[1] if len(op.wires) > 1 else -1
        slot, coef, off, mat = -1, 1.0, 0.0, -1
        if g in (Gate.su4, Gate.unitary):
            m = gate_matrix(op)
            full = np.zeros((4, 4), dtype=np.complex128)
            full[: m.shape[0], : m.shape[1]] = m
            mats.append(full)
            mat = len(mats) - 1
        elif g in (Gate.rx, Gate.ry, Gate.rz, Gate.rzz):
            if slot_of is not None and slot_of[i] is not None:
                slot, coef, off = slot_of[i]
            else:
                off = float(op.params[0])
        elif g in (Gate.csum, Gate.subspace_ry, Gate.subspace_rz):
            raise ValueError("gate_matrix: qudit gates are not supported on the qubit device path")
        ops.append((int(g), q0, q1, slot, coef, off, mat))
    return ops, (np.array(mats) if mats else None)


def _check_qubits(c: Circuit) -> None:
    _require(c.d == 2, "device path: qubit circuits only (d == 2)")


def run(c: Circuit, memory_guard_log2: int = 24) -> StateVector:  # circuit.cpp:304-317
    _require(float(c.d) ** c.n <= 2.0 ** memory_guard_log2, "run: state dimension exceeds memory guard")
    _check_qubits(c)
    ops, mats = _circuit_ops(c)
    ctx = _eng.default_context()
    prog = _eng.Program(ctx, c.n, ops, 0, _precision, mats)
    if c.initial_state is not None:
        _require(np.asarray(c.initial_state).size == 2 ** c.n, "run: initial state size mismatch")
        prog.set_initial_state(c.initial_state)
    amps = _eng.run_state(ctx, prog, np.zeros(0), int(memory_guard_log2))
    return StateVector(c.n, c.d, amps)


def apply_local_unitary(psi: StateVector, u: np.ndarray, wires: Sequence[int]) -> None:
    """In-place U on `wires` (wires[0] most significant), circuit.cpp:78-176."""
    u = np.asarray(u, dtype=np.complex128)
    k = len(wires)
    _require(u.shape == (2 ** k, 2 ** k), "apply_local_unitary: wrong gate size")
    for w in wires:
        _require(0 <= w < psi.n, "apply_local_unitary: wire out of range")
    _require(len(set(wires)) == k, "apply_local_unitary: wires must be distinct")
    _require(1 <= k <= 13, "apply_local_unitary: 1 to 13 wires on the device path")
    psi.amps = _eng.apply_unitary(_eng.default_context(), psi.amps, u, list(wires))


# ---------------------------------------------------------------- Pauli sums
@dataclass
class PauliTerm:  # pauli.hpp:13-17
    weight: complex
    codes: list


class PauliSum:  # pauli.hpp:21-30
    def __init__(self, n: int = 0):
        self.n = n
        self.terms: list[PauliTerm] = []
        self._obs = weakref.WeakKeyDictionary()

    def add(self, weight, codes) -> None:  # pauli.cpp:12-18
        codes = [int(c) for c in codes]
        _require(len(codes) == self.n, "PauliSum::add: wrong code length")
        for c in codes:
            _require(0 <= c <= 3, "PauliSum::add: code out of range")
        w = complex(weight)
        _require(math.isfinite(w.real) and math.isfinite(w.imag), "PauliSum::add: non-finite weight")
        self.terms.append(PauliTerm(w, codes))

    def add_word(self, weight, site_codes) -> None:  # pauli.cpp:20-27
        codes = [0] * self.n
        for site, code in site_codes:
            _require(0 <= site < self.n, "PauliSum::add_word: site out of range")
            codes[site] = code
        self.add(weight, codes)

    def to_json(self) -> str:  # pauli.cpp:29-39: {"n","terms":[{"codes","w_im","w_re"}]}
        return _dump({"n": int(self.n), "terms": [{"w_re": float(t.weight.real), "w_im": float(t.weight.imag),
                                                    "codes": [int(c) for c in t.codes]} for t in self.terms]})

    @staticmethod
    def from_json(text: str) -> "PauliSum":  # pauli.cpp:41-50
        j = json.loads(text)
        h = PauliSum(j["n"])
        for t in j["terms"]:
            h.add(complex(t["w_re"], t["w_im"]), t["codes"])
        return h

    def arrays(self):
        codes = np.array([t.codes for t in self.terms], dtype=np.int8).reshape(len(self.terms), self.n)
        w = np.array([t.weight for t in self.terms], dtype=np.complex128)
        return codes, w

    def _content_key(self):
        return (self.n, tuple((complex(t.weight), tuple(int(c) for c in t.codes)) for t in self.terms))

    def observable(self, ctx=None) -> _eng.Observable:
        """Device copy for `ctx`, keyed on the context object (weakly) and on the
        sum's content: `terms` is public and may be edited in place."""
        ctx = ctx or _eng.default_context()
        if not isinstance(self._obs, weakref.WeakKeyDictionary):
            self._obs = weakref.WeakKeyDictionary()
        key = self._content_key()
        hit = self._obs.get(ctx)
        if hit is None or hit[0] != key:
            codes, w = self.arrays()
            hit = (key, _eng.Observable(ctx, self.n, codes, w))
            self._obs[ctx] = hit
        return hit[1]


class Lattice:
    """Chain subset of qforge::Lattice (lattice.hpp:30-45): sites + order-1 edges."""

    def __init__(self, n: int, edges):
        self.n = n
        self.edges_by_order = {1: list(edges)} if edges else {}

    def num_sites(self) -> int:
        return self.n


def build_lattice(kind: str, size, pbc, lattice_constant: float = 1.0, neighbor_order: int = 1) -> Lattice:
    """build_lattice(chain, {n}, {pbc}) with the neighbour-shell rule of
    lattice.cpp:89-122 (pairs sorted by distance, then i, then j)."""
    _require(kind == "chain", "build_lattice: only the chain lattice is on the device hot path")
    _require(lattice_constant > 0.0, "build_lattice: lattice_constant must be > 0")
    n = int(size[0])
    _require(n >= 1, "build_lattice: size entries must be >= 1")
    if pbc[0]:
        _require(n >= 3, "build_lattice: periodic dimension needs extent >= 3")
    pairs = []
    for i in range(n):
        for j in range(i + 1, n):
            d = abs(i - j) * lattice_constant
            if pbc[0]:
                d = min(abs((i - j + m * n) * lattice_constant) for m in (-1, 0, 1))
            pairs.append((d, i, j))
    pairs.sort()
    edges, order, shell = [], 0, -1.0
    for d, i, j in pairs:
        if d <= 0.0:
            continue
        if shell < 0.0 or d > shell * (1.0 + 1e-6):
            order += 1
            shell = d
        if order > neighbor_order:
            break
        if order == 1:
            edges.append((i, j))
    return Lattice(n, edges)


def tfim_terms(l: Lattice, g: float) -> PauliSum:  # pauli.cpp:181-189
    h = PauliSum(l.num_sites())
    _require(1 in l.edges_by_order, "tfim_terms: lattice has no order-1 edges")
    for i, j in l.edges_by_order[1]:
        h.add_word(-1.0, [(i, 3), (j, 3)])
    for i in range(h.n):
        h.add_word(-g, [(i, 1)])
    return h


def heisenberg_terms(l: Lattice, jx: float, jy: float, jz: float) -> PauliSum:  # pauli.cpp:191-203
    h = PauliSum(l.num_sites())
    _require(1 in l.edges_by_order, "heisenberg_terms: lattice has no order-1 edges")
    js = (jx, jy, jz)
    for i, j in l.edges_by_order[1]:
        for axis in range(3):
            if js[axis] != 0.0:
                h.add_word(js[axis], [(i, axis + 1), (j, axis + 1)])
    return h


def random_pauli_sum(n: int, terms: int, rng, real_weights: bool = True) -> PauliSum:
    """tests/helpers.hpp:52-63 draw order (codes, then weight).  For complex
    weights the reference's cplx(rng.normal(), rng.normal()) is evaluated
    right-to-left by gcc (pinned by oracle/_ref), so the imaginary part is drawn
    first."""
    h = PauliSum(n)
    for _ in range(terms):
        codes = [rng.uniform_below(4) for _ in range(n)]
        if real_weights:
            w = complex(rng.normal(), 0.0)
        else:
            im = rng.normal()
            re = rng.normal()
            w = complex(re, im)
        h.add(w, codes)
    return h


class SparseCOO:  # include/qforge/sparse.hpp:12-36 (canonical coordinate format)
    def __init__(self, dim: int = 0, rows=None, cols=None, vals=None):
        self.dim = dim
        self.rows = np.zeros(0, np.int64) if rows is None else rows
        self.cols = np.zeros(0, np.int64) if cols is None else cols
        self.vals = np.zeros(0, np.complex128) if vals is None else vals

    def nnz(self) -> int:
        return int(len(self.vals))

    def to_dense(self) -> np.ndarray:  # sparse.cpp:59-65 (test helper)
        m = np.zeros((self.dim, self.dim), dtype=np.complex128)
        np.add.at(m, (self.rows, self.cols), self.vals)
        return m


def pauli_sum_to_coo(h: PauliSum, n_guard: int = 26, workers: int = 1) -> SparseCOO:
    """pauli.cpp:89-153 on the GPU (qf_pauli_sum_to_coo); `workers` is accepted for
    signature compatibility (the output never depends on it)."""
    _require(h.n >= 1, "pauli_sum_to_coo: empty system")
    _require(h.n <= n_guard, "pauli_sum_to_coo: qubit count exceeds memory guard")
    ctx = _eng.default_context()
    rows, cols, vals = _eng.pauli_sum_to_coo(ctx, h.observable(ctx), n_guard)
    return SparseCOO(1 << h.n, rows, cols, vals)


def expectation_pauli(psi: StateVector, obs: PauliSum) -> complex:  # circuit.cpp:319-347
    _require(psi.d == 2, "expectation_pauli: qubits only")
    _require(obs.n == psi.n, "expectation_pauli: size mismatch")
    ctx = _eng.default_context()
    prog = _eng.Program(ctx, psi.n, [], 0, _precision)
    prog.set_initial_state(psi.amps)
    return _eng.expectation(ctx, prog, obs.observable(ctx), np.zeros(0))


# ---------------------------------------------------------------- variational
class GradMode(enum.IntEnum):  # variational.hpp:30 (+ adjoint)
    parameter_shift = 0
    finite_diff = 1
    adjoint = 2


class AnsatzSpec:  # variational.hpp:14-21
    def __init__(self, n_params: int = 0, builder: Optional[Callable] = None, shift_eligible=None):
        self.n_params = n_params
        self.builder = builder
        self.shift_eligible = list(shift_eligible) if shift_eligible is not None else []
        self._programs = weakref.WeakKeyDictionary()  # ctx -> {(precision, n_params, builder): Program}

    def validate(self) -> None:  # variational.cpp:11-16
        _require(self.n_params >= 0, "AnsatzSpec: negative parameter count")
        _require(self.builder is not None, "AnsatzSpec: missing builder")
        _require(len(self.shift_eligible) == self.n_params,
                 "AnsatzSpec: eligibility tags do not match parameter count")

    # -- parameter-slot discovery: the builder is opaque, so probe it
    def program(self, precision: Optional[str] = None, ctx=None) -> _eng.Program:
        precision = precision or _precision
        ctx = ctx or _eng.default_context()
        if not isinstance(self._programs, weakref.WeakKeyDictionary):
            self._programs = weakref.WeakKeyDictionary()
        per_ctx = self._programs.setdefault(ctx, {})
        key = (precision, self.n_params, id(self.builder), self.builder)  # builder/n_params are public fields
        if key not in per_ctx:
            per_ctx[key] = _compile_ansatz(self, precision, ctx)
        return per_ctx[key]


class TemplateUnavailable(ValueError):
    """The builder cannot be mapped to one fixed template (structure or initial
    state depends on theta, non-affine angles, theta feeding su4/unitary): the
    energy-only paths then evaluate it per parameter set (_per_theta_energies)."""


def _require_template(cond: bool, msg: str) -> None:
    if not cond:
        raise TemplateUnavailable(msg)


def _probe(builder, P: int, values: np.ndarray) -> Circuit:
    return builder(values.copy())


def ansatz_template(a: AnsatzSpec):
    """Parameter-slot discovery.  The builder is opaque
    (std::function in the reference, variational.hpp:16), so it is probed with
    four parameter vectors: every rotation angle must be coef * theta[slot] +
    offset for a single slot, with a theta-independent gate structure.
    Returns (n, ops, mats, initial_state) with ops in qf_op tuple form."""
    a.validate()
    P = a.n_params
    j = np.arange(P, dtype=np.float64)
    t0 = np.zeros(P)
    ta = 1.0 + 1e-3 * j + 0.137
    tb = ta * (2.0 + 1e-3 * j)
    tc = np.cos(3.7 * j + 0.3) * 2.1 + 0.05
    c0, ca, cb, cc = (_probe(a.builder, P, t) for t in (t0, ta, tb, tc))
    for c in (ca, cb, cc):
        _require_template(len(c.ops) == len(c0.ops) and c.n == c0.n and
                 all(x.name == y.name and x.wires == y.wires for x, y in zip(c.ops, c0.ops)),
                 "AnsatzSpec: builder structure depends on theta (device path needs a fixed structure)")
        _require_template((c.initial_state is None) == (c0.initial_state is None) and
                          (c.initial_state is None or np.array_equal(np.asarray(c.initial_state),
                                                                     np.asarray(c0.initial_state))),
                          "AnsatzSpec: theta feeds the initial state (not supported on the device path)")
    _check_qubits(c0)
    slot_of = []
    ratios = tb / ta if P else np.zeros(0)
    for i, op in enumerate(c0.ops):
        if Gate(op.name) not in (Gate.rx, Gate.ry, Gate.rz, Gate.rzz):
            for c in (ca, cb, cc):
                _require_template(np.array_equal(np.asarray(c.ops[i].params, dtype=float), np.asarray(op.params, dtype=float)) and
                         (op.matrix is None or np.array_equal(c.ops[i].matrix, op.matrix)),
                         "AnsatzSpec: theta feeds a gate without a Pauli generator "
                         "(su4/unitary parameters are not supported on the device path)")
            slot_of.append(None)
            continue
        o = float(op.params[0])
        da = float(ca.ops[i].params[0]) - o
        db = float(cb.ops[i].params[0]) - o
        if da == 0.0 and db == 0.0:
            _require_template(float(cc.ops[i].params[0]) == o, "AnsatzSpec: builder is not affine in theta")
            slot_of.append(None)
            continue
        _require_template(da != 0.0 and P > 0, "AnsatzSpec: builder is not affine in theta")
        s = int(np.argmin(np.abs(ratios - db / da)))
        coef = da / ta[s]
        pred = coef * tc[s] + o
        _require_template(abs(pred - float(cc.ops[i].params[0])) <= 1e-9 * max(1.0, abs(pred)),
                 "AnsatzSpec: builder is not affine in a single theta slot")
        slot_of.append((s, coef, o))
    ops, mats = _circuit_ops(c0, slot_of)
    return c0.n, ops, mats, c0.initial_state


def _compile_ansatz(a: AnsatzSpec, precision: str, ctx) -> _eng.Program:
    n, ops, mats, init = ansatz_template(a)
    prog = _eng.Program(ctx, n, ops, a.n_params, precision, mats)
    if init is not None:
        prog.set_initial_state(init)
    return prog


def tfim_chain_ansatz(n: int, layers: int) -> AnsatzSpec:  # variational.cpp:18-36
    _require(n >= 2, "tfim_chain_ansatz: n must be >= 2")
    _require(layers >= 1, "tfim_chain_ansatz: layers must be >= 1")

    def builder(theta):
        c = Circuit(n)
        for q in range(n):
            c.h(q)
        k = 0
        for _ in range(layers):
            for i in range(n):
                c.rx(i, theta[k]); k += 1
            for i in range(n - 1):
                c.rzz(i, i + 1, theta[k]); k += 1
        return c

    P = layers * (2 * n - 1)
    return AnsatzSpec(P, builder, [True] * P)


def hea_ansatz(n: int, layers: int) -> AnsatzSpec:
    """Synthetic hardware-efficient ansatz of the benchmark configs:
    per layer ry on every site, rz on every site, then cx(q, q+1) for q = 0..n-2."""
    _require(n >= 2, "hea_ansatz: n must be >= 2")
    _require(layers >= 1, "hea_ansatz: layers must be >= 1")

    def builder(theta):
        c = Circuit(n)
        k = 0
        for _ in range(layers):
            for q in range(n):
                c.ry(q, theta[k]); k += 1
            for q in range(n):
                c.rz(q, theta[k]); k += 1
            for q in range(n - 1):
                c.cx(q, q + 1)
        return c

    P = 2 * n * layers
    return AnsatzSpec(P, builder, [True] * P)


def _per_theta_energies(ansatz: AnsatzSpec, th: np.ndarray, h, precision: Optional[str] = None) -> np.ndarray:
    """The reference's own energy path (variational.cpp:38-52: build, run,
    expectation) for builders without a fixed template, one parameter set at a
    time, on the device: each circuit becomes a constant program (the generated
    kernels do not depend on angle values, so they come from the kernel cache)."""
    ctx = _eng.default_context()
    precision = precision or _precision
    E = np.zeros(th.shape[0])
    for b in range(th.shape[0]):
        c = ansatz.builder(th[b].copy())
        _check_qubits(c)
        ops, mats = _circuit_ops(c)
        prog = _eng.Program(ctx, c.n, ops, 0, precision, mats)
        if c.initial_state is not None:
            prog.set_initial_state(c.initial_state)
        if isinstance(h, SparseCOO):
            E[b] = _eng.sparse_energy(ctx, prog, np.zeros((1, 0)), h.dim, h.rows, h.cols, h.vals)[0]
        else:
            _require(h.n == c.n, "expectation_pauli: size mismatch")
            E[b] = _eng.energy_grad_batch(ctx, prog, h.observable(ctx), np.zeros((1, 0)), False)[0][0]
    return E


def energy_gradient_batch(ansatz: AnsatzSpec, thetas, h: PauliSum, grads: bool = True,
                          precision: Optional[str] = None):
    """Batched energy + adjoint gradient: (E[B], G[B, P]).  Energies of builders
    without a fixed template fall back to per-parameter-set evaluation; the
    adjoint gradient needs the template and raises its error."""
    ansatz.validate()
    th = np.asarray(thetas, dtype=np.float64)
    if ansatz.n_params == 0:
        th = th.reshape(th.shape[0] if th.ndim == 2 else 1, 0)
    else:
        th = th.reshape(-1, ansatz.n_params)
    ctx = _eng.default_context()
    try:
        prog = ansatz.program(precision, ctx)
    except TemplateUnavailable:
        if grads:
            raise
        return _per_theta_energies(ansatz, th, h, precision), None
    _require(h.n == prog.n, "expectation_pauli: size mismatch")
    return _eng.energy_grad_batch(ctx, prog, h.observable(ctx), th, grads)


def energy(ansatz: AnsatzSpec, theta, h) -> float:  # variational.cpp:38-43 (PauliSum), :45-52 (SparseCOO)
    ansatz.validate()
    theta = np.asarray(theta, dtype=np.float64).reshape(-1)
    _require(theta.size == ansatz.n_params, "energy: parameter count mismatch")
    if isinstance(h, SparseCOO):
        ctx = _eng.default_context()
        try:
            prog = ansatz.program(None, ctx)
        except TemplateUnavailable:
            return float(_per_theta_energies(ansatz, theta[None, :], h)[0])
        E = _eng.sparse_energy(ctx, prog, theta[None, :], h.dim, h.rows, h.cols, h.vals)
        return float(E[0])
    E, _ = energy_gradient_batch(ansatz, theta[None, :], h, grads=False)
    return float(E[0])


def gradient(ansatz: AnsatzSpec, theta, h: PauliSum, mode: GradMode, fd_step: float = 1e-5,
             workers: int = 1) -> np.ndarray:
    """variational.cpp:54-81.  parameter_shift / finite_diff keep the reference's
    2P-energy rule but evaluate all shifted energies as ONE device batch;
    GradMode.adjoint is one forward + one adjoint pass.  `workers` is accepted
    for signature compatibility (results never depend on it)."""
    ansatz.validate()
    theta = np.asarray(theta, dtype=np.float64).reshape(-1)
    _require(theta.size == ansatz.n_params, "gradient: parameter count mismatch")
    P = ansatz.n_params
    if mode == GradMode.adjoint:
        _, G = energy_gradient_batch(ansatz, theta[None, :], h)
        return G[0]
    if mode == GradMode.parameter_shift:
        for j in range(P):
            _require(ansatz.shift_eligible[j], "gradient: parameter not shift-eligible, use finite_diff")
    else:
        _require(fd_step > 0.0, "gradient: finite-diff step must be positive")
    shift = math.pi / 2.0 if mode == GradMode.parameter_shift else fd_step
    denom = 2.0 if mode == GradMode.parameter_shift else 2.0 * fd_step
    if P == 0:
        return np.zeros(0)
    T = np.repeat(theta[None, :], 2 * P, axis=0)
    for j in range(P):
        T[2 * j, j] = theta[j] + shift
        T[2 * j + 1, j] = theta[j] - shift
    E, _ = energy_gradient_batch(ansatz, T, h, grads=False)
    return (E[0::2] - E[1::2]) / denom


@dataclass
class AdamState:  # variational.hpp:39-43
    m: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None
    t: int = 0


def adam_step(state: AdamState, theta: np.ndarray, grad: np.ndarray, lr: float, beta1: float = 0.9,
              beta2: float = 0.999, eps: float = 1e-8) -> None:  # variational.cpp:83-101
    _require(theta.size == grad.size, "adam_step: shape mismatch")
    if state.t == 0:
        state.m = np.zeros(theta.size)
        state.v = np.zeros(theta.size)
    _require(state.m.size == theta.size, "adam_step: state shape mismatch")
    state.t += 1
    state.m = beta1 * state.m + (1.0 - beta1) * grad
    state.v = beta2 * state.v + (1.0 - beta2) * (grad * grad)
    c1 = 1.0 - beta1 ** state.t
    c2 = 1.0 - beta2 ** state.t
    mhat = state.m / c1
    vhat = state.v / c2
    theta -= lr * mhat / (np.sqrt(vhat) + eps)


@dataclass
class VqeResult:  # variational.hpp:48-53
    traces: list
    final_thetas: list
    best_energy: float = 0.0
    best_index: int = -1


def vqe_run(ansatz: AnsatzSpec, theta0_batch, h: PauliSum, steps: int, lr: float, grad_mode: GradMode,
            workers: int = 1) -> VqeResult:
    """variational.cpp:103-143 on the device: the whole batch advances together;
    theta, Adam m/v stay resident; one batched energy+gradient per step."""
    from .vqe import vqe_run_device

    try:
        ansatz.program(None, _eng.default_context())
    except TemplateUnavailable:
        if grad_mode == GradMode.adjoint:
            raise
        return _vqe_run_per_theta(ansatz, theta0_batch, h, steps, lr, grad_mode)
    return vqe_run_device(ansatz, theta0_batch, h, steps, lr, grad_mode)


def _vqe_run_per_theta(ansatz, theta0_batch, h, steps, lr, grad_mode) -> VqeResult:
    """variational.cpp:103-143 step for step (trace energy, gradient, Adam per
    seed) for builders without a fixed template; energies on the device."""
    _require(len(theta0_batch) > 0, "vqe_run: empty batch")
    _require(steps >= 1, "vqe_run: steps must be >= 1")
    traces, finals = [], []
    for th0 in theta0_batch:
        th = np.asarray(th0, dtype=np.float64).copy()
        st = AdamState()
        tr = []
        for _ in range(steps):
            tr.append(energy(ansatz, th, h))
            adam_step(st, th, gradient(ansatz, th, h, grad_mode), lr)
        tr.append(energy(ansatz, th, h))
        traces.append(tr)
        finals.append(th)
    res = VqeResult(traces, finals)
    for i, tr in enumerate(traces):
        if res.best_index < 0 or tr[-1] < res.best_energy:
            res.best_energy, res.best_index = tr[-1], i
    return res


# ---------------------------------------------------------------- noise (noise.hpp / noise.cpp)
class KrausChannel:  # noise.hpp:15-23
    def __init__(self, name: str = "", arity: int = 1, operators=None):
        self.name = name
        self.arity = arity
        self.operators = [np.asarray(k, dtype=np.complex128) for k in (operators or [])]

    def completeness_defect(self) -> float:  # noise.cpp:10-16
        if not self.operators:
            return 1.0
        d = self.operators[0].shape[0]
        acc = sum(k.conj().T @ k for k in self.operators)
        return float(np.abs(acc - np.eye(d)).max())

    def validate(self) -> None:  # noise.cpp:18-25
        _require(bool(self.operators), "KrausChannel: no operators")
        d = 1 << self.arity
        for k in self.operators:
            _require(k.shape == (d, d), "KrausChannel: wrong operator shape")
        _require(self.completeness_defect() <= 1e-10, "KrausChannel: completeness violated")


_PAULI = [np.eye(2, dtype=complex), np.array([[0, 1], [1, 0]], complex), np.array([[0, -1j], [1j, 0]]),
          np.diag([1.0 + 0j, -1.0])]


def depolarizing_channel(p: float, k: int = 1) -> KrausChannel:  # noise.cpp:27-60
    _require(0.0 <= p <= 1.0, "depolarizing_channel: p out of range")
    _require(1 <= k <= 3, "depolarizing_channel: arity out of range")
    words = 4 ** k
    pw = p / (words - 1)
    ops = []
    for w in range(words):
        weight = 1.0 - p if w == 0 else pw
        if weight == 0.0:
            continue
        op = np.eye(1, dtype=complex)
        ww = w
        for _ in range(k):  # site 0 is the least significant Kronecker factor
            op = np.kron(_PAULI[ww % 4], op)
            ww //= 4
        ops.append(np.sqrt(weight) * op)
    ch = KrausChannel("depolarizing", k, ops)
    ch.validate()
    return ch


def amplitude_damping_channel(gamma: float) -> KrausChannel:  # noise.cpp:62-72
    _require(0.0 <= gamma <= 1.0, "amplitude_damping_channel: gamma out of range")
    ch = KrausChannel("amplitude_damping", 1, [np.array([[1, 0], [0, np.sqrt(1.0 - gamma)]], complex),
                                               np.array([[0, np.sqrt(gamma)], [0, 0]], complex)])
    ch.validate()
    return ch


def phase_damping_channel(lam: float) -> KrausChannel:  # noise.cpp:74-84
    _require(0.0 <= lam <= 1.0, "phase_damping_channel: lambda out of range")
    ch = KrausChannel("phase_damping", 1, [np.array([[1, 0], [0, np.sqrt(1.0 - lam)]], complex),
                                           np.array([[0, 0], [0, np.sqrt(lam)]], complex)])
    ch.validate()
    return ch


def reset_channel(p: float) -> KrausChannel:  # noise.cpp:86-97
    _require(0.0 <= p <= 1.0, "reset_channel: p out of range")
    sp, sq = np.sqrt(p), np.sqrt(1.0 - p)
    ch = KrausChannel("reset", 1, [sq * np.eye(2, dtype=complex), np.array([[sp, 0], [0, 0]], complex),
                                   np.array([[0, sp], [0, 0]], complex)])
    ch.validate()
    return ch


def thermal_relaxation_channel(gamma: float, lam: float) -> KrausChannel:  # noise.cpp:99-111
    ad, pd = amplitude_damping_channel(gamma), phase_damping_channel(lam)
    ch = KrausChannel("thermal_relaxation", 1, [k2 @ k1 for k2 in pd.operators for k1 in ad.operators])
    ch.validate()
    return ch


class NoiseConf:  # noise.hpp:37-60, noise.cpp:113-145
    def __init__(self):
        self.rules = []  # (gate name or "", wires or None, predicate or None, channel)

    def attach(self, gate: str, channel: KrausChannel) -> None:
        channel.validate()
        self.rules.append((gate, None, None, channel))

    def attach_on_wires(self, gate: str, wires, channel: KrausChannel) -> None:
        channel.validate()
        _require(channel.arity == len(wires), "NoiseConf: channel arity does not match wire tuple")
        self.rules.append((gate, list(wires), None, channel))

    def attach_predicate(self, pred, channel: KrausChannel) -> None:
        channel.validate()
        self.rules.append(("", None, pred, channel))

    def match(self, instr) -> list:
        out = []
        for gate, wires, pred, ch in self.rules:
            if gate and gate != gate_name(Gate(instr.name)):
                continue
            if wires is not None and wires != list(instr.wires):
                continue
            if pred is not None and not pred(instr):
                continue
            if ch.arity != len(instr.wires):
                continue
            out.append(ch)
        return out


class Trajectory:  # noise.hpp:62-65
    def __init__(self, state: StateVector, log_prob: float):
        self.state = state
        self.log_prob = log_prob


def mc_trajectories(c: Circuit, conf: NoiseConf, rng, count: int) -> list:
    """`count` consecutive mc_trajectory(c, conf, rng) calls (noise.cpp:162-197) as
    one batched GPU run: the uniforms are drawn from `rng` in the same order."""
    _require(c.d == 2, "mc_trajectory: qubits only")
    ops, mats = _circuit_ops(c)
    chans, index, op_channels = [], {}, []
    for instr in c.ops:
        ids = []
        for ch in conf.match(instr):
            if id(ch) not in index:
                index[id(ch)] = len(chans)
                chans.append(ch.operators)
            ids.append(index[id(ch)])
        op_channels.append(ids)
    n_apps = sum(len(x) for x in op_channels)
    u = np.array([[rng.uniform() for _ in range(n_apps)] for _ in range(count)]).reshape(count, n_apps)
    ctx = _eng.default_context()
    states, logp, _ = _eng.noise_trajectories(ctx, c.n, ops, mats, op_channels, chans, u, _precision,
                                              init=c.initial_state)
    return [Trajectory(StateVector(c.n, 2, states[t]), float(logp[t])) for t in range(count)]


def mc_trajectory(c: Circuit, conf: NoiseConf, rng) -> Trajectory:  # noise.cpp:162-197
    return mc_trajectories(c, conf, rng, 1)[0]
