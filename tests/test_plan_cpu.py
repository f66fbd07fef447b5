"""Host-side scheduler checks (no GPU): the fused-sweep plan produced by
libqforge_b200.so (qf_plan_describe) is replayed in numpy.

 * forward: gates in sweep/phase order reproduce program order (the reordering
   only swaps commuting gates);
 * adjoint: inverse gates in the scheduled order, with Im<lambda|G|psi> taps
   taken where the plan puts them, reproduce the reference's parameter-shift
   gradient (oracle) -- this validates the commutation-DAG argument of
   DESIGN.md for reordered adjoint taps;
 * tile / register-bit constraints of every op.
Small tiles (QF_GEOM_C64) force many sweeps at small n."""
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import engine

G = po.GID
DK_TX, DK_TY, DK_TZ, DK_TZZ = 8, 9, 10, 11


def gate_matrix(kind, p, mats=None, mat=-1):
    c, s = math.cos(p / 2), math.sin(p / 2)
    isq = 1 / math.sqrt(2)
    if kind == G["h"]:
        return np.array([[isq, isq], [isq, -isq]], complex)
    if kind == G["x"]:
        return np.array([[0, 1], [1, 0]], complex)
    if kind == G["y"]:
        return np.array([[0, -1j], [1j, 0]])
    if kind == G["z"]:
        return np.diag([1, -1]).astype(complex)
    if kind == G["s"]:
        return np.diag([1, 1j])
    if kind == G["rx"]:
        return np.array([[c, -1j * s], [-1j * s, c]])
    if kind == G["ry"]:
        return np.array([[c, -s], [s, c]], complex)
    if kind == G["rz"]:
        return np.diag([np.exp(-0.5j * p), np.exp(0.5j * p)])
    if kind == G["rzz"]:
        return np.diag([np.exp(-0.5j * p), np.exp(0.5j * p), np.exp(0.5j * p), np.exp(-0.5j * p)])
    if kind == G["cx"]:
        return np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], complex)
    if kind == G["cz"]:
        return np.diag([1, 1, 1, -1]).astype(complex)
    m = np.asarray(mats[mat], complex)
    return m if m.shape == (4, 4) and kind in (G["su4"], G["unitary"]) and mat >= 0 else m


def apply(psi, n, u, wires):
    """wires[0] most significant local bit; site q = tensor axis q."""
    k = len(wires)
    t = psi.reshape([2] * n)
    t = np.moveaxis(t, wires, list(range(k)))
    sh = t.shape
    t = (u @ t.reshape(1 << k, -1)).reshape(sh)
    return np.moveaxis(t, list(range(k)), wires).reshape(-1)


GEN = {G["rx"]: np.array([[0, 1], [1, 0]], complex), G["ry"]: np.array([[0, -1j], [1j, 0]]),
       G["rz"]: np.diag([1, -1]).astype(complex), G["rzz"]: np.diag([1, -1, -1, 1]).astype(complex)}


def template_ops(ops, theta):
    out = []
    for o in ops:
        kind, q0, q1, slot, coef, off, mat = o
        p = coef * theta[slot] + off if slot >= 0 else off
        out.append((kind, [q0] if q1 < 0 else [q0, q1], p))
    return out


def hamil_dense_apply(h, psi, n):
    out = np.zeros_like(psi)
    P = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1, -1])]
    for t in range(len(h.wr)):
        v = psi
        for q, c in enumerate(h.codes[t]):
            if c:
                v = apply(v, n, P[c].astype(complex), [q])
        out += h.wr[t] * v  # Hermitian part (Re w): what energy and gradient depend on
    return out


def random_template(n, depth, rng):
    ops, slot = [], 0
    for layer in range(depth):
        for q in range(n):
            r = rng.uniform_below(6)
            kind = [G["h"], G["rx"], G["ry"], G["rz"], G["s"], G["x"]][r]
            if kind in (G["rx"], G["ry"], G["rz"]):
                ops.append((kind, q, -1, slot, 1.0 + 0.25 * rng.uniform(), 0.1 * rng.normal(), -1))
                slot += 1
            else:
                ops.append((kind, q, -1, -1, 1.0, 0.0, -1))
        for q in range(layer % 2, n - 1, 2):
            r = rng.uniform_below(3)
            if r == 0:
                ops.append((G["cx"], q, q + 1, -1, 1.0, 0.0, -1))
            elif r == 1:
                ops.append((G["rzz"], q + 1, q, slot, 1.0, 0.0, -1))
                slot += 1
            else:
                ops.append((G["cz"], q, q + 1, -1, 1.0, 0.0, -1))
    return ops, slot


CASES = [("hea7", *po.hea_template(7, 3)[1:], "6,3,5,2"),
         ("tca8", *po.tca_template(8, 2)[1:], "5,2,4,2"),
         ("hea9", *po.hea_template(9, 2)[1:], "6,3,5,3")]


@pytest.fixture(autouse=True)
def _small_tiles(monkeypatch):
    yield


def _plan(n, ops, P, geom, monkeypatch):
    monkeypatch.setenv("QF_GEOM_C64", geom)
    return engine.describe_plan(n, ops, P, "c64")


@pytest.mark.parametrize("name,ops,P,geom", CASES + [
    ("rand6", *random_template(6, 4, po.Rng(101)), "4,2,4,2"),
    ("rand8", *random_template(8, 3, po.Rng(102)), "5,3,5,2")])
def test_schedule_replays_program(name, ops, P, geom, monkeypatch):
    n = max(max(o[1], o[2]) for o in ops) + 1
    plan = _plan(n, ops, P, geom, monkeypatch)
    rng = np.random.default_rng(7)
    theta = rng.normal(size=P)
    concrete = template_ops(ops, theta)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi0 /= np.linalg.norm(psi0)
    ref = psi0.copy()
    for kind, w, p in concrete:
        ref = apply(ref, n, gate_matrix(kind, p), w)
    for pname in ("fwd", "bwd"):
        pp = plan["passes"][pname]
        seen = []
        for sw in pp["sweeps"]:
            tb = set(sw["tile_bits"])
            assert len(tb) == pp["k"]
            if n > pp["k"]:
                assert {0, 1} <= tb  # coalescing bits always resident
            for ph in sw["phases"]:
                reg = set(ph["reg_bits"])
                assert reg <= tb and len(reg) == pp["R"]
                for dk, g, tap in ph["ops"]:
                    if dk in (DK_TX, DK_TY, DK_TZ, DK_TZZ):
                        continue
                    seen.append(g)
                    kind, q0, q1 = ops[g][0], ops[g][1], ops[g][2]
                    need = []
                    if kind in (G["h"], G["x"], G["y"], G["rx"], G["ry"]):
                        need = [q0]
                    elif kind == G["cx"]:
                        need = [q1]
                    assert {n - 1 - q for q in need} <= reg, (pname, g)
        assert sorted(seen) == list(range(len(ops)))
        if pname == "fwd":
            psi = psi0.copy()
            for g in seen:
                kind, w, p = concrete[g]
                psi = apply(psi, n, gate_matrix(kind, p), w)
            assert np.abs(psi - ref).max() < 1e-12
        else:
            psi = ref.copy()
            for g in seen:
                kind, w, p = concrete[g]
                psi = apply(psi, n, gate_matrix(kind, p).conj().T, w)
            assert np.abs(psi - psi0).max() < 1e-12


@pytest.mark.parametrize("name,ops,P,geom", CASES)
def test_scheduled_adjoint_matches_parameter_shift(name, ops, P, geom, monkeypatch):
    n = max(max(o[1], o[2]) for o in ops) + 1
    plan = _plan(n, ops, P, geom, monkeypatch)
    h = po.heisenberg(n, 1.0, 0.7, 0.5)
    r = po.Rng(55)
    theta = np.array([r.normal() for _ in range(P)])
    concrete = template_ops(ops, theta)
    psi = po.run(n, ops, theta)
    lam = hamil_dense_apply(h, psi, n)
    bwd = plan["passes"]["bwd"]
    taps = np.zeros(bwd["n_taps"])
    for sw in bwd["sweeps"]:
        for ph in sw["phases"]:
            for dk, g, tap in ph["ops"]:
                kind, w, p = concrete[g]
                if dk in (DK_TX, DK_TY, DK_TZ, DK_TZZ):
                    gp = apply(psi, n, GEN[kind], w)
                    taps[sw["tap_begin"] + tap] = np.vdot(lam, gp).imag
                    continue
                u = gate_matrix(kind, p).conj().T
                psi = apply(psi, n, u, w)
                lam = apply(lam, n, u, w)
    grad = np.zeros(P)
    for t, (slot, coef) in enumerate(bwd["taps"]):
        grad[slot] += coef * taps[t]
    gs = po.gradient(po.Ansatz(n, ops, P), theta, h, "parameter_shift")
    assert np.abs(grad - gs).max() <= 1e-11 * max(1.0, np.abs(gs).max())


def test_default_geometry_sweep_counts():
    """The C2 schedule (20-qubit HEA depth 8) needs far fewer sweeps than one
    per layer per tile arrangement (S*D = 16 forward)."""
    _, ops, P = po.hea_template(20, 8)
    plan = engine.describe_plan(20, ops, P, "c64")
    assert len(plan["passes"]["fwd"]["sweeps"]) <= 16
    assert len(plan["passes"]["bwd"]["sweeps"]) <= 16
    assert plan["passes"]["bwd"]["n_taps"] == P


def test_invalid_programs_raise_value_error():
    with pytest.raises(ValueError, match="wire out of range"):
        engine.describe_plan(3, [(G["rx"], 3, -1, -1, 1.0, 0.0, -1)], 0)
    with pytest.raises(ValueError, match="duplicate wires"):
        engine.describe_plan(3, [(G["cx"], 1, 1, -1, 1.0, 0.0, -1)], 0)
    with pytest.raises(ValueError, match="non-finite"):
        engine.describe_plan(3, [(G["rx"], 1, -1, -1, 1.0, float("nan"), -1)], 0)
    with pytest.raises(ValueError, match="qudit"):
        engine.describe_plan(3, [(G["csum"], 0, 1, -1, 1.0, 0.0, -1)], 0)
    with pytest.raises(ValueError, match="not unitary"):
        engine.describe_plan(2, [(G["unitary"], 0, 1, -1, 1.0, 0.0, 0)], 0, mats=[2 * np.eye(4)])


def test_searched_schedule_of_the_headline_config():
    """The C2 template (n = 20, HEA depth 8, complex64) is scheduled by the tile and
    phase searches into 6 forward + 6 adjoint sweeps with at most 53 phases (the
    greedy schedule needed 9 + 13 sweeps and 75 phases); every sweep's tile is
    k bits and every phase's register set R bits."""
    n, D = 20, 8
    ops, P = [], 0
    for _ in range(D):
        for q in range(n):
            ops.append((G["ry"], q, -1, P, 1.0, 0.0, -1)); P += 1
        for q in range(n):
            ops.append((G["rz"], q, -1, P, 1.0, 0.0, -1)); P += 1
        for q in range(n - 1):
            ops.append((G["cx"], q, q + 1, -1, 1.0, 0.0, -1))
    d = engine.describe_plan(n, ops, P, "c64")["passes"]
    assert len(d["fwd"]["sweeps"]) == 6 and len(d["bwd"]["sweeps"]) == 6
    phases = sum(len(s["phases"]) for p in ("fwd", "bwd") for s in d[p]["sweeps"])
    assert phases <= 53, phases
    for p in ("fwd", "bwd"):
        k, R = d[p]["k"], d[p]["R"]
        for s in d[p]["sweeps"]:
            assert len(s["tile_bits"]) == k
            assert all(len(ph["reg_bits"]) == R for ph in s["phases"])
