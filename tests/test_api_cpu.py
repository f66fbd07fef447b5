"""Host logic of the Python mirror of the reference API (no GPU): validation and
error behaviour (require() -> ValueError), model builders against the oracle,
RngStream against the reference header's golden values, wire formats, and the
parameter-slot discovery of opaque ansatz builders."""
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import qforge as qf
from paper_2602_14167_b200.rng import RngStream


def test_rngstream_matches_reference_golden():
    path = os.path.join(os.path.dirname(__file__), "golden", "rng_known_answers.txt")
    r3, r7, r11 = RngStream(3), RngStream(7), RngStream(11)
    kids = RngStream(0).split(8)
    for l in (l.split() for l in open(path)):
        if l[0] == "normal3":
            assert r3.normal() == float(l[1])
        elif l[0] == "u64_7":
            assert r7.next_u64() == int(l[1])
        elif l[0] == "split0":
            assert kids[int(l[1])].normal() == float(l[2])
        elif l[0] == "below5":
            assert r11.uniform_below(5) == int(l[1])
        elif l[0] == "uniform":
            assert r11.uniform() == float(l[1])


def test_random_pauli_sum_matches_oracle_draw_order():
    for real in (True, False):
        h = qf.random_pauli_sum(7, 25, RngStream(2005), real)
        ho = po.random_sum(7, 25, po.Rng(2005), real)
        codes, w = h.arrays()
        assert codes.tolist() == ho.codes.tolist()
        assert np.array_equal(w.real, ho.wr) and np.array_equal(w.imag, ho.wi)


def test_builders_match_oracle():
    for n in (2, 3, 10, 20):
        for pbc in (False, True):
            if pbc and n < 3:
                continue
            lat = qf.build_lattice("chain", [n], [pbc])
            for mine, ref in ((qf.tfim_terms(lat, 0.7), po.tfim(n, 0.7, pbc)),
                              (qf.heisenberg_terms(lat, 1.0, 0.0, 0.5), po.heisenberg(n, 1.0, 0.0, 0.5, pbc))):
                codes, w = mine.arrays()
                assert codes.tolist() == ref.codes.tolist()
                assert np.array_equal(w.real, ref.wr)


def test_circuit_validation_mirrors_reference():
    """circuit.cpp:178-186 / 188-200: wire range, duplicates, finite params, su4 arity, unitarity."""
    c = qf.Circuit(3)
    with pytest.raises(ValueError, match="wire out of range"):
        c.rx(3, 0.1)
    with pytest.raises(ValueError, match="duplicate wires"):
        c.cx(1, 1)
    with pytest.raises(ValueError, match="non-finite"):
        c.ry(0, float("inf"))
    with pytest.raises(ValueError, match="15 parameters"):
        c.su4(0, 1, [0.1] * 3)
    with pytest.raises(ValueError, match="not unitary"):
        c.unitary([0], np.array([[1, 1], [0, 1]]))
    c.h(0).cx(0, 1).rzz(1, 2, 0.3)
    c2 = qf.Circuit.from_json(c.to_json())
    assert [(o.name, o.wires, o.params) for o in c2.ops] == [(o.name, o.wires, o.params) for o in c.ops]


def test_pauli_sum_validation_and_json():
    h = qf.PauliSum(2)
    with pytest.raises(ValueError, match="wrong code length"):
        h.add(1.0, [1])
    with pytest.raises(ValueError, match="code out of range"):
        h.add(1.0, [4, 0])
    with pytest.raises(ValueError, match="non-finite"):
        h.add(float("nan"), [1, 0])
    with pytest.raises(ValueError, match="site out of range"):
        h.add_word(1.0, [(2, 1)])
    h.add(complex(0.5, -0.25), [2, 3])
    h2 = qf.PauliSum.from_json(h.to_json())
    assert h2.terms[0].weight == complex(0.5, -0.25) and h2.terms[0].codes == [2, 3]


def test_gate_matrix_conventions():
    """circuit.cpp:202-302."""
    t = 0.7
    c, s = math.cos(t / 2), math.sin(t / 2)
    assert np.allclose(qf.gate_matrix(qf.GateInstruction(qf.Gate.rx, [0], [t])), [[c, -1j * s], [-1j * s, c]])
    assert np.allclose(qf.gate_matrix(qf.GateInstruction(qf.Gate.rz, [0], [t])),
                       np.diag([np.exp(-0.5j * t), np.exp(0.5j * t)]))
    su4 = qf.gate_matrix(qf.GateInstruction(qf.Gate.su4, [0, 1], [0.1 * k for k in range(15)]))
    assert np.allclose(su4.conj().T @ su4, np.eye(4), atol=1e-12)


def test_slot_discovery_tca_and_hea_match_oracle_templates():
    for spec, ref in ((qf.tfim_chain_ansatz(5, 3), po.tca_template(5, 3)),
                      (qf.hea_ansatz(6, 2), po.hea_template(6, 2))):
        n, ops, mats, init = qf.ansatz_template(spec)
        assert n == ref[0] and len(ops) == len(ref[1])
        for mine, r in zip(ops, ref[1]):
            assert tuple(mine[:4]) == tuple(r[:4]) and float(mine[4]) == r[4] and float(mine[5]) == r[5]


def test_slot_discovery_affine_maps_and_errors():
    def builder(th):
        c = qf.Circuit(2)
        c.rx(0, 2.0 * th[1] - 0.5).ry(1, th[0]).rz(0, 0.25).cx(0, 1).rzz(0, 1, -th[1])
        return c

    n, ops, _, _ = qf.ansatz_template(qf.AnsatzSpec(2, builder, [True, True]))
    assert ops[0][3] == 1 and ops[0][4] == pytest.approx(2.0) and ops[0][5] == pytest.approx(-0.5)
    assert ops[1][3] == 0 and ops[1][4] == 1.0 and ops[1][5] == 0.0
    assert ops[2][3] == -1 and ops[2][5] == 0.25
    assert ops[4][3] == 1 and ops[4][4] == pytest.approx(-1.0)

    def nonaffine(th):
        return qf.Circuit(1).rx(0, math.sin(th[0]))

    with pytest.raises(ValueError, match="affine"):
        qf.ansatz_template(qf.AnsatzSpec(1, nonaffine, [True]))

    def structural(th):
        c = qf.Circuit(2)
        if th[0] > 0.5:
            c.h(1)
        return c.rx(0, th[0])

    with pytest.raises(ValueError, match="structure"):
        qf.ansatz_template(qf.AnsatzSpec(1, structural, [True]))
    with pytest.raises(ValueError, match="eligibility tags"):
        qf.ansatz_template(qf.AnsatzSpec(2, builder, [True]))
    # the template failures are TemplateUnavailable (the energy paths then evaluate
    # per parameter set); spec validation errors are plain ValueErrors
    for bad in (nonaffine, structural):
        with pytest.raises(qf.TemplateUnavailable):
            qf.ansatz_template(qf.AnsatzSpec(1, bad, [True]))

    def init_feed(th):
        c = qf.Circuit(1)
        c.initial_state = np.array([math.cos(th[0]), math.sin(th[0])], complex)
        return c.rx(0, 0.3)

    with pytest.raises(qf.TemplateUnavailable, match="initial state"):
        qf.ansatz_template(qf.AnsatzSpec(1, init_feed, [True]))
    try:
        qf.ansatz_template(qf.AnsatzSpec(2, builder, [True]))
    except qf.TemplateUnavailable:
        pytest.fail("a spec validation error must not select the per-theta path")
    except ValueError:
        pass


def test_adam_step_mirror():
    """variational.cpp:83-101, test_variational.cpp:167-177."""
    st = qf.AdamState()
    th = np.zeros(2)
    qf.adam_step(st, th, np.array([0.3, -7.0]), 0.05)
    assert th[0] == pytest.approx(-0.05, rel=1e-6) and th[1] == pytest.approx(0.05, rel=1e-6)


def test_kraus_channels_and_noise_rules():
    """noise.cpp:10-145 restated in qforge.py: completeness, operator counts and
    shapes, arity / range validation, rule matching (gate name, wire tuple,
    predicate, arity) in insertion order."""
    from paper_2602_14167_b200 import qforge as qf
    for ch, count in [(qf.depolarizing_channel(0.05, 1), 4), (qf.depolarizing_channel(0.05, 2), 16),
                      (qf.depolarizing_channel(0.0, 1), 1), (qf.amplitude_damping_channel(0.3), 2),
                      (qf.phase_damping_channel(0.4), 2), (qf.reset_channel(0.2), 3),
                      (qf.thermal_relaxation_channel(0.1, 0.2), 4)]:
        assert len(ch.operators) == count and ch.completeness_defect() < 1e-12
        assert all(k.shape == (1 << ch.arity, 1 << ch.arity) for k in ch.operators)
    # depolarizing: site 0 is the least significant Kronecker factor (noise.cpp:44-55)
    X = np.array([[0, 1], [1, 0]])
    d2 = qf.depolarizing_channel(0.3, 2).operators
    assert np.allclose(d2[1], np.sqrt(0.3 / 15) * np.kron(np.eye(2), X))
    for bad in (lambda: qf.depolarizing_channel(1.5), lambda: qf.depolarizing_channel(0.1, 4),
                lambda: qf.amplitude_damping_channel(-0.1), lambda: qf.reset_channel(2.0)):
        with pytest.raises(ValueError):
            bad()
    conf = qf.NoiseConf()
    dep2 = qf.depolarizing_channel(0.05, 2)
    conf.attach("cx", dep2)
    conf.attach("", qf.amplitude_damping_channel(0.1))
    conf.attach_on_wires("h", [1], qf.phase_damping_channel(0.2))
    conf.attach_predicate(lambda op: op.wires == [0], qf.reset_channel(0.1))
    with pytest.raises(ValueError, match="arity"):
        conf.attach_on_wires("cx", [0], dep2)
    c = qf.Circuit(3)
    c.h(0).h(1).cx(0, 1)
    names = [[ch.name for ch in conf.match(op)] for op in c.ops]
    assert names == [["amplitude_damping", "reset"], ["amplitude_damping", "phase_damping"], ["depolarizing"]]
