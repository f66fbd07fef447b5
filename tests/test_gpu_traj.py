"""Trajectory workload on the GPU: MIPT-Haar trajectories
(reference experiments.cpp:210-250) against the numpy restatement in
oracle/pyoracle.py, per trajectory."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,depth,p,traj", [(2, 3, 0.5, 4), (5, 6, 0.3, 6), (6, 10, 0.2, 8), (8, 8, 0.1, 5),
                                            (10, 3, 1.0, 3), (7, 0, 0.5, 2), (9, 5, 0.0, 3), (12, 6, 0.1, 3),
                                            (14, 4, 0.2, 2)])
@pytest.mark.parametrize("prec,tol", [("c128", 1e-9), ("c64", 2e-4)])
def test_mipt_haar_matches_oracle(ctx, n, depth, p, traj, prec, tol):
    ref = po.mipt_haar(n, depth, p, traj, 1234 + n)
    got, nmeas = engine.mipt_haar(ctx, n, depth, p, traj, 1234 + n, prec)
    assert np.abs(got - ref).max() <= tol, (got, ref)
    if p == 1.0:
        assert nmeas == n * depth * traj and np.abs(got).max() < 1e-6  # every qubit collapsed
    if p == 0.0:
        assert nmeas == 0


def test_mipt_haar_deterministic_and_validated(ctx):
    a, _ = engine.mipt_haar(ctx, 8, 6, 0.2, 6, 99, "c64")
    b, _ = engine.mipt_haar(ctx, 8, 6, 0.2, 6, 99, "c64")
    assert np.array_equal(a, b)
    for bad, msg in [((1, 4, 0.1, 2), "N must lie"), ((21, 4, 0.1, 2), "N must lie"), ((6, 4, 1.5, 2), "p must lie"),
                     ((6, 4, 0.1, 0), "trajectories")]:
        with pytest.raises(ValueError, match=msg):
            engine.mipt_haar(ctx, *bad, 1, "c64")


def test_mipt_haar_precisions_agree_at_size(ctx):
    """n = 16 (256 x 256 Schmidt problem, many tiny Schmidt values): complex64
    trajectories give the complex128 entropies to 1e-4 (the spectrum is always
    computed in double precision)."""
    a, na = engine.mipt_haar(ctx, 16, 12, 0.1, 4, 31, "c64")
    b, nb_ = engine.mipt_haar(ctx, 16, 12, 0.1, 4, 31, "c128")
    assert na == nb_ and np.abs(a - b).max() < 1e-4, (a, b)


@pytest.mark.parametrize("n,m,depth", [(1, 20, 0), (5, 64, 2), (8, 100, 3), (11, 40, 2)])
def test_shadow_snapshots_match_oracle(ctx, n, m, depth):
    """shadow_snapshots (shadows.cpp:50-85) with the shadow-gen randomness
    (experiments.cpp:252-274): identical outcome bits (complex128)."""
    ops, bases, us = po.shadow_gen_inputs(n, m, depth, 77 + n)
    psi = po.run(n, ops)
    ref = po.shadow_snapshots(psi, n, bases, us)
    prep = engine.Program(ctx, n, ops, 0, "c128")
    got = engine.shadow_snapshots(ctx, prep, None, bases, us)
    assert np.array_equal(got, ref)
    with pytest.raises(ValueError, match="bad basis code"):
        engine.shadow_snapshots(ctx, prep, None, np.zeros((2, n), np.int8), us[:2])


def test_shadow_gen_cli_dataset(ctx, tmp_path):
    from paper_2602_14167_b200 import cli
    args = ["shadow-gen", "--seed", "5", "--set", "n=6", "--set", "M=30", "--set", "depth=2"]
    assert cli.main(args + ["--out", str(tmp_path)]) == 0
    ds = [f for f in tmp_path.iterdir() if f.name.endswith(".dataset.csv")][0]
    lines = ds.read_text().splitlines()
    assert lines[0] == "6,30" and len(lines) == 31
    ops, bases, us = po.shadow_gen_inputs(6, 30, 2, 5)
    ref = po.shadow_snapshots(po.run(6, ops), 6, bases, us)
    for r, line in enumerate(lines[1:]):
        b, o = line.split(";")
        assert b == "".join(str(c) for c in bases[r]) and o == "".join(str(x) for x in ref[r])
    assert cli.main(["shadow-gen", "--out", str(tmp_path), "--set", "n=25"]) == 2


def _noisy_circuit(n, depth, rng):
    ops = []
    for _ in range(depth):
        for q in range(n):
            ops.append((po.GID["h"], q, -1, -1, 1.0, 0.0, -1))
            ops.append((po.GID["rx"], q, -1, -1, 1.0, 3.0 * rng.uniform() - 1.5, -1))
        for q in range(n - 1):
            ops.append((po.GID["cx"], q, q + 1, -1, 1.0, 0.0, -1))
        ops.append((po.GID["ry"], n - 1, -1, -1, 1.0, rng.uniform(), -1))
    return ops


def _channels_for(ops):
    from paper_2602_14167_b200 import qforge as qf
    chans = [qf.depolarizing_channel(0.05, 2).operators, qf.amplitude_damping_channel(0.08).operators,
             qf.phase_damping_channel(0.1).operators, qf.thermal_relaxation_channel(0.2, 0.3).operators,
             qf.reset_channel(0.15).operators]
    by = {po.GID["cx"]: [0], po.GID["h"]: [1], po.GID["rx"]: [2], po.GID["ry"]: [3, 4]}
    return [by.get(op[0], []) for op in ops], chans


@pytest.mark.parametrize("n,depth", [(2, 2), (4, 2), (6, 1)])
def test_noise_trajectories_match_oracle(ctx, n, depth):
    """mc_trajectory (noise.cpp:162-197) per trajectory with the same uniforms:
    states and log-probabilities (complex128), and the energy output path."""
    rng = po.Rng(40 + n)
    ops = _noisy_circuit(n, depth, rng)
    op_ch, chans = _channels_for(ops)
    T = 12
    n_apps = sum(len(x) for x in op_ch)
    u = np.array([[rng.uniform() for _ in range(n_apps)] for _ in range(T)])
    h = po.tfim(n, 0.7)
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    states, logp, ev = engine.noise_trajectories(ctx, n, ops, None, op_ch, chans, u, "c128", obs=obs)
    for t in range(T):
        ref_s, ref_l = po.mc_trajectory(n, ops, op_ch, chans, u[t])
        assert np.abs(states[t] - ref_s).max() < 1e-10 and abs(logp[t] - ref_l) < 1e-10
        assert abs(ev[t] - po.expectation(n, ref_s, h).real) < 1e-10


@pytest.mark.parametrize("n,depth,prec,tol", [(6, 2, "c128", 1e-10), (14, 2, "c128", 1e-10), (14, 1, "c64", 2e-5)])
def test_noise_sparse_channels_fused_runs(ctx, n, depth, prec, tol):
    """Channels only on cx: the channel-free h/rx runs between them go through
    compiled fused-sweep programs, the cx channels through the device-side branch
    picks (n = 14 uses 16 rho partials per state).  Same uniforms as the oracle."""
    rng = po.Rng(70 + n)
    ops = _noisy_circuit(n, depth, rng)
    op_ch, chans = _channels_for(ops)
    op_ch = [ch if op[0] == po.GID["cx"] else [] for ch, op in zip(op_ch, ops)]
    T = 6
    n_apps = sum(len(x) for x in op_ch)
    u = np.array([[rng.uniform() for _ in range(n_apps)] for _ in range(T)])
    states, logp, _ = engine.noise_trajectories(ctx, n, ops, None, op_ch, chans, u, prec)
    for t in range(T):
        ref_s, ref_l = po.mc_trajectory(n, ops, op_ch, chans, u[t])
        assert np.abs(states[t] - ref_s).max() < tol and abs(logp[t] - ref_l) < tol * 10


def test_noise_trajectory_reference_cases(ctx):
    """test_noise.cpp:175-214: empty configuration = pure run (log_prob 0); certain
    decay lands in the ground state; the trajectory average of <Z_0> matches the
    exact channel average within three sigma."""
    from paper_2602_14167_b200 import qforge as qf
    from paper_2602_14167_b200.rng import RngStream
    c = qf.Circuit(4)
    for q in range(4):
        c.h(q)
        c.rx(q, 0.3 + q)
    c.cx(0, 1).cx(1, 2)
    t = qf.mc_trajectory(c, qf.NoiseConf(), RngStream(3))
    assert np.abs(t.state.amps - qf.run(c).amps).max() < 1e-12 and t.log_prob == 0.0
    conf = qf.NoiseConf()
    conf.attach("x", qf.amplitude_damping_channel(1.0))
    one = qf.Circuit(1)
    one.x(0)
    for tr in qf.mc_trajectories(one, conf, RngStream(5), 20):
        assert abs(abs(tr.state.amps[0]) - 1.0) < 1e-12 and abs(tr.log_prob) < 1e-12
    rng = po.Rng(11)
    for rep in range(3):
        ops = _noisy_circuit(4, 2, rng)
        op_ch, chans = _channels_for(ops)
        exact = po.density_matrix_expect_z0(4, ops, op_ch, chans)
        T = 4000
        n_apps = sum(len(x) for x in op_ch)
        r2 = po.Rng(100 + rep)
        u = np.array([[r2.uniform() for _ in range(n_apps)] for _ in range(T)])
        z0 = engine.Observable(ctx, 4, np.array([[3, 0, 0, 0]], np.int8), np.array([1.0]))
        _, _, ev = engine.noise_trajectories(ctx, 4, ops, None, op_ch, chans, u, "c128", obs=z0, want_states=False)
        assert abs(ev.mean() - exact) < 3.0 / np.sqrt(T)


@pytest.mark.parametrize("m,batch", [(1, 2), (2, 3), (33, 2), (256, 2), (1024, 2), (1500, 1)])
def test_hermitian_eigvals_kernel(ctx, m, batch):
    """The MIPT entropy's own eigen-solver (Householder tridiagonalisation + Sturm
    bisection, eig.cu) against numpy eigvalsh: random Hermitian matrices and
    rank-deficient density matrices rho = A^H A (the MIPT case: many zero or tiny
    eigenvalues), absolute error <= 1e-12 * ||rho||."""
    rng = np.random.default_rng(m)
    mats = []
    for b in range(batch):
        if b % 2 == 0:
            x = rng.normal(size=(m, m)) + 1j * rng.normal(size=(m, m))
            mats.append((x + x.conj().T) / 2)
        else:
            r = max(1, m // 8)
            a = rng.normal(size=(r, m)) + 1j * rng.normal(size=(r, m))
            rho = a.conj().T @ a
            mats.append(rho / np.trace(rho).real)
    mats = np.array(mats)
    got = engine.hermitian_eigvals(ctx, mats)
    for b in range(batch):
        ref = np.linalg.eigvalsh(mats[b])
        scale = max(1.0, np.abs(ref).max())
        assert np.abs(got[b] - ref).max() <= 1e-12 * scale * max(1, m / 64), (b, np.abs(got[b] - ref).max())


@pytest.mark.parametrize("prec,tol", [("c128", 1e-10), ("c64", 2e-5)])
def test_noise_folded_branches_all_arities(ctx, prec, tol):
    """The last channel's Kraus branch of an op is folded into the next noisy op's
    pass when their wires are disjoint (apply2_rho): 1q -> 1q, 1q -> 2q, 2q -> 1q
    and 2q -> 2q hand-overs, plus overlapping ones that are applied alone; states
    and log-probabilities against the oracle per trajectory."""
    n = 6
    ops = []
    rng = po.Rng(91)
    for layer in range(3):
        ops += [(po.GID["cx"], 0, 1, -1, 1.0, 0.0, -1), (po.GID["cx"], 2, 3, -1, 1.0, 0.0, -1),  # 2q -> 2q
                (po.GID["h"], 4, -1, -1, 1.0, 0.0, -1),                                          # 2q -> 1q
                (po.GID["cx"], 0, 5, -1, 1.0, 0.0, -1),                                          # 1q -> 2q
                (po.GID["rx"], 1, -1, -1, 1.0, 3.0 * rng.uniform() - 1.5, -1),                   # 2q -> 1q
                (po.GID["rx"], 2, -1, -1, 1.0, 3.0 * rng.uniform() - 1.5, -1),                   # 1q -> 1q
                (po.GID["cx"], 2, 4, -1, 1.0, 0.0, -1)]                                          # overlap
    op_ch, chans = _channels_for(ops)
    op_ch = [[0] if op[0] == po.GID["cx"] else ([1, 2] if op[0] == po.GID["h"] else [2]) for op in ops]
    T = 8
    n_apps = sum(len(x) for x in op_ch)
    u = np.array([[rng.uniform() for _ in range(n_apps)] for _ in range(T)])
    states, logp, _ = engine.noise_trajectories(ctx, n, ops, None, op_ch, chans, u, prec)
    for t in range(T):
        ref_s, ref_l = po.mc_trajectory(n, ops, op_ch, chans, u[t])
        assert np.abs(states[t] - ref_s).max() < tol and abs(logp[t] - ref_l) < tol * 10
