"""Trajectory workload on the GPU: MIPT-Haar trajectories
(reference experiments.cpp:210-250) against the numpy restatement in
oracle/pyoracle.py, per trajectory."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,depth,p,traj", [(2, 3, 0.5, 4), (5, 6, 0.3, 6), (6, 10, 0.2, 8), (8, 8, 0.1, 5),
                                            (10, 3, 1.0, 3), (7, 0, 0.5, 2), (9, 5, 0.0, 3)])
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
