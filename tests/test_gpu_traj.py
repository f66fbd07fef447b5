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
