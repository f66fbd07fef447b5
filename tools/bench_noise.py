#!/usr/bin/env python
"""Batched noise trajectories (qf_noise_trajectories): HEA-like circuit with a
channel after every gate (depolarizing on cx, amplitude damping on ry, phase
damping on rz) or on cx only (the rotation runs between go through fused sweeps), T trajectories, per-trajectory time; CPU baseline: the numpy
oracle restatement on one trajectory."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200 import qforge as qf  # noqa: E402

ctx = engine.default_context(0)
for n, layers, T, sparse in [(16, 4, 1000, False), (20, 4, 256, False), (16, 4, 1000, True), (20, 4, 256, True)]:
    rng = po.Rng(9)
    ops = []
    for _ in range(layers):
        for q in range(n):
            ops.append((po.GID["ry"], q, -1, -1, 1.0, rng.uniform(), -1))
            ops.append((po.GID["rz"], q, -1, -1, 1.0, rng.uniform(), -1))
        for q in range(n - 1):
            ops.append((po.GID["cx"], q, q + 1, -1, 1.0, 0.0, -1))
    chans = [qf.depolarizing_channel(0.01, 2).operators, qf.amplitude_damping_channel(0.02).operators,
             qf.phase_damping_channel(0.02).operators]
    by = {po.GID["cx"]: [0], po.GID["ry"]: [1], po.GID["rz"]: [2]}
    op_ch = [by[o[0]] if (not sparse or o[0] == po.GID["cx"]) else [] for o in ops]
    n_apps = sum(len(c) for c in op_ch)
    u = np.array([[rng.uniform() for _ in range(n_apps)] for _ in range(T)])
    h = po.tfim(n, 1.0)
    obs = engine.Observable(ctx, n, h.codes, h.wr + 1j * h.wi)
    engine.noise_trajectories(ctx, n, ops, None, op_ch, chans, u[:2], "c64", obs=obs, want_states=False)
    dt = None
    for _rep in range(3):  # best of three calls (wall clock of one call is noisy)
        t0 = time.perf_counter()
        _, logp, ev = engine.noise_trajectories(ctx, n, ops, None, op_ch, chans, u, "c64", obs=obs, want_states=False)
        dt = min(dt, time.perf_counter() - t0) if dt is not None else time.perf_counter() - t0
    rec = {"n": n, "layers": layers, "gates": len(ops), "channel_applications": n_apps, "channels": "cx only (rotation runs fused)" if sparse else "after every gate", "trajectories": T,
           "precision": "c64", "seconds": dt, "s_per_traj": dt / T, "mean_energy": float(ev.mean())}
    if n <= 16:
        t0 = time.perf_counter()
        po.mc_trajectory(n, ops, op_ch, chans, u[0])
        rec["cpu_oracle_s_per_traj"] = time.perf_counter() - t0
    print(json.dumps(rec), flush=True)
