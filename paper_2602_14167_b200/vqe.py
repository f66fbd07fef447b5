"""vqe_run on the device (reference src/variational.cpp:103-143).

The reference loops per batch entry on CPU threads: energy -> gradient (2P
energies) -> adam_step, `steps` times, then a final energy and best-of-batch.
Here the whole batch advances in lock step inside one native call (qf_vqe_run,
csrc/capi.cpp): theta, the Adam moments and the energy traces stay resident in
HBM, each step is one batched energy + gradient evaluation (adjoint: one forward
+ one adjoint pass; parameter_shift / finite_diff: one batched call over the 2P
shifted parameter sets, same rule as the reference) followed by one Adam kernel.
Trace semantics are the reference's: trace[s] is the energy before update s, the
final energy is appended, best is the first strict minimum.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import engine as _eng


def vqe_run_device(ansatz, theta0_batch, h, steps: int, lr: float, grad_mode, precision=None):
    from .qforge import GradMode, VqeResult, _require

    ansatz.validate()
    theta0 = [np.asarray(t, dtype=np.float64).reshape(-1) for t in theta0_batch]
    _require(len(theta0) > 0, "vqe_run: empty batch")
    _require(steps >= 1, "vqe_run: steps must be >= 1")
    P = ansatz.n_params
    for t in theta0:
        _require(t.size == P, "gradient: parameter count mismatch")
    mode = GradMode(grad_mode)
    if mode == GradMode.parameter_shift:
        for j in range(P):
            _require(ansatz.shift_eligible[j], "gradient: parameter not shift-eligible, use finite_diff")
    ctx = _eng.default_context()
    prog = ansatz.program(precision, ctx)
    obs = h.observable(ctx)
    _require(h.n == prog.n, "expectation_pauli: size mismatch")
    B = len(theta0)
    th = np.ascontiguousarray(np.stack(theta0)) if P else np.zeros((B, 0))
    traces = np.empty((B, steps + 1), dtype=np.float64)
    fin = np.empty((B, P), dtype=np.float64)
    best_e = ctypes.c_double()
    best_i = ctypes.c_int()
    _eng.check(ctx.lib.qf_vqe_run(ctx.handle, prog.handle, obs.handle, B, _eng.dptr(th), int(steps), float(lr),
                                  int(mode), 1e-5, _eng.dptr(traces), _eng.dptr(fin), ctypes.byref(best_e),
                                  ctypes.byref(best_i)))
    return VqeResult([list(map(float, traces[b])) for b in range(B)], [fin[b].copy() for b in range(B)],
                     float(best_e.value), int(best_i.value))
