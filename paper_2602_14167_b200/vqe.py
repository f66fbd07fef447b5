"""vqe_run on the device (reference src/variational.cpp:103-143).

The reference loops per batch entry on CPU threads: energy -> gradient (2P
energies) -> adam_step, `steps` times, then a final energy and best-of-batch.
Here the whole batch advances in lock step on the GPU: theta and the Adam
moments stay resident in HBM, each step is one batched energy + gradient call
(adjoint: one forward + one adjoint pass; parameter_shift / finite_diff: one
batched call over the 2P shifted parameter sets, same rule as the reference)
followed by one Adam kernel.  Trace semantics are the reference's: trace[s] is
the energy before update s, the final energy is appended, best is the first
strict minimum.
"""
from __future__ import annotations

import math

import numpy as np

from . import engine as _eng


def vqe_run_device(ansatz, theta0_batch, h, steps: int, lr: float, grad_mode, precision=None):
    import torch

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
    dev = torch.device("cuda", ctx.device)
    ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
    with torch.cuda.stream(ext):
        theta = torch.tensor(np.stack(theta0), dtype=torch.float64, device=dev).contiguous()
        m = torch.zeros_like(theta)
        v = torch.zeros_like(theta)
        g = torch.zeros_like(theta)
        trace = torch.zeros((steps + 1, B), dtype=torch.float64, device=dev)
        if mode != GradMode.adjoint:
            shift = math.pi / 2.0 if mode == GradMode.parameter_shift else 1e-5
            denom = 2.0 if mode == GradMode.parameter_shift else 2.0e-5
            eye = torch.eye(P, dtype=torch.float64, device=dev) * shift
            Es = torch.zeros(B * 2 * P, dtype=torch.float64, device=dev)
        for s in range(steps):
            if mode == GradMode.adjoint:
                _eng.energy_grad_batch_device(ctx, prog, obs, theta, trace[s], g)
            else:
                _eng.energy_grad_batch_device(ctx, prog, obs, theta, trace[s], None)
                if P:
                    T = torch.stack([theta[:, None, :] + eye[None], theta[:, None, :] - eye[None]], dim=2)
                    T = T.reshape(B * 2 * P, P).contiguous()
                    _eng.energy_grad_batch_device(ctx, prog, obs, T, Es, None)
                    E2 = Es.view(B, P, 2)
                    g.copy_((E2[:, :, 0] - E2[:, :, 1]) / denom)
            _eng.adam_step_device(ctx, theta, m, v, g, s + 1, lr)
        _eng.energy_grad_batch_device(ctx, prog, obs, theta, trace[steps], None)
        tr = trace.t().contiguous().cpu().numpy()
        fin = theta.cpu().numpy()
    torch.cuda.synchronize(dev)
    best_e, best_i = math.inf, -1
    for b in range(B):  # strict <, first index wins (variational.cpp:133-141)
        if tr[b, steps] < best_e:
            best_e, best_i = float(tr[b, steps]), b
    return VqeResult([list(map(float, tr[b])) for b in range(B)], [fin[b].copy() for b in range(B)],
                     best_e, best_i)
