"""Thin Python handles over the C-ABI objects (qf_ctx, qf_program, qf_observable).

The numerics live in libqforge_b200.so (sm_100a kernels + C++ scheduler); this
module only moves host buffers in and out.  Nothing here computes amplitudes.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import QfOp, check, dptr

PRECISIONS = {"c64": _lib.QF_C64, "c128": _lib.QF_C128, _lib.QF_C64: _lib.QF_C64,
              _lib.QF_C128: _lib.QF_C128}


class Context:
    """One GPU (qf_ctx): stream, scratch buffers, optional NCCL communicator."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        self.device = device
        h = ctypes.c_void_p()
        check(self.lib.qf_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.rank, self.world = 0, 1

    @property
    def stream(self) -> int:
        return self.lib.qf_ctx_stream(self.handle) or 0

    def set_memory_budget(self, nbytes: int) -> None:
        check(self.lib.qf_ctx_set_memory_budget(self.handle, int(nbytes)))

    def set_timing(self, on) -> None:
        """False/0 off, True/1 per kernel class, 2 also per launch (launch_times)."""
        check(self.lib.qf_ctx_set_timing(self.handle, int(on)))

    def flops(self):
        """Canonical algorithmic flops per kernel class since reset_stats."""
        f = np.zeros(4)
        check(self.lib.qf_ctx_flops(self.handle, dptr(f)))
        return f.tolist()

    def launch_times(self) -> dict:
        """{launch id: (ms, count)} since reset_stats (timing level 2): forward sweep i,
        1000 = H|psi>, 2000 + i = adjoint sweep i."""
        n = ctypes.c_int()
        check(self.lib.qf_ctx_launch_times(self.handle, 0, None, None, None, ctypes.byref(n)))
        ids = (ctypes.c_int * max(1, n.value))()
        ms = np.zeros(max(1, n.value))
        cnt = (ctypes.c_longlong * max(1, n.value))()
        check(self.lib.qf_ctx_launch_times(self.handle, n.value, ids, dptr(ms), cnt, ctypes.byref(n)))
        return {int(ids[i]): (float(ms[i]), int(cnt[i])) for i in range(n.value)}

    def reset_stats(self) -> None:
        check(self.lib.qf_ctx_reset_stats(self.handle))

    def stats(self):
        """(launches, launches per class, ms per class, algorithmic bytes per class);
        classes: forward sweeps, H|psi>, adjoint sweeps, reductions."""
        launches = ctypes.c_longlong()
        cl = (ctypes.c_longlong * 4)()
        ms = (ctypes.c_double * 4)()
        by = (ctypes.c_double * 4)()
        check(self.lib.qf_ctx_stats(self.handle, ctypes.byref(launches), cl, ms, by))
        return int(launches.value), list(cl), list(ms), list(by)

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _lib.load()
        buf = (ctypes.c_uint8 * 128)()
        check(lib.qf_nccl_unique_id(buf))
        return bytes(buf)

    def set_comm(self, rank: int, world: int, uid: Optional[bytes]) -> None:
        buf = (ctypes.c_uint8 * 128)(*(uid or bytes(128)))
        check(self.lib.qf_ctx_set_comm(self.handle, rank, world, buf))
        self.rank, self.world = rank, world

    def close(self) -> None:
        if self.handle:
            self.lib.qf_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: Optional[int] = None) -> Context:
    if device is None:
        try:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:
            device = 0
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _op_array(ops):
    arr = (QfOp * max(1, len(ops)))()
    for i, op in enumerate(ops):
        kind, q0, q1, slot, coef, offset, mat = op
        if isinstance(kind, str):
            kind = _lib.GATE_ID[kind]
        arr[i] = QfOp(int(kind), int(q0), int(q1), int(slot), float(coef), float(offset), int(mat), 0)
    return arr


def _mats_array(mats):
    if mats is not None and len(mats):
        m = np.ascontiguousarray(np.asarray(mats, dtype=np.complex128).reshape(-1, 4, 4))
        return m.view(np.float64).reshape(-1), m.shape[0]
    return None, 0


def describe_plan(n: int, ops: Sequence, n_params: int, precision="c128", mats=None) -> dict:
    """The fused-sweep schedule of a circuit template (host only, no GPU)."""
    import json

    lib = _lib.load()
    arr = _op_array(ops)
    mv, nm = _mats_array(mats)
    need = ctypes.c_size_t()
    check(lib.qf_plan_describe(n, len(ops), arr, dptr(mv), nm, n_params, PRECISIONS[precision], None, 0,
                               ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib.qf_plan_describe(n, len(ops), arr, dptr(mv), nm, n_params, PRECISIONS[precision], buf, need.value,
                               ctypes.byref(need)))
    return json.loads(buf.value.decode())


def jit_compile_check(n: int, ops: Sequence, n_params: int, precision="c128", mats=None) -> int:
    """NVRTC-compile every specialised sweep kernel of the template (host only)."""
    lib = _lib.load()
    arr = _op_array(ops)
    mv, nm = _mats_array(mats)
    k = ctypes.c_int()
    check(lib.qf_jit_compile_check(n, len(ops), arr, dptr(mv), nm, n_params, PRECISIONS[precision], ctypes.byref(k)))
    return k.value


def jit_hpsi_check(n: int, codes, weights, precision="c128") -> bool:
    """NVRTC-compile the specialised H|psi> kernel of a Pauli sum (host only);
    False when the sum is above the specialisation limit (generic kernel)."""
    lib = _lib.load()
    codes = np.ascontiguousarray(np.asarray(codes, dtype=np.int8).reshape(-1, n))
    w = np.asarray(weights, dtype=np.complex128).reshape(-1)
    wr, wi = np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag)
    k = ctypes.c_int()
    check(lib.qf_jit_hpsi_check(n, int(w.size), ctypes.c_void_p(codes.ctypes.data), dptr(wr), dptr(wi),
                                PRECISIONS[precision], ctypes.byref(k)))
    return bool(k.value)


class Program:
    """A compiled circuit template (qf_program).

    ops: sequence of (kind, q0, q1, slot, coef, offset, mat) with kind a gate
    name or qforge::Gate number; mats: [M, 4, 4] complex constant matrices.
    """

    def __init__(self, ctx: Context, n: int, ops: Sequence, n_params: int, precision="c128",
                 mats: Optional[np.ndarray] = None):
        self.ctx, self.n, self.n_params = ctx, n, n_params
        self.precision = PRECISIONS[precision]
        arr = _op_array(ops)
        mv, nm = _mats_array(mats)
        self._mats_keepalive = mv
        h = ctypes.c_void_p()
        check(ctx.lib.qf_program_create(ctx.handle, n, len(ops), arr, dptr(mv), nm, n_params,
                                        self.precision, ctypes.byref(h)))
        self.handle = h

    def set_initial_state(self, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(np.asarray(amps, dtype=np.complex128).reshape(-1))
        if a.size != (1 << self.n):
            raise ValueError("run: initial state size mismatch")
        check(self.ctx.lib.qf_program_set_initial_state(self.handle, dptr(a.view(np.float64))))

    def info(self) -> dict:
        v = [ctypes.c_int() for _ in range(4)]
        check(self.ctx.lib.qf_program_info(self.handle, *[ctypes.byref(x) for x in v]))
        return {"fwd_sweeps": v[0].value, "bwd_sweeps": v[1].value, "fwd_tile_bits": v[2].value,
                "bwd_tile_bits": v[3].value}

    def jit_status(self) -> dict:
        """Specialised-kernel status (NVRTC): active, kernels compiled / loaded from cache, seconds."""
        a, c, k = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        sec = ctypes.c_double()
        err = ctypes.c_char_p()
        check(self.ctx.lib.qf_program_jit_status(self.handle, ctypes.byref(a), ctypes.byref(c), ctypes.byref(k),
                                                 ctypes.byref(sec), ctypes.byref(err)))
        return {"active": bool(a.value), "compiled": c.value, "cached": k.value, "seconds": sec.value,
                "error": (err.value or b"").decode()}

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.qf_program_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Observable:
    """A Pauli sum on the device (qf_observable). codes [T, n] int8, weights complex [T]."""

    def __init__(self, ctx: Context, n: int, codes: np.ndarray, weights: np.ndarray):
        self.ctx, self.n = ctx, n
        codes = np.ascontiguousarray(np.asarray(codes, dtype=np.int8).reshape(-1, n) if n else codes)
        w = np.asarray(weights, dtype=np.complex128).reshape(-1)
        self.n_terms = int(w.size)
        wr = np.ascontiguousarray(w.real)
        wi = np.ascontiguousarray(w.imag)
        h = ctypes.c_void_p()
        check(ctx.lib.qf_observable_create(ctx.handle, n, self.n_terms,
                                           codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                                           dptr(wr), dptr(wi), ctypes.byref(h)))
        self.handle = h

    def set_sharding(self, mode: int) -> None:
        check(self.ctx.lib.qf_observable_set_sharding(self.handle, int(mode)))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.qf_observable_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def energy_grad_batch(ctx: Context, prog: Program, obs: Observable, thetas: np.ndarray,
                      grads: bool = True):
    """Host-buffer evaluation (qf_energy_grad_batch): returns (E[B], G[B, P] or None)."""
    th = np.asarray(thetas, dtype=np.float64)
    th = np.ascontiguousarray(th.reshape(-1, prog.n_params) if prog.n_params
                              else np.zeros((th.shape[0] if th.ndim == 2 else 1, 0)))
    B = th.shape[0]
    E = np.empty(B, dtype=np.float64)
    G = np.empty((B, prog.n_params), dtype=np.float64) if grads else None
    check(ctx.lib.qf_energy_grad_batch(ctx.handle, prog.handle, obs.handle, B, dptr(th), dptr(E),
                                       dptr(G) if grads else None))
    return E, G


def energy_grad_batch_partial(ctx: Context, prog: Program, obs: Observable, thetas: np.ndarray, rank: int,
                              world: int, grads: bool = True):
    """The contribution rank `rank` of `world` makes before the all-reduce
    (qf_energy_grad_batch_partial): the multi-GPU split replayed on one GPU."""
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(-1, prog.n_params))
    B = th.shape[0]
    E = np.empty(B, dtype=np.float64)
    G = np.empty((B, prog.n_params), dtype=np.float64) if grads else None
    check(ctx.lib.qf_energy_grad_batch_partial(ctx.handle, prog.handle, obs.handle, B, dptr(th), int(rank),
                                               int(world), dptr(E), dptr(G) if grads else None))
    return E, G


def energy_grad_batch_device(ctx: Context, prog: Program, obs: Observable, d_thetas, d_energies,
                             d_grads=None) -> None:
    """Device-buffer evaluation (torch CUDA float64 tensors), ordered on ctx.stream."""
    B = int(d_energies.shape[0])
    check(ctx.lib.qf_energy_grad_batch_device(
        ctx.handle, prog.handle, obs.handle, B, ctypes.c_void_p(d_thetas.data_ptr()),
        ctypes.c_void_p(d_energies.data_ptr()),
        ctypes.c_void_p(d_grads.data_ptr()) if d_grads is not None else None))


def run_state(ctx: Context, prog: Program, theta: np.ndarray, guard_log2: int = 24) -> np.ndarray:
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    out = np.empty(1 << prog.n, dtype=np.complex128)
    check(ctx.lib.qf_run_state(ctx.handle, prog.handle, dptr(th) if th.size else None, int(guard_log2),
                               dptr(out.view(np.float64))))
    return out


def expectation(ctx: Context, prog: Program, obs: Observable, theta: np.ndarray) -> complex:
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    out = np.empty(2, dtype=np.float64)
    check(ctx.lib.qf_expectation(ctx.handle, prog.handle, obs.handle, dptr(th) if th.size else None,
                                 dptr(out)))
    return complex(out[0], out[1])


def pauli_sum_to_coo(ctx: Context, obs: Observable, n_guard: int = 26, device: bool = False):
    """Canonical COO of the observable (qf_pauli_sum_to_coo): numpy arrays
    (rows, cols, vals complex128), or torch CUDA tensors when device=True."""
    nnz = ctypes.c_int64()
    check(ctx.lib.qf_pauli_sum_to_coo(ctx.handle, obs.handle, n_guard, 0, None, None, None, 0, ctypes.byref(nnz)))
    m = nnz.value
    if device:
        import torch
        dev = torch.device("cuda", ctx.device)
        rows = torch.empty(m, dtype=torch.int64, device=dev)
        cols = torch.empty(m, dtype=torch.int64, device=dev)
        vals = torch.empty(m, dtype=torch.complex128, device=dev)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if m else None  # noqa: E731
        check(ctx.lib.qf_pauli_sum_to_coo(ctx.handle, obs.handle, n_guard, 1, ptr(rows), ptr(cols), ptr(vals), m,
                                          ctypes.byref(nnz)))
        return rows, cols, vals
    rows = np.empty(m, dtype=np.int64)
    cols = np.empty(m, dtype=np.int64)
    vals = np.empty(m, dtype=np.complex128)
    if m:
        check(ctx.lib.qf_pauli_sum_to_coo(ctx.handle, obs.handle, n_guard, 0, ctypes.c_void_p(rows.ctypes.data),
                                          ctypes.c_void_p(cols.ctypes.data), ctypes.c_void_p(vals.ctypes.data), m,
                                          ctypes.byref(nnz)))
    return rows, cols, vals


def sparse_energy(ctx: Context, prog: Program, thetas, dim: int, rows, cols, vals) -> np.ndarray:
    """energy(ansatz, theta, SparseCOO) for each parameter row (qf_sparse_energy,
    variational.cpp:45-52).  rows/cols/vals: numpy (int64, int64, complex128), or
    torch CUDA tensors of the same dtypes (used in place, e.g. the output of
    pauli_sum_to_coo(..., device=True))."""
    th = np.asarray(thetas, dtype=np.float64)
    th = np.ascontiguousarray(th.reshape(-1, prog.n_params) if prog.n_params
                              else np.zeros((th.shape[0] if th.ndim == 2 else 1, 0)))
    B = th.shape[0]
    out = np.zeros(B)
    on_dev = hasattr(vals, "is_cuda") and vals.is_cuda
    if on_dev:
        import torch
        assert rows.dtype == torch.int64 and cols.dtype == torch.int64 and vals.dtype == torch.complex128
        nnz = int(vals.numel())
        ptrs = [ctypes.c_void_p(t.data_ptr()) if nnz else None for t in (rows, cols, vals)]
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.complex128)
        nnz = int(vals.size)
        ptrs = [ctypes.c_void_p(a.ctypes.data) if nnz else None for a in (rows, cols, vals)]
    check(ctx.lib.qf_sparse_energy(ctx.handle, prog.handle, B, dptr(th), int(dim), nnz, *ptrs, 1 if on_dev else 0,
                                   dptr(out)))
    return out


def mipt_haar(ctx: Context, n: int, depth: int, p: float, trajectories: int, seed: int, precision="c64"):
    """Half-chain entropies of MIPT-Haar trajectories (qf_mipt_haar, reference
    experiments.cpp:210-250); returns (entropies[trajectories], measurement count)."""
    out = np.zeros(int(trajectories))
    cnt = ctypes.c_longlong()
    check(ctx.lib.qf_mipt_haar(ctx.handle, int(n), int(depth), float(p), int(trajectories), int(seed),
                               PRECISIONS[precision], dptr(out), ctypes.byref(cnt)))
    return out, int(cnt.value)


def apply_unitary(ctx: Context, amps: np.ndarray, u, wires: Sequence[int]) -> np.ndarray:
    """apply_local_unitary on a complex128 state (qf_apply_unitary): returns the new amplitudes."""
    st = np.ascontiguousarray(np.asarray(amps, np.complex128)).copy()
    n = int(st.size).bit_length() - 1
    um = np.ascontiguousarray(np.asarray(u, np.complex128)).view(np.float64)
    w = (ctypes.c_int * max(1, len(wires)))(*[int(x) for x in wires])
    check(ctx.lib.qf_apply_unitary(ctx.handle, n, dptr(st.view(np.float64)), len(wires), w, dptr(um)))
    return st


def hermitian_eigvals(ctx: Context, a) -> np.ndarray:
    """Ascending eigenvalues of a batch of Hermitian matrices [batch, m, m] through the
    device tridiagonalisation + bisection kernels (qf_hermitian_eigvals)."""
    a = np.asarray(a, np.complex128)
    if a.ndim == 2:
        a = a[None]
    B, m = int(a.shape[0]), int(a.shape[1])
    buf = np.ascontiguousarray(np.transpose(a, (0, 2, 1))).view(np.float64)  # column-major per matrix
    w = np.zeros((B, m))
    check(ctx.lib.qf_hermitian_eigvals(ctx.handle, m, B, dptr(buf), dptr(w)))
    return w


def shadow_snapshots(ctx: Context, prep: Program, theta, bases, u) -> np.ndarray:
    """Classical-shadow outcomes (qf_shadow_snapshots, shadows.cpp:50-85):
    bases [m, n] codes 1/2/3, u [m] uniforms -> outcomes [m, n] bits (int8)."""
    th = np.ascontiguousarray(np.asarray(theta if theta is not None else np.zeros(0), dtype=np.float64).reshape(-1))
    bases = np.ascontiguousarray(np.asarray(bases, dtype=np.int8).reshape(-1, prep.n))
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(-1))
    m = bases.shape[0]
    if u.size != m:
        raise ValueError("shadow_snapshots: one uniform per snapshot")
    out = np.zeros((m, prep.n), dtype=np.int8)
    check(ctx.lib.qf_shadow_snapshots(ctx.handle, prep.handle, dptr(th), m, ctypes.c_void_p(bases.ctypes.data), dptr(u),
                                      ctypes.c_void_p(out.ctypes.data)))
    return out


def noise_trajectories(ctx: Context, n: int, ops: Sequence, mats, op_channels, channels, u, precision="c128",
                       init=None, obs: Optional["Observable"] = None, want_states: bool = True):
    """Batched mc_trajectory (qf_noise_trajectories, noise.cpp:162-197).
    op_channels[j]: channel indices firing after op j; channels[c]: list of D x D
    Kraus matrices; u: [T, n_apps] uniforms (one per channel application, in
    order).  Returns (states [T, 2^n] complex or None, log_probs [T], energies [T] or None)."""
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    T = int(u.shape[0])
    ptr = [0]
    flat = []
    for j in range(len(ops)):
        chs = list(op_channels[j]) if j < len(op_channels) else []
        flat += chs
        ptr.append(len(flat))
    kptr = [0]
    kr = []
    for ops_k in channels:
        for k in ops_k:
            k = np.asarray(k, dtype=np.complex128)
            full = np.zeros((4, 4), np.complex128)
            full[: k.shape[0], : k.shape[1]] = k
            kr.append(full)
        kptr.append(len(kr))
    if u.ndim != 2 or u.shape[1] != ptr[-1]:
        raise ValueError("noise_trajectories: u must be [trajectories, channel applications]")
    as_i = lambda v: (ctypes.c_int * max(1, len(v)))(*v)  # noqa: E731
    kr_v = np.ascontiguousarray(np.array(kr if kr else [np.zeros((4, 4))], np.complex128)).view(np.float64).reshape(-1)
    arr = _op_array(ops)
    mv, nm = _mats_array(mats)
    init_v = None
    if init is not None:
        init_v = np.ascontiguousarray(np.asarray(init, np.complex128).reshape(-1)).view(np.float64)
    states = np.zeros((T, 1 << n), np.complex128) if want_states else None
    logp = np.zeros(T)
    ev = np.zeros(T) if obs is not None else None
    check(ctx.lib.qf_noise_trajectories(
        ctx.handle, n, len(ops), arr, dptr(mv), nm, as_i(ptr), as_i(flat), as_i(kptr), dptr(kr_v), dptr(init_v), T,
        dptr(u), PRECISIONS[precision], dptr(states.view(np.float64)) if states is not None else None, dptr(logp),
        obs.handle if obs is not None else None, dptr(ev) if ev is not None else None))
    return states, logp, ev


def adam_step_device(ctx: Context, theta, m, v, g, t: int, lr: float, beta1=0.9, beta2=0.999,
                     eps=1e-8) -> None:
    B, P = (int(theta.shape[0]), int(theta.shape[1])) if theta.dim() == 2 else (1, int(theta.numel()))
    check(ctx.lib.qf_adam_step_device(ctx.handle, B, P, ctypes.c_void_p(theta.data_ptr()),
                                      ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(v.data_ptr()),
                                      ctypes.c_void_p(g.data_ptr()), int(t), float(lr), float(beta1),
                                      float(beta2), float(eps)))
