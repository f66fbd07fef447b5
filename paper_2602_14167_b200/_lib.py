"""ctypes binding of the C-ABI in include/qforge_b200.h (libqforge_b200.so).

The shared library is built in-tree (``__graft_entry__.build()`` /
``make -C paper_2602_14167_b200/csrc``).  There is no CPU fallback: if the
library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqforge_b200.so")

QF_OK, QF_EINVAL, QF_ERUNTIME, QF_ENOMEM, QF_ECUDA, QF_ENCCL = range(6)
QF_C64, QF_C128 = 0, 1
QF_SHARD_BATCH, QF_SHARD_TERMS = 0, 1

# gate numbering of qforge::Gate (reference include/qforge/circuit.hpp:14-23)
GATES = ["h", "x", "y", "z", "s", "rx", "ry", "rz", "rzz", "cx", "cz", "su4", "csum",
         "subspace_ry", "subspace_rz", "unitary"]
GATE_ID = {g: i for i, g in enumerate(GATES)}


class QfOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("slot", ctypes.c_int32), ("coef", ctypes.c_double), ("offset", ctypes.c_double),
                ("mat", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# name -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "qf_abi_version": (_I, []),
    "qf_last_error": (ctypes.c_char_p, []),
    "qf_ctx_create": (_I, [_I, ctypes.POINTER(_P)]),
    "qf_ctx_destroy": (_I, [_P]),
    "qf_ctx_set_memory_budget": (_I, [_P, ctypes.c_size_t]),
    "qf_nccl_unique_id": (_I, [ctypes.POINTER(ctypes.c_uint8)]),
    "qf_ctx_set_comm": (_I, [_P, _I, _I, ctypes.POINTER(ctypes.c_uint8)]),
    "qf_ctx_stream": (_P, [_P]),
    "qf_program_create": (_I, [_P, _I, _I, ctypes.POINTER(QfOp), _D, _I, _I, _I, ctypes.POINTER(_P)]),
    "qf_program_set_initial_state": (_I, [_P, _D]),
    "qf_program_destroy": (_I, [_P]),
    "qf_program_info": (_I, [_P] + [ctypes.POINTER(_I)] * 4),
    "qf_debug_copy_state": (_I, [_P, _I, _P, ctypes.c_size_t]),
    "qf_program_jit_status": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I), _D,
                                   ctypes.POINTER(ctypes.c_char_p)]),
    "qf_observable_create": (_I, [_P, _I, _I, ctypes.POINTER(ctypes.c_int8), _D, _D, ctypes.POINTER(_P)]),
    "qf_observable_destroy": (_I, [_P]),
    "qf_observable_set_sharding": (_I, [_P, _I]),
    "qf_run_state": (_I, [_P, _P, _D, _I, _D]),
    "qf_expectation": (_I, [_P, _P, _P, _D, _D]),
    "qf_energy_grad_batch": (_I, [_P, _P, _P, _I, _D, _D, _D]),
    "qf_energy_grad_batch_device": (_I, [_P, _P, _P, _I, _P, _P, _P]),
    "qf_energy_grad_batch_partial": (_I, [_P, _P, _P, _I, _D, _I, _I, _D, _D]),
    "qf_vqe_run": (_I, [_P, _P, _P, _I, _D, _I, ctypes.c_double, _I, ctypes.c_double, _D, _D, _D,
                        ctypes.POINTER(_I)]),
    "qf_shard_range": (_I, [ctypes.c_int64, _I, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "qf_adam_step_device": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double]),
    "qf_plan_describe": (_I, [_I, _I, ctypes.POINTER(QfOp), _D, _I, _I, _I, ctypes.c_char_p, ctypes.c_size_t,
                              ctypes.POINTER(ctypes.c_size_t)]),
    "qf_jit_compile_check": (_I, [_I, _I, ctypes.POINTER(QfOp), _D, _I, _I, _I, ctypes.POINTER(_I)]),
    "qf_sparse_energy": (_I, [ctypes.c_void_p, ctypes.c_void_p, _I, _D, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _I, _D]),
    "qf_mipt_haar": (_I, [ctypes.c_void_p, _I, _I, ctypes.c_double, _I, ctypes.c_uint64, _I, _D,
                         ctypes.POINTER(ctypes.c_longlong)]),
    "qf_apply_unitary": (_I, [ctypes.c_void_p, _I, _D, _I, ctypes.POINTER(_I), _D]),
    "qf_hermitian_eigvals": (_I, [ctypes.c_void_p, _I, _I, _D, _D]),
    "qf_shadow_snapshots": (_I, [ctypes.c_void_p, ctypes.c_void_p, _D, _I, ctypes.c_void_p, _D, ctypes.c_void_p]),
    "qf_noise_trajectories": (_I, [ctypes.c_void_p, _I, _I, ctypes.POINTER(QfOp), _D, _I, ctypes.POINTER(_I),
                                  ctypes.POINTER(_I), ctypes.POINTER(_I), _D, _D, _I, _D, _I, _D, _D, ctypes.c_void_p,
                                  _D]),
    "qf_jit_hpsi_check": (_I, [_I, _I, ctypes.c_void_p, _D, _D, _I, ctypes.POINTER(_I)]),
    "qf_pauli_sum_to_coo": (_I, [_P, _P, _I, _I, _P, _P, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "qf_ctx_set_timing": (_I, [_P, _I]),
    "qf_ctx_reset_stats": (_I, [_P]),
    "qf_ctx_flops": (_I, [_P, _D]),
    "qf_ctx_launch_times": (_I, [_P, _I, ctypes.POINTER(_I), _D, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(_I)]),
    "qf_ctx_stats": (_I, [_P, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong), _D, _D]),
}

_lib = None


def load():
    """Load libqforge_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the engine has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a qf_status to the reference's exception convention
    (require() -> std::invalid_argument, common.hpp:24-26 -> ValueError)."""
    if rc == QF_OK:
        return
    msg = load().qf_last_error().decode()
    if rc == QF_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def dptr(a):
    """double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_D)
