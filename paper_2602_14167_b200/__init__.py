"""B200-native batched state-vector VQE engine (energy + adjoint gradient).

Drop-in for the hot path of the reference qforge library (TensorCircuit-NG
restatement, arXiv 2602.14167): include/qforge/{circuit,pauli,variational}.hpp.
Public C-ABI: include/qforge_b200.h (libqforge_b200.so, sm_100a kernels).
Python mirror of the reference API: paper_2602_14167_b200.qforge.
"""
from . import _lib  # noqa: F401
from .rng import RngStream  # noqa: F401

__all__ = ["qforge", "engine", "RngStream", "lib_path"]


def lib_path() -> str:
    return _lib.LIB_PATH
