"""The C-ABI library (libqforge_b200.so) loads on a CPU-only host, exports every
entry point include/qforge_b200.h declares, and its specialised-kernel generator
compiles for sm_100a through NVRTC (no GPU needed).  No compute calls here."""
import ctypes
import os
import re

import pytest

from oracle import pyoracle as po
from paper_2602_14167_b200 import _lib, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "qforge_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_abi_version_and_error_string():
    lib = _lib.load()
    assert lib.qf_abi_version() == 1
    assert isinstance(lib.qf_last_error(), bytes)


def test_library_links_only_expected_runtime_deps():
    """cudart is static (independent of torch's libcudart); NVRTC/NCCL are dlopen'ed."""
    out = os.popen(f"ldd {_lib.LIB_PATH}").read()
    assert "libcudart" not in out
    assert "libnccl" not in out and "libnvrtc" not in out


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_specialised_kernels_compile_for_sm100a(prec):
    n, ops, P = po.hea_template(6, 2)
    assert engine.jit_compile_check(n, ops, P, prec) == 2  # one forward + one adjoint sweep
    n, ops, P = po.tca_template(5, 1)
    assert engine.jit_compile_check(n, ops, P, prec) == 2


def test_specialised_kernels_compile_all_gate_kinds(monkeypatch):
    """Every device op kind (G1, R1, RX, X1, CX reg/thread control, D1, D2, G2 and all
    taps) in a multi-sweep schedule."""
    import numpy as np
    monkeypatch.setenv("QF_GEOM_C64", "6,3,5,2")
    G = po.GID
    u = np.linalg.qr(np.random.default_rng(0).normal(size=(4, 4)) + 1j * np.random.default_rng(1).normal(size=(4, 4)))[0]
    ops = [(G["h"], 0, -1, -1, 1, 0, -1), (G["x"], 7, -1, -1, 1, 0, -1), (G["y"], 3, -1, -1, 1, 0, -1),
           (G["rx"], 1, -1, 0, 1, 0, -1), (G["ry"], 6, -1, 1, 1, 0, -1), (G["rz"], 5, -1, 2, 1, 0, -1),
           (G["rzz"], 2, 6, 3, 1, 0, -1), (G["cx"], 0, 7, -1, 1, 0, -1), (G["cx"], 6, 5, -1, 1, 0, -1),
           (G["cz"], 1, 4, -1, 1, 0, -1), (G["s"], 2, -1, -1, 1, 0, -1), (G["z"], 3, -1, -1, 1, 0, -1),
           (G["unitary"], 3, 4, -1, 1, 0, 0), (G["rzz"], 0, 7, 4, 1, 0, -1)]
    k = engine.jit_compile_check(8, ops, 5, "c64", mats=[u])
    assert k >= 2


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_specialised_hpsi_compiles_for_sm100a(prec):
    """qf_jit_hpsi_check: the observable-specialised H|psi> kernel (jit.cpp) for
    TFIM / XXZ / complex random sums; sums above the limit use the generic kernel."""
    from oracle import pyoracle as po
    for h in [po.tfim(12, 0.7), po.heisenberg(9, 1.0, 0.5, 0.25), po.random_sum(7, 30, po.Rng(3), False),
              po.random_sum(3, 5, po.Rng(4), True)]:
        assert engine.jit_hpsi_check(h.n, h.codes, h.wr + 1j * h.wi, prec)
    big = po.random_sum(10, 300, po.Rng(5), True)
    assert not engine.jit_hpsi_check(big.n, big.codes, big.wr + 1j * big.wi, prec)
