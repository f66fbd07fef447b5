"""The C++ drop-in layer (include/qforge/*.hpp over the C-ABI): it builds and
links on the CPU host; on the GPU it runs the reference's hot-path test cases
ported to C++ (cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "cpp", "test_dropin")


def test_dropin_links():
    assert os.path.exists(BIN), "build() compiles cpp/test_dropin"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libqforge.so =>" in out and "libqforge_b200.so =>" in out
    assert "not found" not in out


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(ctx):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
