"""C++ drop-in JSON wire formats (Circuit/PauliSum::to_json / from_json,
reference proj/src/circuit.cpp:524-571, proj/src/pauli.cpp:29-50): the ported
reference round-trip tests and malformed-input errors (cpp/test_json.cpp, no
device needed), and byte-identical documents from the C++ headers and the
Python mirror (both follow nlohmann::json::dump(): compact, sorted keys)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "cpp", "test_json")


def _binary():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "cpp"), "test_json"], check=True, capture_output=True)
    return BIN


def test_cpp_json_round_trips():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok")


def test_cpp_and_python_documents_identical():
    sys.path.insert(0, ROOT)
    from paper_2602_14167_b200 import qforge as qf
    out = subprocess.run([_binary(), "dump"], capture_output=True, text=True, timeout=120, check=True).stdout.split("\n")
    c = qf.Circuit(3)
    c.h(0).rx(1, 0.25).ry(2, -1.5e-7).rz(0, 3.0).rzz(0, 2, 1e20).cx(1, 2).cz(0, 1)
    c.su4(0, 1, [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0, 1.1, 1.2, 1.3, 1.4, 1.5])
    s = np.sqrt(0.5)
    c.unitary([2], np.array([[s, 1j * s], [1j * s, s]]))
    h = qf.PauliSum(3)
    h.add(1.0, [1, 0, 3])
    h.add(-0.5 + 0.125j, [2, 2, 0])
    h.add(1e-5 - 3j, [0, 0, 0])
    assert out[0] == c.to_json()
    assert out[1] == h.to_json()
    # and each side reads the other's documents
    c2 = qf.Circuit.from_json(out[0])
    assert [o.name for o in c2.ops] == [o.name for o in c.ops]
    assert qf.PauliSum.from_json(out[1]).to_json() == out[1]
