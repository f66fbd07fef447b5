#!/usr/bin/env python
"""Development probe: C2 step time when the batch is evaluated in chunks small
enough that a chunk's psi + lambda stay resident in the 126 MB L2 across all of
its sweeps (memory budget -> chunk size).  Prints one JSON line per chunk size:
plain step ms (CUDA events, no per-launch instrumentation) and the per-launch
split of one instrumented step.

  python tools/l2_chunk_probe.py [config] [batch] [chunk,chunk,...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = dict(bench.CONFIGS[cfg_name])
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["batch"]
chunks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1024,16,8,4,2").split(",")]
steps = int(os.environ.get("QF_PROBE_STEPS", "3"))

ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian(cfg_name, cfg)
ctx = engine.default_context(0)
prog = engine.Program(ctx, cfg["n"], ops, P, cfg["prec"])
obs = h.observable(ctx)
dev = torch.device("cuda", 0)
th = torch.tensor(bench.thetas_for(cfg_name, B, P), device=dev)
ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
N = 1 << cfg["n"]
b = 8 if cfg["prec"] == "c64" else 16
ref = None
for bc in chunks:
    E = torch.zeros(B, dtype=torch.float64, device=dev)
    G = torch.zeros((B, P), dtype=torch.float64, device=dev)
    # per-entry bytes: psi + lambda + tap partials + matrices (generous: 5 % over)
    ctx.set_memory_budget(int(bc * (2 * N * b) * 1.05) if bc < B else 0)

    def run(k):
        with torch.cuda.stream(ext):
            for _ in range(k):
                engine.energy_grad_batch_device(ctx, prog, obs, th, E, G)
        torch.cuda.synchronize()

    run(2)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    run(steps)
    e1.record(ext)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.reset_stats()
    ctx.set_timing(2)
    run(1)
    lt = ctx.launch_times()
    ctx.set_timing(0)
    Eh, Gh = E.cpu().numpy(), G.cpu().numpy()
    if ref is None:
        ref = (Eh, Gh)
    out = {"config": cfg_name, "batch": B, "chunk": bc, "ms_per_step": ms, "evals_per_s": B / ms * 1e3,
           "max_abs_dE_vs_first": float(np.abs(Eh - ref[0]).max()),
           "max_abs_dG_vs_first": float(np.abs(Gh - ref[1]).max()),
           "launch_ms_total": {str(k): round(v[0], 3) for k, v in sorted(lt.items())}}
    print(json.dumps(out), flush=True)
