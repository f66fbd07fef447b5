#!/usr/bin/env python
"""Build the C2 program (NVRTC sweep kernels) in one process; run several of
these at once against an empty QF_JIT_CACHE to check the cross-process compile
claim: the kernels are compiled once in total, the other processes load them
from the cache.  Prints one JSON line with this process's jit_status."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
ctx = engine.default_context(0)
t0 = time.time()
prog = engine.Program(ctx, cfg["n"], ops, P, cfg["prec"])
st = prog.jit_status()
print(json.dumps(dict(pid=os.getpid(), wall_s=round(time.time() - t0, 2), **st)))
