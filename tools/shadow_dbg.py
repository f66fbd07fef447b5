import sys, time
sys.path.insert(0, '.')
from oracle import pyoracle as po
from paper_2602_14167_b200 import engine
ctx = engine.default_context(0)
for prec in ["c64", "c128", "c64"]:
    ops, bases, us = po.shadow_gen_inputs(20, 256, 4, 2024)
    prep = engine.Program(ctx, 20, ops, 0, prec)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); engine.shadow_snapshots(ctx, prep, None, bases, us); ts.append(time.perf_counter() - t0)
    print(prec, [round(t * 1000, 1) for t in ts], prep.info() if hasattr(prep, "info") else "")
