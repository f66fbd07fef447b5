"""development: do two concurrent engine contexts (own streams / buffers) overlap
on one B200?  C2 at batch B as one context vs two contexts x B/2 on two threads."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_14167_b200 import engine  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = bench.CONFIGS["C2"]
ops, P = bench.hea_template(cfg["n"], cfg["layers"])
h = bench.hamiltonian("C2", cfg)
th = bench.thetas_for("C2", B, P)
ctxs = [engine.Context(0), engine.Context(0)]
progs = [engine.Program(c, cfg["n"], ops, P, "c64") for c in ctxs]
obss = [h.observable(c) for c in ctxs]
for c, p, o in zip(ctxs, progs, obss):
    engine.energy_grad_batch(c, p, o, th[: B // 2])  # warm-up / buffers
engine.energy_grad_batch(ctxs[0], progs[0], obss[0], th)

def one(i, rows):
    engine.energy_grad_batch(ctxs[i], progs[i], obss[i], rows)

for rep in range(3):
    t0 = time.perf_counter()
    one(0, th)
    t_single = time.perf_counter() - t0
    t0 = time.perf_counter()
    ts = [threading.Thread(target=one, args=(i, th[i * B // 2:(i + 1) * B // 2])) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    t_pair = time.perf_counter() - t0
    print(f"B={B} one context {t_single*1000:.1f} ms ({B/t_single:.0f} evals/s); two contexts {t_pair*1000:.1f} ms "
          f"({B/t_pair:.0f} evals/s)", flush=True)
