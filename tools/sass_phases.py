#!/usr/bin/env python
"""Per-segment (between BAR.SYNC) instruction and stall-sample breakdown from an
`ncu --page source --csv --print-source sass` export.  Development tool."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
col = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
seg, segs = Counter(), []
cur = {"inst": 0, "samples": Counter(), "ops": Counter(), "first": None}
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[col["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    ie = int(r[col["Instructions Executed"]] or 0)
    cur["inst"] += ie
    cur["ops"][op.split(".")[0]] += ie
    for k in reasons:
        cur["samples"][k] += int(r[col[k]] or 0)
    if op.startswith("BAR"):
        segs.append(cur)
        cur = {"inst": 0, "samples": Counter(), "ops": Counter(), "first": None}
segs.append(cur)
tot = sum(sum(s["samples"].values()) for s in segs)
for i, s in enumerate(segs):
    ss = sum(s["samples"].values())
    if not s["inst"]:
        continue
    top = ", ".join(f"{k[6:]} {100*v/max(ss,1):.0f}%" for k, v in s["samples"].most_common(4))
    fma = sum(v for k, v in s["ops"].items() if k in ("FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD"))
    print(f"seg {i:2d}: inst {s['inst']:11d} fma {100*fma/s['inst']:4.0f}%  samples {100*ss/tot:5.1f}%  "
          f"samples/inst {ss/s['inst']*1e3:6.2f}e-3  {top}")
