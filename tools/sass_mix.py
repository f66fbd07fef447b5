#!/usr/bin/env python
"""Opcode histogram (executed warp instructions, stall samples) from an
`ncu --page source --csv --print-source sass` export.  Development tool.
  python tools/sass_mix.py export.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix, ie, iss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
cnt, smp = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    op = r[ix].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0] if not o.startswith(("FFMA2", "FMUL2", "FADD2")) else o.split(".")[0]
    cnt[o] += int(r[ie] or 0)
    smp[o] += int(r[iss] or 0)
tot, stot = sum(cnt.values()), sum(smp.values())
print(f"total warp instructions {tot:.4e}, stall samples {stot}")
for o, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{o:10s} {c:14d} {100 * c / tot:6.2f}%   samples {100 * smp[o] / max(stot, 1):6.2f}%")
