"""Summarise an ncu report (run here, no GPU): per-kernel duration, DRAM bytes,
occupancy, issue activity, top stall reasons, and the instruction mix."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else r[4]
    out = {k: r[hdr.index(k)] for k in keys if k in hdr}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.1:
                stalls[h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = round(v, 2)
    print(name[:60])
    for k, v in out.items():
        print(f"   {k:60s} {v}")
    print("   stalls:", dict(sorted(stalls.items(), key=lambda x: -x[1])))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    cnt = collections.Counter()
    tot = 0
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) > 5 and r[5].isdigit():
            t = r[1].split()
            op = (t[1] if t and t[0].startswith("@") else t[0]).split(".")[0] if t else "?"
            cnt[op] += int(r[5])
            tot += int(r[5])
    print("instruction mix (first kernel):", tot)
    for op, n in cnt.most_common(16):
        print(f"   {op:10s} {n:12d} {100 * n / tot:5.1f}%")
