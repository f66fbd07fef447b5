"""Per-launch table from an `ncu --metrics ... --csv` log (run here, no GPU)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
i_id, i_m, i_v, i_u = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
d = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[i_v].replace(",", "")) if r[i_v] not in ("", "n/a") else 0.0
    if r[i_u] == "ns":
        v /= 1e6
    elif r[i_u] == "us":
        v /= 1e3
    elif r[i_u] == "ms":
        pass
    elif r[i_u] == "Kbyte":
        v *= 1e3
    elif r[i_u] == "Mbyte":
        v *= 1e6
    elif r[i_u] == "Gbyte":
        v *= 1e9
    d.setdefault(int(r[i_id]), {})[r[i_m]] = v
S = ["no_instruction", "short_scoreboard", "barrier", "math_pipe_throttle", "long_scoreboard", "mio_throttle", "wait",
     "dispatch_stall", "not_selected"]
print("id     ms   Minst  fma%  iss%  bankM fmaI% lsuI% aluI% | " + " ".join(s[:5] for s in S) + " |  GB")
tot = 0.0
for k, m in d.items():
    ms = m.get("gpu__time_duration.sum", 0)
    tot += ms
    inst = max(m.get("smsp__inst_executed.sum", 1), 1)
    st = [m.get("smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % x, 0) for x in S]
    gb = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{k:2d} {ms:7.3f} {inst / 1e6:7.1f} {m.get('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f} "
          f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f} "
          f"{m.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 0) / 1e6:6.1f} "
          f"{100 * m.get('smsp__inst_executed_pipe_fma.sum', 0) / inst:5.1f} {100 * m.get('smsp__inst_executed_pipe_lsu.sum', 0) / inst:5.1f} "
          f"{100 * m.get('smsp__inst_executed_pipe_alu.sum', 0) / inst:5.1f} | " + " ".join(f"{x:5.2f}" for x in st) + f" | {gb:5.2f}")
print("total ms", round(tot, 3))
