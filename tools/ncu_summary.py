"""One-screen summary of an ncu --set full report: python tools/ncu_summary.py <rep.ncu-rep> [title].
Per kernel: duration, DRAM bytes (and per cell-step if CELLS=<n> is given as argv[3]), IPC, issue
activity, registers, the top warp-stall reasons and the executed-instruction mix (SASS page)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
cells = float(sys.argv[3]) if len(sys.argv) > 3 else None


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u = raw[0], raw[1]
print(f"# {title}")
for row in raw[2:]:
    d = dict(zip(h, row))
    g = lambda k: float(d[k].replace(",", "")) if d.get(k, "") not in ("", "n/a") else float("nan")
    print(d["Kernel Name"][:90])
    t = g("gpu__time_duration.sum")
    tu = u[h.index("gpu__time_duration.sum")]
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    bu = u[h.index("dram__bytes_read.sum")]
    print(f"    duration {t:.3f} {tu}; dram read {rd:.4f} + write {wr:.4f} {bu}")
    if cells:
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
        print(f"    dram bytes per cell-step {(rd + wr) * sc / cells:.2f}")
    for k in ("sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"):
        if k in d:
            print(f"    {k} {d[k]}")
    st = {}
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(d[k].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    print("    stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(src) > 2:
    hh = src[1]
    iE = hh.index("Instructions Executed")
    op = collections.Counter()
    for r in src[2:]:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        try:
            op[m.group(2) if m else "?"] += float(r[iE] or 0)
        except ValueError:
            pass
    tot = sum(op.values()) or 1.0
    print("    instruction mix (first kernel): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in op.most_common(14)))
