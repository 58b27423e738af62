"""Summarise an ncu report: duration, DRAM throughput, issue activity and top stall reasons
per kernel.  python tools/stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ("gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread")
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:60])
    for k in KEYS:
        if k in d:
            print(f"    {k:60s} {d[k]}")
    st = {}
    for k, v in d.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and "not_issued" not in k:
            try:
                st[k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = float(v.replace(",", ""))
            except ValueError:
                pass
    print("    stalls:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:7]))
