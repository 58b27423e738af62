"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_summary.py <csv> <out> <title> -> per-launch rows + per-kernel shares."""
import collections
import csv
import sys

rows, hdr = [], None
for r in csv.reader(open(sys.argv[1])):
    if "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
lines = [f"# {sys.argv[3]}", "# cold-cache, serialised ncu replays: compare SHARES, not absolutes", "id,kernel,duration_us"]
tot = collections.defaultdict(lambda: [0, 0.0])
for d in rows:
    us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    k = d["Kernel Name"].split("(")[0]
    lines.append(f"{d['ID']},{k},{us:.2f}")
    tot[k][0] += 1
    tot[k][1] += us
a = sum(v[1] for v in tot.values()) or 1.0
for k, (c, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"# {k}: {c} launches, {us:.1f} us, {100 * us / a:.1f}%")
open(sys.argv[2], "w").write("\n".join(lines) + "\n")
print("\n".join(lines[-12:]))
