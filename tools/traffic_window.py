"""Steady-state DRAM traffic per launch of each config's step kernel:
python tools/traffic_window.py <tag> <csv>... -> profiles/traffic.json (+ a summary per config).

Each csv is an ncu launch list of >= 10 CONSECUTIVE launches of one step kernel taken with
  ncu --replay-mode application --cache-control none --clock-control none
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:<kernel> -s 5 -c 12
(no cache flush between launches: the dirty L2 lines a launch leaves behind are written back
during the next one, so the per-launch average is the steady-state traffic, not the flushed
single-launch figure).  The csv file name is tw_<config>.csv."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CELLS = {"config2": 4096 * 4096, "config3": 512 ** 3, "config3_fp32": 512 ** 3, "config4": 4096 * 4097,
         "config5": 512 ** 3}
B_ALG = {"config2": 24, "config3": 34, "config3_fp32": 36, "config4": 40, "config5": 72}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
         "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}

tag = sys.argv[1]
out_path = ROOT / "profiles" / "traffic.json"
data = json.loads(out_path.read_text()) if out_path.exists() else {}
data = {k: v for k, v in data.items() if isinstance(v, dict)}
lines = []
for f in sys.argv[2:]:
    key = Path(f).stem.replace("tw_", "")
    hdr, per = None, defaultdict(dict)
    for r in csv.reader(open(f)):
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", ""), 1.0)
            per[int(d["ID"])][d["Metric Name"]] = v
            per[int(d["ID"])]["kernel"] = d["Kernel Name"].split("(")[0]
    ids = sorted(per)
    if len(ids) < 10:
        raise SystemExit(f"{f}: {len(ids)} launches, need >= 10 consecutive")
    byt = [per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"] for i in ids]
    t = [per[i]["gpu__time_duration.sum"] for i in ids]
    mean_b, mean_t = sum(byt) / len(byt), sum(t) / len(t)
    data[key] = {"kernel": per[ids[0]]["kernel"], "dram_bytes_per_launch": mean_b, "launches": len(ids),
                 "bytes_per_cell_step": mean_b / CELLS[key], "algorithmic_bytes_per_cell_step": B_ALG[key],
                 "mean_launch_s": mean_t,
                 "source": f"profiles/{tag}_traffic_window.txt (ncu --replay-mode application --cache-control none, "
                           f"{len(ids)} consecutive launches, dram__bytes_read.sum + dram__bytes_write.sum)"}
    lines.append(f"{key}: {data[key]['kernel']} x{len(ids)}: {mean_b / 1e9:.4f} GB/launch = "
                 f"{mean_b / CELLS[key]:.2f} B/cell-step (algorithmic {B_ALG[key]}), {mean_t * 1e6:.1f} us/launch "
                 f"under ncu, min/max bytes {min(byt) / 1e9:.4f}/{max(byt) / 1e9:.4f} GB")
out_path.write_text(json.dumps(data, indent=1) + "\n")
(ROOT / "profiles" / f"{tag}_traffic_window.txt").write_text(
    "# steady-state DRAM traffic windows: ncu --replay-mode application --cache-control none --clock-control none\n"
    "# (per-launch dram__bytes_read.sum + dram__bytes_write.sum averaged over consecutive launches)\n" + "\n".join(lines) + "\n")
print("\n".join(lines))
