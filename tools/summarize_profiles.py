"""Turn tools/gpu_checkpoint.sh outputs into the committed profiles/ summaries:
python tools/summarize_profiles.py <tag>   (e.g. r1)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
CELLS = 4096 * 4096

# launch list
rows, hdr = [], None
for r in csv.reader(open(OUT / "ck_launches_raw.csv")):
    if "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
by = defaultdict(dict)
for d in rows:
    by[int(d["ID"])]["kernel"] = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    if d["Metric Name"] == "gpu__time_duration.sum":
        by[int(d["ID"])]["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    else:
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(unit, 1e-6)
        by[int(d["ID"])][d["Metric Name"]] = v * scale
lines = [f"# {tag} launch list: python tools/profile_step.py 20 (config 2, 4096^2, fp16 op3), ncu --clock-control none",
         "# cold-cache, serialised replays: compare SHARES, not absolutes",
         "# per run: one-time setup (plane rounding, k_cheap_div_table, ghosts, E(0) energy + epilogue), then one",
         "# k_ac2d_fused launch per leapfrog step -- the bench's timed region is the k_ac2d_fused launches only",
         "id,kernel,duration_us,dram_read_MB,dram_write_MB"]
tot = defaultdict(lambda: [0, 0.0])
for i in sorted(by):
    d = by[i]
    lines.append(f"{i},{d['kernel']},{d.get('us', 0):.2f},{d.get('dram__bytes_read.sum', 0):.1f},"
                 f"{d.get('dram__bytes_write.sum', 0):.1f}")
    tot[d["kernel"]][0] += 1
    tot[d["kernel"]][1] += d.get("us", 0)
all_us = sum(v[1] for v in tot.values())
for k, (cnt, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"# {k}: {cnt} launches, {us:.1f} us, {100 * us / all_us:.1f}%")
(PROF / f"{tag}_launches.csv").write_text("\n".join(lines) + "\n")

# --set full capture of the step kernel
raw = subprocess.run(["ncu", "-i", str(OUT / "ck_fused_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, d = r[0], dict(zip(r[0], r[1])), dict(zip(r[0], r[2]))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def num(k):
    v = float(d[k].replace(",", ""))
    u = units.get(k, "")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


txt = [f"# {tag} ncu --set full --clock-control none: {d['Kernel Name'].split('(')[0]} (config 2, 4096^2, fp16 op3), "
       "launch 6 of tools/profile_step.py 20"]
for k in keys:
    if k in d:
        txt.append(f"{k:65s} {d[k]} {units.get(k, '')}")
st = {}
for k, v in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and "not_issued" not in k:
        st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v.replace(",", ""))
s = sum(st.values())
txt.append("stall samples (% of all): " + ", ".join(f"{k} {100 * v / s:.1f}" for k, v in
                                                  sorted(st.items(), key=lambda kv: -kv[1])[:8]))
traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
txt.append(f"dram bytes per launch {traffic:.4g} = {traffic / CELLS:.2f} B per cell-step (algorithmic 24)")
(PROF / f"{tag}_fused_ncu_summary.txt").write_text("\n".join(txt) + "\n")
(PROF / "traffic.json").write_text(json.dumps({
    "kernel": d["Kernel Name"].split("(")[0],
    "dram_bytes_per_launch": traffic,
    "source": f"profiles/{tag}_fused_ncu_summary.txt (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"},
    indent=1) + "\n")
for f in ("ck_bench.jsonl", "ck_bench_ref.jsonl"):
    if (OUT / f).exists():
        (PROF / f"{tag}_{'bench_full' if f == 'ck_bench.jsonl' else 'bench_reference'}.jsonl").write_text(
            (OUT / f).read_text())
print("\n".join(txt))
