"""Instruction counts per source line of one kernel: ncu SASS page (executed counts) joined
with nvdisasm -g line info.  python tools/sass_lines.py <ncu_sass.csv> <nvdisasm_fn.txt> [top]
(ncu -i r.ncu-rep --page source --csv --print-source sass > a.csv; nvdisasm -g x.cubin, cut to
the kernel's .text section)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
cnt = {int(r[0], 16) - base: (float(r[iE] or 0), float(r[iS] or 0)) for r in data}
cur, byline = None, collections.defaultdict(lambda: [0.0, 0.0])
for line in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        e, s = cnt.get(int(m.group(1), 16), (0.0, 0.0))
        byline[cur][0] += e
        byline[cur][1] += s
te = sum(v[0] for v in byline.values()) or 1.0
ts = sum(v[1] for v in byline.values()) or 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for (f, l), (e, s) in sorted(byline.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * e / te:5.1f}% inst {100 * s / ts:5.1f}% stall  {f}:{l}")
