"""Aggregate an ncu SASS source page (csv) by CUDA source line using the
line table of the locally built cubin (nvdisasm -g). Usage:
  python tools/ncu_lines.py <sass_page.csv> <function-sass-dump> [top]"""
import csv
import re
import sys
from collections import defaultdict

page, dump = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None
amap = {}
for l in open(dump):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(page)))
h = rows[1]
ai, ie = h.index("Address"), h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][ai], 16)
agg = defaultdict(lambda: [0, 0])
for r in rows[2:]:
    try:
        a = int(r[ai], 16) - base
    except ValueError:
        continue
    agg[amap.get(a, ("?", 0))][0] += int(r[ws] or 0)
    agg[amap.get(a, ("?", 0))][1] += int(r[ie] or 0)
totw = sum(v[0] for v in agg.values()) or 1
tot = sum(v[1] for v in agg.values()) or 1
srcs = {}
for (f, ln), (w, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if f not in srcs:
        try:
            import glob
            p = glob.glob(f"paper_2511_20432_b200/csrc/**/{f}", recursive=True)
            srcs[f] = open(p[0]).read().splitlines() if p else []
        except Exception:
            srcs[f] = []
    s = srcs[f][ln - 1].strip()[:80] if 0 < ln <= len(srcs[f]) else ""
    print(f"{w / totw * 100:5.1f}% stall {n / tot * 100:5.1f}% inst {f}:{ln:<4d} {s}")
