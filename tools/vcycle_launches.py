"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
tools/vcycle_once.py by level: kernel count and summed duration per grid size
class, to see where a V-cycle's time goes at the coarse levels."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Value")}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
data = []
for r in rows[hdr + 1:]:
    if len(r) < len(h) or not r[ix["Metric Value"]].replace(".", "").replace(",", "").isdigit():
        continue
    data.append((int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0], r[ix["Grid Size"]],
                 float(r[ix["Metric Value"]].replace(",", "")) / 1000.0))
data = data[skip:]
tot = sum(d[3] for d in data)
print(f"{len(data)} launches, {tot:.1f} us of kernel time")
by = defaultdict(lambda: [0, 0.0])
for _, name, grid, us in data:
    by[(name, grid)][0] += 1
    by[(name, grid)][1] += us
for (name, grid), (n, us) in sorted(by.items(), key=lambda kv: -kv[1][1])[:60]:
    print(f"{us:10.1f} us {n:5d} x {us / n:8.1f}  {name[:60]:60s} {grid}")
