"""Top stall sites of an ncu report's SASS source page (with -lineinfo builds):
  python tools/ncu_src_top.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[iss]) for r in data if r[iss].isdigit())
print(rows[0][1][:120], "samples", tot)
for i in sorted(range(len(data)), key=lambda i: -int(data[i][iss]))[:N]:
    r = data[i]
    print(f"{i:5d} {int(r[iss]):8d} {100 * int(r[iss]) / tot:5.1f}% {r[iex]:>10} {r[isrc][:90]}")
