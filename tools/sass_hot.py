"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > iex]
tot = sum(int(r[iss]) for r in body)
print(f"{len(body)} instructions, {tot} samples")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = {r[ia]: i for i, r in enumerate(body)}
for r in sorted(body, key=lambda r: -int(r[iss]))[:top]:
    print(f"{int(r[iss]):7d} {100 * int(r[iss]) / tot:5.1f}%  #{idx[r[ia]]:5d} ex={r[iex]:>10s}  {r[isrc].strip()}")
