"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi, ui, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit'), h.index('Grid Size')
    scale = {'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'nsecond': 1e-3, 'ms': 1e3, 'msecond': 1e3}
    tot, cnt, seq = collections.OrderedDict(), collections.Counter(), []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0].replace('unnamed>::', '').replace('void ', '')
        us = float(r[vi].replace(',', '')) * scale[r[ui]]
        tot[name] = tot.get(name, 0.0) + us
        cnt[name] += 1
        seq.append((name, us, r[gi]))
    total = sum(tot.values())
    lines = [f"{len(seq)} launches, {total / 1e3:.3f} ms total (cold-cache, serialised)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{v / 1e3:9.3f} ms {100 * v / total:5.1f}%  {cnt[k]:5d} x {v / cnt[k]:9.1f} us  {k}")
    return "\n".join(lines), seq


if __name__ == "__main__":
    s, _ = summarise(sys.argv[1])
    print(s)
