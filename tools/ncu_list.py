"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import io
import sys
from collections import OrderedDict

text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
agg = OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "")[:60]
    key = (name, r["Grid Size"], r["Block Size"])
    t = float(r["Metric Value"])
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += t
total = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'grid':>14s} {'n':>4s} {'us/launch':>10s} {'share':>6s}")
for (name, grid, blk), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:60s} {grid:>14s} {n:4d} {t / n / 1e3:10.2f} {t / total:6.1%}")
print(f"total {total / 1e3:.1f} us over {len(rows)} launches")
