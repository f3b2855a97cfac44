"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel count and total,
for the launches after the first `skip` fraction (default: the second half, i.e. the repeat)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
h, out = None, []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        out.append((d["Kernel Name"][:70], float(d["Metric Value"].replace(",", ""))))
tail = out[int(len(out) * frac):]
agg = defaultdict(lambda: [0, 0.0])
for k, v in tail:
    agg[k][0] += 1
    agg[k][1] += v
print("launches", len(tail), "total us", sum(v for _, v in tail) / 1000)
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{n:5d} {v / 1000:9.1f} us  {k}")
