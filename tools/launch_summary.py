"""Per-kernel mean duration from an ncu launch-list CSV (gpu__time_duration.sum), in launch order."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
d = collections.OrderedDict()
for r in rows[i + 1:]:
    x = dict(zip(h, r))
    if x.get("Metric Name") != "gpu__time_duration.sum":
        continue
    d.setdefault(x["Kernel Name"].split("(")[0][:48], []).append(float(x["Metric Value"]))
tot = 0.0
for n, v in d.items():
    m = sum(v) / len(v) / 1000
    print(f"{n:48s} n={len(v):3d} mean={m:8.1f}us")
