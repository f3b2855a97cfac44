"""Last N rows of an ncu --csv launch list: kernel, grid, duration (us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][:40], d["Grid Size"], float(d["Metric Value"]) / 1e3))
for k, g, t in out[-n:]:
    print(f"{k:42s} {g:>16s} {t:9.2f} us")
