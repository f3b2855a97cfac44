"""Hottest SASS instructions (warp-stall samples) and per-reason totals of one kernel in an ncu report."""
import csv
import subprocess
import sys
from collections import Counter

rep, kid = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-id",
                      f"::regex:{kid}:1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, ins = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        ins.append(dict(zip(hdr, r)))
reasons = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for d in ins:
    for r in reasons:
        try:
            tot[r] += int(d[r] or 0)
        except ValueError:
            pass
S = sum(tot.values())
print("samples", S, {k: v for k, v in tot.most_common(8)})


def si(x):
    try:
        return int(x or 0)
    except ValueError:
        return 0


for d in sorted(ins, key=lambda d: -si(d["Warp Stall Sampling (All Samples)"]))[:n]:
    top = sorted(((si(d[r]), r[6:]) for r in reasons), reverse=True)[:2]
    print(f'{d["Address"][-5:]} {si(d["Warp Stall Sampling (All Samples)"]):6d} exec {si(d["Instructions Executed"]):7d} '
          f'{d["Source"].strip()[:58]:58s} {top}')
