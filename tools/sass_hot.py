"""Summarise an ncu source page (SASS view): instruction mix and hottest instructions."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
pick = sys.argv[3] if len(sys.argv) > 3 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
ins = []
take = pick is None
for r in rows:
    if r and r[0] == "Kernel Name":
        take = pick is None or pick in r[1]
        hdr = None
        continue
    if not take:
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            ie = int(d["Instructions Executed"] or 0)
            st = int(d["Warp Stall Sampling (All Samples)"] or 0)
            th = float(d["Avg. Threads Executed"] or 0)
        except ValueError:
            continue
        ins.append((d["Address"], d["Source"].strip(), ie, st, th))
tot = sum(i[2] for i in ins)
tst = sum(i[3] for i in ins)
print("instructions", tot, "stall samples", tst)
mix = Counter()
for a, s, ie, st, th in ins:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    mix[op.split(".")[0]] += ie
print("mix:", ", ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in mix.most_common(25)))
print("--- hottest by stall samples")
for a, s, ie, st, th in sorted(ins, key=lambda x: -x[3])[:n]:
    print(f"{a[-5:]} st{100 * st / max(tst, 1):5.1f}% ie{ie:>9} thr{th:5.1f} {s[:80]}")
