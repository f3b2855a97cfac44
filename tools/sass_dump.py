"""Dump the SASS listing of one kernel from an ncu report with per-instruction exec counts.
usage: sass_dump.py REP KERNEL_SUBSTR [min_exec]"""
import csv
import subprocess
import sys

rep, pick = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
take, hdr, seen = False, None, False
for r in csv.reader(txt.splitlines()):
    if r and r[0] == "Kernel Name":
        if seen and take:
            break
        take = pick in r[1]
        seen = seen or take
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
        if ie >= mn:
            print(f"{d['Address'][-5:]} {ie:>9} {st:>5} {th:5.1f} {d['Source'].strip()[:90]}")
