"""Instructions executed and stall samples per CUDA source line (ncu --print-source cuda,sass)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kid:
    cmd += ["--kernel-id", f"::regex:{kid}:1"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
hdr, cur_file = None, ""
ins, st, src = defaultdict(int), defaultdict(int), {}
line = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        line = (cur_file, r[0])
        src[line] = r[1]
    try:
        ie = int(r[7] or 0)
        s = int(r[4] or 0)
    except ValueError:
        continue
    if line:
        ins[line] += ie
        st[line] += s
tot, tst = sum(ins.values()), sum(st.values())
print(f"instructions {tot}  stall samples {tst}")
for k in sorted(ins, key=lambda k: -ins[k])[:n]:
    print(f"{100*ins[k]/max(tot,1):5.1f}% inst {100*st[k]/max(tst,1):5.1f}% stall  {k[0]}:{k[1]:>5s}  {src[k].strip()[:80]}")
