"""Group consecutive SASS instructions of one kernel (ncu source page) by execution count: prints
each run of instructions with its count, average active threads and stall share (regions ~ basic blocks)."""
import csv
import subprocess
import sys

rep, pick = sys.argv[1], sys.argv[2]
minfrac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{pick}"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, ins, seen = None, [], set()
for r in rows:
    if r and r[0] == "Kernel Name":
        if ins:
            break  # first matching kernel only
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            ins.append((d["Address"][-5:], d["Source"].strip(), int(d["Instructions Executed"] or 0),
                        int(d["Warp Stall Sampling (All Samples)"] or 0), float(d["Avg. Threads Executed"] or 0)))
        except ValueError:
            pass
tot = sum(i[2] for i in ins)
tst = max(1, sum(i[3] for i in ins))
print(f"{pick}: {tot} warp instructions, {len(ins)} SASS lines")
runs = []
for a, s, ie, st, th in ins:
    if runs and runs[-1][2] == ie:
        runs[-1][1] = a
        runs[-1][3] += 1
        runs[-1][4] += st
        runs[-1][5].append(s.split()[0] if not s.startswith("@") else s.split()[1])
    else:
        runs.append([a, a, ie, 1, st, [s.split()[0] if not s.startswith("@") else s.split()[1]], th])
for a0, a1, ie, n, st, ops, th in runs:
    if ie * n >= minfrac * tot or st >= minfrac * tst:
        print(f"{a0}-{a1} n={n:4d} x{ie:>9} = {100 * ie * n / tot:5.1f}% inst  stall {100 * st / tst:5.1f}%  thr {th:4.1f}  "
              + " ".join(o.split(".")[0] for o in ops[:12]))
