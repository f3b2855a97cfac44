"""One-line-per-kernel summary of an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
want = {"Duration": "dur", "Executed Ipc Active": "ipc", "Issued Instructions": "inst", "Achieved Occupancy": "occ",
        "Theoretical Occupancy": "theo", "Registers Per Thread": "regs", "DRAM Throughput": "dram%",
        "L2 Hit Rate": "l2hit", "Warp Cycles Per Issued Instruction": "cpi", "Avg. Active Threads Per Warp": "thr",
        "Grid Size": "grid", "Block Size": "blk", "Memory Throughput": "mem", "Compute (SM) Throughput": "sm%"}
cur, acc = None, {}
out = []
for r in rows[1:]:
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0][-28:])
    if key != cur:
        if cur:
            out.append((cur, acc))
        cur, acc = key, {}
    n = d["Metric Name"]
    if n in want:
        acc[want[n]] = d["Metric Value"] + ("" if d["Metric Unit"] in ("", "inst", "register/thread", "cycle") else d["Metric Unit"][:6])
if cur:
    out.append((cur, acc))
for (i, k), a in out:
    print(f"{i:>3} {k:28s} " + " ".join(f"{x}={a.get(x, '-')}" for x in ["dur", "inst", "ipc", "cpi", "occ", "theo", "regs", "thr", "grid", "blk", "mem", "dram%", "sm%"]))
