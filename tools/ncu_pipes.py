"""Pipe utilisation, thread efficiency and stall reasons (per issued instruction) of every
kernel in an ncu report: python tools/ncu_pipes.py report.ncu-rep"""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
PIPES = ["fma", "alu", "fp64", "xu", "lsu", "adu", "cbu", "uniform"]
for r in rows[2:]:
    d = dict(zip(h, r))
    f = lambda k: float(d[k].replace(",", "")) if d.get(k, "") not in ("", "n/a") else float("nan")  # noqa: E731
    print(d["Kernel Name"].split("(")[0])
    print("  threads/warp-inst %.2f  issue active %.1f%%  warps active %.1f%%  regs %s" % (
        f("smsp__thread_inst_executed_per_inst_executed.ratio"),
        f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        f("sm__warps_active.avg.pct_of_peak_sustained_active"), d.get("launch__registers_per_thread")))
    print("  pipes (% of peak, active cycles): " + "  ".join(
        "%s %.1f" % (p, f(f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active")) for p in PIPES))
    st = sorted(((f(k), k.split("stalled_")[1].split("_per_issue")[0]) for k in h
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                reverse=True)
    print("  stalls (warps per issued instruction): " + "  ".join("%s %.2f" % (n, v) for v, n in st if v >= 0.05))
