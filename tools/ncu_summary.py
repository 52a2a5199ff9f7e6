"""Summarise an ncu report: per-opcode instruction counts and stall shares per unit of work."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
kf = sys.argv[4] if len(sys.argv) > 4 else None  # kernel-name regex for multi-kernel reports
kargs = ["-k", "regex:" + kf] if kf else []
out = subprocess.run(["ncu", "-i", rep] + kargs + ["--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# first kernel section only (a report can list the same launch more than once)
_ks = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(_ks) > 1:
    rows = rows[:_ks[1]]
h = rows[1]
ie = h.index("Instructions Executed")
ss = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
op, st = collections.Counter(), collections.Counter()
tot = totst = 0.0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n = float(r[ie] or 0)
        s = float(r[ss] or 0)
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[src])
    o = m.group(2).split(".")[0] if m else "?"
    op[o] += n
    st[o] += s
    tot += n
    totst += s
print(f"warp instructions per unit: {tot / units:.1f}")
for o, n in op.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 14):
    print(f"  {o:8s} {n / units:9.1f}  {100 * n / tot:5.1f}%  stall {100 * st[o] / max(totst, 1):5.1f}%")
raw = subprocess.run(["ncu", "-i", rep] + kargs + ["--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rr = list(csv.reader(raw))
keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in rr[0]:
        i = rr[0].index(k)
        print(f"  {k} = {rr[2][i]} {rr[1][i]}")
