"""Print the hot loop of an ncu report (SASS rows executed >= threshold) with their stall samples."""
import csv
import subprocess
import sys

rep, thr = sys.argv[1], float(sys.argv[2])
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep] + kf + ["--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# first kernel section only (a report can list the same launch more than once)
_ks = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(_ks) > 1:
    rows = rows[:_ks[1]]
h = rows[1]
ie, src, ss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
cols = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_barrier", "stall_math", "stall_not_selected",
        "stall_selected", "stall_mio", "stall_lg", "stall_branch_resolving", "stall_dispatch", "stall_no_inst"]
idx = [h.index(c) for c in cols]
tot = {c: 0.0 for c in cols}
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n = float(r[ie] or 0)
    except ValueError:
        continue
    for c, i in zip(cols, idx):
        tot[c] += float(r[i] or 0)
    if n >= thr:
        print(f"{r[src].strip()[:64]:64s} S={r[ss]:>5s} " +
              " ".join(f"{c[6:11]}={r[i]}" for c, i in zip(cols, idx) if r[i] not in ("0", "")))
print("TOTAL", sorted(((round(v), k) for k, v in tot.items()), reverse=True))
