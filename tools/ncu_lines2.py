"""Per-CUDA-source-line stall breakdown of an ncu report (top N lines)."""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
src, ss, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ln = h.index("#") if "#" in h else 0
cols = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_math", "stall_selected", "stall_not_selected", "stall_branch_resolving", "stall_mio"]
idx = [h.index(c) for c in cols]
data = []
for r in rows[hi + 1:]:
    if len(r) <= ss:
        continue
    try:
        s = float(r[ss] or 0)
    except ValueError:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
for s, r in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% L{r[ln]:>4s} inst={r[ie]:>9s} " + " ".join(f"{c[6:11]}={r[i]}" for c, i in zip(cols, idx) if r[i] not in ("0", "")) + "  | " + r[src].strip()[:90])
