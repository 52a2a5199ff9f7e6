"""Per-source-line instruction counts and stall samples from an ncu report (cuda,sass view)."""
import collections
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
kf = sys.argv[5] if len(sys.argv) > 5 else None
out = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + kf] if kf else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
fname = None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
hdr = None
cur_line = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ie:
        continue
    if r[0]:
        cur_line = (fname, int(r[0]))
        agg[cur_line][2] = r[1][:70]
    try:
        n = float(r[ie] or 0)
        s = float(r[ss] or 0)
    except ValueError:
        continue
    if cur_line:
        agg[cur_line][0] += n
        agg[cur_line][1] += s
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "stall" else 0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{k[0]}:{k[1]:4d} inst {v[0] / units:8.1f} ({100 * v[0] / tot:4.1f}%) stall {100 * v[1] / tots:4.1f}%  {v[2]}")
