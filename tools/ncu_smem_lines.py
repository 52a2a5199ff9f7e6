"""Per-CUDA-source-line shared-memory wavefronts (total / excessive) of an ncu report (cuda,sass view)."""
import collections
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
kf = sys.argv[4] if len(sys.argv) > 4 else None  # kernel-name regex for multi-kernel reports
out = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + kf] if kf else []) +
                     ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname = hdr = cur = None
for r in csv.reader(out):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        wf, ex = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
        continue
    if hdr is None or len(r) <= ex:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1].strip()[:80]
    try:
        agg[cur][0] += float(r[wf] or 0)
        agg[cur][1] += float(r[ex] or 0)
    except (ValueError, KeyError):
        continue
tw = sum(v[0] for v in agg.values())
print(f"shared wavefronts per unit {tw / units:.1f}, excessive {sum(v[1] for v in agg.values()) / units:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:4d} wf {v[0] / units:7.1f} excess {v[1] / units:7.1f} | {v[2]}")
