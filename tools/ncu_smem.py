"""Per-source-line shared-memory wavefronts (total and excessive = bank conflicts)."""
import collections
import csv
import subprocess
import sys

rep, kf = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr, cur = None, None, None
for r in csv.reader(out):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iw, ie = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
        continue
    if hdr is None or len(r) <= iw:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1][:80]
    try:
        agg[cur][0] += float(r[iw] or 0)
        agg[cur][1] += float(r[ie] or 0)
    except (ValueError, TypeError):
        pass
tw = sum(v[0] for v in agg.values())
te = sum(v[1] for v in agg.values())
print(f"shared wavefronts per unit {tw / units:.1f}, excessive {te / units:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    if v[0] == 0:
        continue
    print(f"{k[0]}:{k[1]:4d} wavefronts {v[0] / units:8.1f} excessive {v[1] / units:8.1f}  {v[2]}")
