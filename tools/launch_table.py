"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum etc.)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    per[(r[0], r[ki])][r[mi]] = r[vi]
agg = collections.OrderedDict()
for (i, k), m in per.items():
    name = k.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = name[5:] if name.startswith("void ") else name
    name = name.split("(")[0]
    a = agg.setdefault(name, {"n": 0, "ns": 0.0, "extra": m})
    a["n"] += 1
    a["ns"] += float(m.get("gpu__time_duration.sum", "0").replace(",", ""))
for k, a in agg.items():
    ex = {kk.split("__")[-1][:30]: v for kk, v in a["extra"].items() if kk != "gpu__time_duration.sum"}
    print(f"{k[:70]:70s} n={a['n']:4d} total={a['ns']/1e3:9.1f} us avg={a['ns']/a['n']/1e3:8.1f} us {ex}")
