"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum [+ launch__grid_size]); with
--grid, the per-launch durations of kernels matching a substring."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
d = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    e = d[r[ii]]
    e["name"] = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    v = r[vi].replace(",", "")
    if r[mi] == "gpu__time_duration.sum":
        e["us"] = float(v) * {"usecond": 1, "msecond": 1e3, "nsecond": 1e-3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(r[ui], 1e-3)
    else:
        e["grid"] = v
agg = collections.defaultdict(lambda: [0, 0.0])
for e in d.values():
    agg[e["name"]][0] += 1
    agg[e["name"]][1] += e.get("us", 0)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 16]:
    print(f"{k[:60]:60s} {v[0]:5d} {v[1] / 1e3:9.2f} ms {100 * v[1] / tot:5.1f}%")
if "--grid" in sys.argv:
    sub = sys.argv[sys.argv.index("--grid") + 1]
    for k in sorted(d, key=int):
        e = d[k]
        if sub in e["name"]:
            print(k, e["name"][:40], e.get("grid"), round(e.get("us", 0), 1))
