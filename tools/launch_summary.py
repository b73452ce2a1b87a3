"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel, the launches
and time of the LAST half of the list (the second of tools/one_step.py's two steps)."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")) if r.get("Metric Name") == "gpu__time_duration.sum"]
ids = sorted({int(r["ID"]) for r in rows})
cut = ids[len(ids) // 2] if len(sys.argv) < 3 else int(sys.argv[2])
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if int(r["ID"]) < cut:
        continue
    k = r["Kernel Name"].split("(")[0].split("<")[0].replace("rb::", "").replace("(anonymous namespace)::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    v = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{k:40s} {n:6d} {t/1e3:9.2f} ms {t/n:9.1f} us {100*t/tot:5.1f}%")
