"""Index (among launches whose kernel name matches a regex, optionally with a given grid size) of
the longest launch in an ncu `--metrics gpu__time_duration.sum[,launch__grid_size] --csv` launch
list — the --launch-skip for a one-launch full capture.

  python tools/pick_launch.py launches.csv REGEX [GRID]"""
import csv
import re
import sys

path, pattern = sys.argv[1], re.compile(sys.argv[2])
want_grid = int(sys.argv[3]) if len(sys.argv) > 3 else None
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
by_id = {}
for r in csv.DictReader(lines):
    if not pattern.search(r.get("Kernel Name", "")):
        continue
    rec = by_id.setdefault(r["ID"], {})
    rec[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
launches = [by_id[k] for k in sorted(by_id, key=int)]
cands = [i for i, rec in enumerate(launches)
         if want_grid is None or int(rec.get("launch__grid_size", -1)) == want_grid]
best = max(cands, key=lambda i: launches[i].get("gpu__time_duration.sum", 0.0))
print(best)
