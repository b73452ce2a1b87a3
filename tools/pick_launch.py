"""Index (among launches whose name matches a regex) of the longest launch in an ncu
`--metrics gpu__time_duration.sum --csv` launch list — the --launch-skip for a full capture."""
import csv
import re
import sys

path, pattern = sys.argv[1], re.compile(sys.argv[2])
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum" and pattern.search(r.get("Kernel Name", "")):
        rows.append(float(r["Metric Value"].replace(",", "")))
best = max(range(len(rows)), key=lambda i: rows[i])
print(best)
