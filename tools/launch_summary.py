"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
data = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]
agg = collections.defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_ns':>14s} {'avg_ns':>12s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):8d} {sum(v):14.0f} {sum(v) / len(v):12.0f} {sum(v) / tot * 100:6.2f}%")
