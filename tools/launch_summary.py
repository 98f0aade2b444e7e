"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count, mean, share."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki].split("(")[0][:70], r[gi])].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for (k, g), v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):5d} x {sum(v) / len(v) / 1000:9.2f} us  share {sum(v) / tot * 100:5.1f}%  grid {g:14s} {k}")
print(f"total {tot / 1e6:.3f} ms over {sum(len(v) for v in agg.values())} launches")
