"""Per-source-line executed instructions (per tile) of the FIRST kernel in an ncu sass,cuda source CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntile = float(sys.argv[2])
agg = {}
fname = None
first_func = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if first_func is None:
            first_func = r[1]
        skip = r[1] != first_func
        continue
    if r[0] == "Line No" or skip:
        continue
    if r[0] != "":
        try:
            n, st = int(r[7]), int(r[4])
        except (ValueError, IndexError):
            continue
        key = (fname, int(r[0]), r[1].strip()[:100])
        a = agg.setdefault(key, [0, 0])
        a[0] += n
        a[1] += st
tot = sum(v[0] for v in agg.values())
print(f"total per tile {tot / ntile:.1f}  (inlined lines counted once per file)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[: int(sys.argv[3]) if len(sys.argv) > 3 else 60]:
    print(f"{v[0] / ntile:7.1f} {v[1]:6d} {k[0][:18]:18s}:{k[1]:4d} {k[2]}")
