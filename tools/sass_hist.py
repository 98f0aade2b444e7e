"""Per-opcode executed-instruction histogram (per tile) of the first kernel in an ncu source-page CSV."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntile = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
ai, ei, si = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
op, st = collections.Counter(), collections.Counter()
tot = totst = 0
hot = []
for r in rows[2:]:
    if len(r) <= ei or r[0] == "Kernel Name":
        break
    try:
        n, s = int(r[ei]), int(r[si])
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[ai])
    name = m.group(2) if m else "?"
    op[name] += n; st[name] += s; tot += n; totst += s
    hot.append((n, s, r[ai].strip()))
for k, v in op.most_common(30):
    print(f"{k:10s} {v / tot * 100:5.1f}%  per-tile {v / ntile:7.1f}  stall {st[k] / max(totst, 1) * 100:5.1f}%")
print("total per tile", tot / ntile)
if "-v" in sys.argv:
    for n, s, src in sorted(hot, key=lambda x: -x[1])[:40]:
        print(f"{n / ntile:7.1f} {s:6d}  {src}")
