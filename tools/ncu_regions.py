"""Split an ncu source-page CSV (tools/gpu_prof.sh) of the decode kernel into prologue / tile loop / epilogue and
print per-chunk executed instructions and stall samples of the loop (instructions per 32-token tile).
    python tools/ncu_regions.py gpurun_out/X.source.csv.gz N_TILES [chunk]"""
import collections
import csv
import gzip
import re
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])))
ntile = float(sys.argv[2])
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hdr = rows[1]
ai, ei, si = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if len(r) <= ei or r[0] == "Kernel Name":
        break
    try:
        recs.append((int(r[0], 16), r[ai].strip(), int(r[ei]), int(r[si])))
    except ValueError:
        pass
# the tile loop: the TRYWAIT executed most often, and the backward branch after it to the smallest target
w = max((i for i, x in enumerate(recs) if "TRYWAIT" in x[1]), key=lambda i: recs[i][2])
addr = {x[0]: i for i, x in enumerate(recs)}
head, be = None, None
for i in range(w, len(recs)):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", recs[i][1])
    if m:
        t = int(m.group(1), 16)
        if t in addr and addr[t] < w and recs[i][2] >= recs[w][2] * 0.9:
            head, be = addr[t], i
            break
tot_i = sum(x[2] for x in recs); tot_s = sum(x[3] for x in recs)
for name, (a, b) in {"pre": (0, head), "loop": (head, be + 1), "post": (be + 1, len(recs))}.items():
    i = sum(x[2] for x in recs[a:b]); s = sum(x[3] for x in recs[a:b])
    print(f"{name:5s} instr {i / tot_i * 100:5.1f}%  samples {s / tot_s * 100:5.1f}%  per-tile instr {i / ntile:.1f}")
for a in range(head, be + 1, chunk):
    b = min(a + chunk, be + 1)
    i = sum(x[2] for x in recs[a:b]); s = sum(x[3] for x in recs[a:b])
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0] for x in recs[a:b])
    print(f"{a:5d} instr/tile {i / ntile:6.1f} samples {s:5d}  ", " ".join(f"{k}:{v}" for k, v in ops.most_common(6)))
