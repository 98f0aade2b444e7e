"""Per-source-line SASS instruction counts of the first kernel in an ncu source export:
    ncu -i rep --page source --csv --print-source sass,cuda > src.csv
    python tools/src_lines.py src.csv N_TILES [top]
SASS rows are attributed to the preceding CUDA source row of the kernel's main file (inlined helpers count
at their own line); counts are per tile (warp-instructions executed / N_TILES)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntile = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
main = None
fname = None
first = None
skip = False
cur = None
per = collections.Counter()
ops = collections.defaultdict(collections.Counter)
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        main = main or fname if fname.startswith("kvt_decode_mma") else main
        continue
    if r[0] == "Function Name":
        first = first or r[1]
        skip = r[1] != first
        continue
    if r[0] == "Line No" or skip:
        continue
    try:
        n = int(r[7])
    except (ValueError, IndexError):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:80]
    elif fname == main:
        per[cur] += n
        op = r[3].split()
        op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
        ops[cur][op] += n
tot = sum(per.values())
# the main-file section lists every SASS instruction of the kernel once per file section it is inlined in;
# normalise by the HMMA count (2 per k-step: 32 per tile) to report per-tile numbers
hm = sum(c["HMMA.16816.F32"] for c in ops.values())
scale = hm / 32.0 if hm else ntile
print(f"normalisation: HMMA/32 = {scale:.0f} (tiles given {ntile:.0f});  total per tile {tot / scale:.1f}")
for k, v in sorted(per.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / scale:6.1f}  L{k[1]:4d} {text.get(k, '')[:70]:70s} " + " ".join(f"{o}:{n / scale:.0f}" for o, n in ops[k].most_common(4)))
