"""Per-SASS-line hot spots of an ncu source export (profiling aid):
    ncu -i REP --page source --csv --print-source sass -k regex:K > f.csv
    python tools/ncu_sass_hot.py f.csv [N]
Prints instruction totals and, per straight-line region (split at branches
and branch targets), its share of executed warp instructions and of stall
samples, top N regions first."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
data = [dict(zip(h, r)) for r in rows[2:end] if len(r) >= len(h) - 1]  # first kernel section
ix = [(int(d["Address"], 16), d["Source"].strip(), int(d["Instructions Executed"] or 0),
       int(d["Warp Stall Sampling (All Samples)"] or 0)) for d in data]
base = ix[0][0]
tot_i = sum(x[2] for x in ix)
tot_s = sum(x[3] for x in ix)
regions, cur = [], []
for i, x in enumerate(ix):
    if cur and (x[2] != cur[-1][2] or re.search(r"\bBRA\b|EXIT|BSYNC|WARPSYNC", ix[i - 1][1])):
        regions.append(cur)
        cur = []
    cur.append(x)
if cur:
    regions.append(cur)
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
rs = sorted(regions, key=lambda r: -sum(x[2] for x in r))
for r in rs[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    ni = sum(x[2] for x in r)
    ns = sum(x[3] for x in r)
    print(f"[{r[0][0] - base:#07x}-{r[-1][0] - base:#07x}] {len(r):4d} instrs x {r[0][2]:>10,} = {100 * ni / tot_i:5.1f}% inst, "
          f"{100 * ns / max(tot_s, 1):5.1f}% stalls | {r[0][1][:46]} .. {r[-1][1][:34]}")
