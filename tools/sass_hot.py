"""Top stall-sampled SASS instructions of an `ncu --page source --csv --print-source sass` dump, with
the preceding context, grouped by the instruction's opcode family."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
data = rows[2:]
S = ix["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S]) for r in data if r[S].isdigit()) or 1
top = sorted(range(len(data)), key=lambda i: -int(data[i][S]) if data[i][S].isdigit() else 0)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for i in top:
    r = data[i]
    print(f"{100 * int(r[S]) / tot:5.1f}%  {i:5d}  {r[ix['Source']].strip()[:90]}")
fam = Counter()
for r in data:
    if r[S].isdigit():
        op = r[ix["Source"]].strip().split()
        op = [t for t in op if not t.startswith("@")]
        fam[op[0].split(".")[0] if op else "?"] += int(r[S])
print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in fam.most_common(14)))
