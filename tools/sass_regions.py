"""Stall reasons per SASS region of an `ncu --page source --csv --print-source sass` dump:
    python tools/sass_regions.py DUMP.csv START:END[:name] ...   (instruction indices, end exclusive)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
data = rows[2:]
S = ix["Warp Stall Sampling (All Samples)"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S]) for r in data if r[S].isdigit()) or 1
for spec in sys.argv[2:]:
    a, b, *nm = spec.split(":")
    ch = data[int(a):int(b)]
    s = sum(int(r[S]) for r in ch if r[S].isdigit())
    rs = {k: sum(int(r[ix[k]]) for r in ch if r[ix[k]].isdigit()) for k in reasons}
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:6]
    print(f"{(nm or [''])[0]:10s} [{a}:{b}] {100 * s / tot:5.1f}% of samples: " +
          ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in top))
