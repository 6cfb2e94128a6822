"""Stall-reason breakdown from an ncu SASS source export (development tool).
usage: python tools/sass_stalls.py kernel.sass.csv[.gz] [block]
Prints per-reason totals and, per block of SASS instructions, executed
instructions and the top stall reasons."""
import csv, gzip, sys
from collections import Counter
p = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 100
op = gzip.open if p.endswith(".gz") else open
rows = list(csv.reader(op(p, "rt")))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
tot = Counter()
for r in data:
    for h in reasons:
        tot[h] += int(r[idx[h]] or 0)
T = sum(tot.values()) or 1
print("total samples", T, " instructions", sum(int(r[iE] or 0) for r in data))
print("  ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in tot.most_common(10)))
for b in range(0, len(data), B):
    blk = data[b:b + B]
    e = sum(int(r[iE] or 0) for r in blk)
    c = Counter()
    for r in blk:
        for h in reasons:
            c[h] += int(r[idx[h]] or 0)
    s = sum(c.values())
    if s > T * 0.01:
        print(f"[{b:5d}] inst {e:>11d} samples {100*s/T:5.1f}%  " +
              " ".join(f"{k[6:]}={100*v/T:.1f}" for k, v in c.most_common(4)))
