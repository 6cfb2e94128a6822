"""Markdown table of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_table.py launches.csv "title" > profiles/x.md"""
import collections, csv, sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    tot[r[ki]] += v; cnt[r[ki]] += 1
all_ns = sum(tot.values()) or 1
print(f"# {title}\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold cache, serialised "
      "launches: compare shares, not absolutes). Unit of the raw metric: ns.\n")
print("| share | launches | total (ms) | kernel |\n|---|---|---|---|")
for k, v in tot.most_common():
    print(f"| {100 * v / all_ns:.1f}% | {cnt[k]} | {v / 1e6:.1f} | `{k[:100]}` |")
