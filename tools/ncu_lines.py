"""Aggregate ncu per-SASS stall samples onto CUDA source lines (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
agg = collections.Counter(); inst = collections.Counter(); src = {}
fname = None; hdr = None; line = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 5:
        continue
    if r[0].strip():
        line = r[0]; src[(fname, line)] = r[1].strip()[:90]
    try:
        s = float(r[4] or 0); e = float(r[7] or 0)
    except ValueError:
        continue
    agg[(fname, line)] += s; inst[(fname, line)] += e
tot = sum(agg.values()) or 1
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{100*v/tot:5.1f}% inst={inst[k]:>9.0f} {k[0]}:{k[1]:<5} {src.get(k,'')}")

if len(sys.argv) > 3:
    # split consumer/producer by source ranges: argv[3] = "file:lo-hi,file:lo-hi" for producer
    rng = []
    for part in sys.argv[3].split(","):
        f, span = part.split(":")
        lo, hi = map(int, span.split("-"))
        rng.append((f, lo, hi))
    def is_prod(k):
        return any(k[0] == f and lo <= int(k[1] or 0) <= hi for f, lo, hi in rng)
    ps = sum(v for k, v in agg.items() if is_prod(k)); pi = sum(v for k, v in inst.items() if is_prod(k))
    cs = sum(v for k, v in agg.items() if not is_prod(k)); ci = sum(v for k, v in inst.items() if not is_prod(k))
    print(f"producer: samples {ps:.0f} inst {pi:.0f} | consumer: samples {cs:.0f} inst {ci:.0f}")
    if len(sys.argv) > 4:
        steps = float(sys.argv[4])
        rows = sorted(((v, k) for k, v in inst.items() if not is_prod(k)), reverse=True)[:40]
        for v, k in rows:
            print(f"{v/steps:7.1f} inst/step  {100*agg[k]/cs:5.1f}% smp  {k[0]}:{k[1]:<5} {src.get(k,'')[:80]}")
