"""Stall-reason totals (warp-stall samples) for one ncu report, optionally
restricted to source lines of a file range: python tools/ncu_stalls.py rep [file:lo-hi]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
rng = None
if len(sys.argv) > 2:
    f, span = sys.argv[2].split(":"); lo, hi = map(int, span.split("-")); rng = (f, lo, hi)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
tot = collections.Counter(); fname = None; hdr = None; line = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0].strip(): line = int(r[0])
    if rng and not (fname == rng[0] and rng[1] <= (line or 0) <= rng[2]): continue
    d = dict(zip(hdr, r))
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try: tot[k] += float(v or 0)
            except ValueError: pass
s = sum(tot.values()) or 1
for k, v in tot.most_common(12): print(f"{100*v/s:5.1f}%  {k}")
