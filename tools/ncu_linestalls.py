"""Per-source-line stall breakdown (top lines) within a file line range.
usage: python tools/ncu_linestalls.py rep file:lo-hi [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; f0, span = sys.argv[2].split(":"); lo, hi = map(int, span.split("-"))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
per = collections.defaultdict(collections.Counter); src = {}; fname = None; hdr = None; line = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0].strip(): line = int(r[0]); src[(fname, line)] = r[1].strip()[:70]
    d = dict(zip(hdr, r))
    key = (fname, line)
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try: per[key][k[6:]] += float(v or 0)
            except ValueError: pass
    try: per[key]["_inst"] += float(d.get("Instructions Executed", 0) or 0)
    except ValueError: pass
# keep the kernel's range; include inlined helpers (other files) too
tot = sum(sum(v for k, v in c.items() if k != "_inst") for c in per.values()) or 1
rows = sorted(per.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_inst"))
for key, c in rows[:top]:
    s = sum(v for k, v in c.items() if k != "_inst")
    if key[0] == f0 and not (lo <= (key[1] or 0) <= hi): continue
    reasons = ", ".join(f"{k}:{100*v/s:.0f}" for k, v in c.most_common(4) if k != "_inst")
    print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]:<4} [{reasons}] {src.get(key,'')}")
