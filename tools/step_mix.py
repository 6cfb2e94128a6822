"""Concurrent train step (both kinds, as bench.py) on subsets of suite16 —
which groups set the step time (development tool)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_07798_b200 import batch
import bench

R = int(os.environ.get("R", "32"))
series, spec, kw = bench.workload_series("suite16")
wl = batch.build_workload(series, spec, restarts=list(range(R)), precision=int(os.environ.get("PREC", "32")), **kw)
dev = batch.DeviceWorkload(wl)
papp = np.array([wl.keys[i][0] for i in wl.pnn_series])
lapp = np.array([wl.keys[i][0] for i in wl.lm_series])
full_p, full_l = dev.pnn_tab, dev.lm_tab
s = torch.cuda.current_stream()

def run(name, drop_p=(), drop_l=(), no_p=False, no_l=False):
    mp = ~np.isin(papp, list(drop_p)) & (not no_p)
    ml = ~np.isin(lapp, list(drop_l)) & (not no_l)
    dev.pnn_tab = np.ascontiguousarray(full_p[mp]); dev.n_p = len(dev.pnn_tab)
    dev.lm_tab = np.ascontiguousarray(full_l[ml]); dev.n_l = len(dev.lm_tab)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); dev.step(); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(json.dumps({"case": name, "ms": round(min(ts), 1), "pnn": dev.n_p, "lm": dev.n_l}), flush=True)

run("all")
run("pnn only", no_l=True)
run("lm only", no_p=True)
if os.environ.get("STEPMIX_CASES") == "3":
    sys.exit(0)
run("-lm gramschmit", drop_l=["gramschmit"])
run("-lm pathfinder,gemm", drop_l=["pathfinder", "gemm"])
run("-pnn pathfinder,gemm", drop_p=["pathfinder", "gemm"])
run("-lm gram,path,gemm -pnn path,gemm", drop_l=["gramschmit", "pathfinder", "gemm"], drop_p=["pathfinder", "gemm"])
run("-lm path,gemm -pnn path,gemm", drop_l=["pathfinder", "gemm"], drop_p=["pathfinder", "gemm"])
run("only gramschmit lm", drop_l=[a for a in set(lapp) if a != "gramschmit"], no_p=True)
