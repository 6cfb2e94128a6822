"""Per-kernel timing on synthetic workloads (development tool)."""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_07798_b200 import batch, engine
from paper_2202_07798_b200._lib import check, lib, ptr, STATUS
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="suite16")
ap.add_argument("--kind", default="both")
ap.add_argument("--precision", type=int, default=32)
ap.add_argument("--restarts", type=int, default=1)
ap.add_argument("--epochs", type=int, default=300)
ap.add_argument("--only-long", action="store_true")
ap.add_argument("--top", type=int, default=0)
ap.add_argument("--app", default=None)
ap.add_argument("--not-app", default=None)
ap.add_argument("--br-epochs", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
series, spec, kw = bench.workload_series(a.workload)
if a.only_long:
    series = sorted(series, key=lambda s: -len(s))[:1]
if a.app:
    apps = set(a.app.split(","))
    series = [s for s in series if s.key[0] in apps]
if a.not_app:
    apps = set(a.not_app.split(","))
    series = [s for s in series if s.key[0] not in apps]
if a.top:
    series = sorted(series, key=lambda s: -len(s))[:a.top]
kinds = {"both": ("pnn", "brbpnn"), "pnn": ("pnn",), "br": ("brbpnn",)}[a.kind]
kw = dict(kw); kw["kinds"] = kinds
wl = batch.build_workload(series, spec, restarts=list(range(a.restarts)), precision=a.precision,
                          pnn_epochs=a.epochs, br_max_epochs=a.br_epochs, **kw)
dev = batch.DeviceWorkload(wl)
s = torch.cuda.current_stream()
so = lib()
def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); fn(); e1.record(s); e1.synchronize(); return e0.elapsed_time(e1)
res = {}
for rep in range(a.reps):
    if len(wl.pnn):
        res["pnn_ms"] = min(res.get("pnn_ms", 1e30), timed(lambda: check(so.bbml_pnn_train(ptr(dev.pnn_tab), len(dev.pnn_tab), ptr(dev.X), ptr(dev.y), wl.train.stride, ptr(dev.weights), None, ptr(dev.status), wl.precision, s.cuda_stream), "pnn")))
    if len(wl.lm):
        off = 8 * int(wl.P_pnn.sum())
        res["lm_ms"] = timed(lambda: check(so.bbml_lm_train(ptr(dev.lm_tab), len(dev.lm_tab), ptr(dev.X), ptr(dev.y), wl.train.stride, ptr(dev.weights) + off, None, ptr(dev.status) + STATUS.itemsize * len(wl.pnn), s.cuda_stream), "lm"))
st = dev.fetch()["status"]
res["n_pnn"], res["n_lm"] = len(wl.pnn), len(wl.lm)
if len(wl.pnn):
    steps = wl.pnn["epochs"] * -(-wl.pnn["n"] // wl.pnn["batch"])
    res["pnn_max_steps"] = int(steps.max())
    res["pnn_us_per_step_critical"] = res["pnn_ms"] * 1e3 / steps.max()
if len(wl.lm):
    sl = st[len(wl.pnn):]
    res["lm_epochs"] = np.percentile(sl["epochs"], [0, 50, 90, 100]).tolist()
    res["lm_trials"] = np.percentile(sl["trials"], [0, 50, 90, 100]).tolist()
    i = int(np.argmax(sl["trials"]))
    res["lm_worst"] = dict(n=int(wl.lm["n"][i]), d=int(wl.lm["d"][i]), h=int(wl.lm["h"][i]), epochs=int(sl["epochs"][i]), trials=int(sl["trials"][i]))
    res["lm_max_n"] = int(wl.lm["n"].max())
res["codes"] = np.bincount(st["code"]).tolist()
print(json.dumps(res))
