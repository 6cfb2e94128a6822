"""Per-app LM (BR-BPNN) or PNN (KIND=pnn) timing on suite16 (development tool)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_07798_b200 import batch
from paper_2202_07798_b200._lib import check, lib, ptr, STATUS
import bench

R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
series, spec, kw = bench.workload_series("suite16")
so = lib()
s = torch.cuda.current_stream()
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for app in sorted({x.key[0] for x in series}):
    if only and app not in only:
        continue
    ss = [x for x in series if x.key[0] == app]
    pnn = os.environ.get("KIND") == "pnn"
    kw2 = dict(kw); kw2["kinds"] = ("pnn",) if pnn else ("brbpnn",)
    wl = batch.build_workload(ss, spec, restarts=list(range(R)), precision=32, **kw2)
    dev = batch.DeviceWorkload(wl)
    ts = []
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if pnn:
            check(so.bbml_pnn_train(ptr(dev.pnn_tab), len(dev.pnn_tab), ptr(dev.X), ptr(dev.y), wl.train.stride,
                                    ptr(dev.weights), None, ptr(dev.status), wl.precision, s.cuda_stream), "pnn")
        else:
            check(so.bbml_lm_train(ptr(dev.lm_tab), len(dev.lm_tab), ptr(dev.X), ptr(dev.y), wl.train.stride,
                                   ptr(dev.weights), None, ptr(dev.status), s.cuda_stream), "lm")
        e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    st = dev.fetch()["status"]
    tab = wl.pnn if pnn else wl.lm
    if pnn:
        print(json.dumps(dict(app=app, ms=round(min(ts), 1), models=len(tab), n_max=int(tab["n"].max()),
                              steps_max=int((tab["epochs"] * -(-tab["n"] // tab["batch"])).max()))), flush=True)
        continue
    print(json.dumps(dict(app=app, ms=round(min(ts), 1), models=len(wl.lm), n_max=int(wl.lm["n"].max()),
                          d=int(wl.lm["d"][0]), h=int(wl.lm["h"][0]),
                          epochs=np.percentile(st["epochs"], [50, 90, 100]).tolist(),
                          trials=np.percentile(st["trials"], [50, 90, 100]).tolist())), flush=True)
