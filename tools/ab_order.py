"""A/B: launch order of the two training calls in DeviceWorkload.step
(device-timed step and e2e fit_predict), suite16 x32 (development tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_07798_b200 import batch
import bench

series, spec, kw = bench.workload_series("suite16")
wl = batch.build_workload(series, spec, restarts=list(range(32)), precision=int(os.environ.get("PREC", "32")), **kw)
dev = batch.DeviceWorkload(wl)
s = torch.cuda.current_stream()
for rep in range(2):
    for first in (False, True):
        dev.pnn_first = first
        for _ in range(2):
            dev.step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); dev.step(); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        es = []
        for _ in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            batch.fit_predict(wl, dev, predictions=False)
            es.append(1e3 * (time.perf_counter() - t0))
        print(json.dumps({"pnn_first": first, "step_ms": [round(x) for x in ts], "e2e_ms": [round(x) for x in es]}), flush=True)
