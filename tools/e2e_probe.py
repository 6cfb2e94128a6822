"""Where an e2e (fit_predict) step's time goes: host enqueue, device span of
the step, D2H (development tool)."""
import gc, json, os, sys, time
GC = []
_t = {}
def _cb(phase, info):
    if phase == "start":
        _t["t"] = time.perf_counter()
    else:
        GC.append((info["generation"], round(1e3 * (time.perf_counter() - _t["t"]), 1)))
gc.callbacks.append(_cb)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_07798_b200 import batch
import bench

series, spec, kw = bench.workload_series("suite16")
wl = batch.build_workload(series, spec, restarts=list(range(32)), precision=32, **kw)
dev = batch.DeviceWorkload(wl)
s = torch.cuda.current_stream()
for _ in range(3):
    dev.step()
torch.cuda.synchronize()
print("objects", len(gc.get_objects()), flush=True)
for k in range(24):
    if k == 100:
        gc.collect(); gc.freeze(); print("freeze", flush=True)
    GC.clear()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    dev.upload()
    e1.record(s)
    t1 = time.perf_counter()
    dev.step()
    t2 = time.perf_counter()
    e2.record(s)
    done_at_fetch = e2.query()
    c0 = time.process_time()
    if False:
        while not e2.query():
            pass
    else:
        e2.synchronize()
    t25 = time.perf_counter()
    out = dev.fetch(False)
    t3 = time.perf_counter()
    cpu = time.process_time() - c0
    print(json.dumps({"wall_ms": round(1e3 * (t3 - t0)), "enqueue_ms": round(1e3 * (t2 - t1), 1),
                      "h2d_ms": round(e0.elapsed_time(e1), 2), "dev_step_ms": round(e1.elapsed_time(e2)),
                      "fetch_ms": round(1e3 * (t3 - t2)), "gc": [g for g in GC if g[1] > 1], "done": done_at_fetch, "wait_e2_ms": round(1e3 * (t25 - t2)), "cpu_ms": round(1e3 * cpu), "spin": bool(k % 2)}), flush=True)
