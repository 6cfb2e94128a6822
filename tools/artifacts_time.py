"""Time run_experiment's artifact writing against training at cfg-4 scale
(10 000 series x 2 kinds), both layouts (development / evidence tool)."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2202_07798_b200 import experiment as E
from paper_2202_07798_b200.traces import SplitMode

series, spec, kw = bench.workload_series("sweep")
cfg = E.ExperimentConfig(split_mode=SplitMode.HIGH_LOW, seed=0)
E.train_many([(s, "pnn") for s in series[:20]], cfg)  # warm the library / module load
res = {}
for layout in ("columnar", "files"):
    with tempfile.TemporaryDirectory() as d:
        t0 = time.perf_counter()
        out = E.run_experiment(series if layout == "columnar" else series[:2000], cfg, d, layout=layout)
        res[layout] = dict(out.timing, models=len(out.rows), wall_s=time.perf_counter() - t0)
print(json.dumps(res))
