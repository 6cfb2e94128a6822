"""Parity of EXACTLY what bench.py times: the suite16 workload (BASELINE
cfg 3: 16 Table-1-shaped apps, random split 0.7, PNN + BR-BPNN, hidden 10 for
gramschmit's BR fits) built by ``batch.build_workload`` and trained /
predicted / scored by ``batch.DeviceWorkload.step`` — at FP64 (the headline)
and FP32 — against the CPU oracle's ``train_one`` on every one of the 1,018
models (restart 0 = run seed 0, the reference's own seeding).

Gates (north star):
  * status: a model fails on the device iff the oracle's fails;
  * PNN predicted counts: FP64 <= 1e-12 relative, FP32 <= 1e-3 relative
    (floor 1e-6 of the series' count scale);
  * BR-BPNN (hidden 1, and hidden 10 for gramschmit at the bench's 1000
    epochs): predicted counts <= max(1e-3, 25 x the oracle's own 1-ulp
    spread) — the spread (the oracle re-run with its normalised training
    targets / features moved by one ulp, oracle.PERTURBATIONS) is computed
    here for every fit that misses 1e-3 and must itself exceed 1e-3/25, so
    no fit passes on an accuracy-only branch;
  * per app x kind: |accuracy_device - accuracy_oracle| <= 0.5 pp, accuracy
    = 100 (1 - mean test MSE) as in experiment.summarize;
  * device test MSE (bbml_metrics) equals the MSE of the device predictions.
The oracle runs in a process pool over the host cores (~15 s on the GPU
box's 16 cores); it is the checker only.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bench  # noqa: E402
from paper_2202_07798_b200 import batch, synth  # noqa: E402
from oracle.pool import oracle_map, rel as _rel, self_spread  # noqa: E402


KW = dict(mode="random", fraction=0.7, base_seed=0)


@pytest.fixture(scope="module")
def suite():
    series, spec, kw = bench.workload_series("suite16")
    jobs = []
    for s in series:
        for kind in ("pnn", "brbpnn"):
            h = synth.suite16_hidden(s.key[0]) if kind == "brbpnn" else 1
            jobs.append((s.key, s.X, s.y, kind, dict(KW, br_hidden=h), None))
    oracle = oracle_map(jobs)
    return series, spec, kw, jobs, dict(zip([(j[0], j[3]) for j in jobs], oracle))


def _device(series, spec, kw, precision):
    wl = batch.build_workload(series, spec, restarts=[0], precision=precision, **kw)
    dev = batch.DeviceWorkload(wl)
    dev.step()
    out = dev.fetch(predictions=True)
    tab = dev.pred_tab
    sids = np.concatenate([wl.pnn_series, wl.lm_series]).astype(np.int64)
    kinds = ["pnn"] * len(wl.pnn) + ["brbpnn"] * len(wl.lm)
    res = {}
    for m, (sid, kind) in enumerate(zip(sids, kinds)):
        off, n = int(tab["out_offset"][m]), int(tab["n"][m])
        pred = out["pred"][off:off + n]
        res[(wl.keys[sid], kind)] = dict(
            code=int(out["status"]["code"][m]), pred_raw=wl.norms[sid].inverse_targets(pred),
            mse=float(out["metrics"][m, 0]), pred=pred,
            yte=wl.test.y[int(wl.test.row_begin[sid]):int(wl.test.row_begin[sid]) + n])
    return wl, res


@pytest.mark.parametrize("precision", [64, 32])
def test_suite16_bench_path_matches_oracle(suite, precision):
    series, spec, kw, jobs, oracle = suite
    wl, dev = _device(series, spec, kw, precision)
    assert len(dev) == len(oracle) == 1018
    scale = {s.key: max(1.0, float(np.max(np.abs(s.y)))) for s in series}
    errs = {"pnn": [], "br1": [], "br10": []}
    spread_needed = []
    acc = {}
    for (key, kind), o in oracle.items():
        d = dev[(key, kind)]
        o_err, o_mse, o_pred, n_te = o.error, o.mse, o.pred_raw, o.n_test
        assert (d["code"] == 0) == (o_err is None), (key, kind, d["code"], o_err)
        if o_err is not None:
            continue
        assert len(d["pred_raw"]) == n_te
        # the device metric is the MSE of the device predictions
        assert abs(d["mse"] - float(np.mean((d["pred"] - d["yte"]) ** 2))) <= 1e-12 * max(1.0, d["mse"])
        e = _rel(d["pred_raw"], o_pred, 1e-6 * scale[key])
        h = synth.suite16_hidden(key[0])
        if kind == "pnn":
            errs["pnn"].append(e)
            assert e <= (1e-12 if precision == 64 else 1e-3), (key, e)
        else:
            errs["br1" if h == 1 else "br10"].append(e)
            if e > 1e-3:
                spread_needed.append((key, h, e))
        acc.setdefault((key[0], kind), ([], []))
        acc[(key[0], kind)][0].append(d["mse"])
        acc[(key[0], kind)][1].append(o_mse)
    # BR fits beyond 1e-3: gate at 25x the oracle's own 1-ulp spread
    if spread_needed:
        by_key = {s.key: s for s in series}
        for key, h, e in spread_needed:
            s = by_key[key]
            spread = self_spread(key, s.X, s.y, "brbpnn", dict(KW, br_hidden=h),
                                 oracle[(key, "brbpnn")].pred_raw, 1e-6 * scale[key])
            print(f"BR h={h} {key}: device {e:.2e} vs oracle 1-ulp spread {spread:.2e}")
            assert spread * 25 >= 1e-3 and e <= 25 * spread, (key, e, spread)
    for (app, kind), (dm, om) in sorted(acc.items()):
        a_d, a_o = 100 * (1 - np.mean(dm)), 100 * (1 - np.mean(om))
        assert abs(a_d - a_o) <= 0.5, (app, kind, a_d, a_o)
    q = {k: (np.percentile(v, [50, 99, 100]).tolist() if v else None) for k, v in errs.items()}
    print(f"precision {precision}: rel err p50/p99/max {q}; BR beyond 1e-3: {len(spread_needed)}")
