"""Batched drop-in for ``bbcount.experiment`` (reference
``pkg/src/bbcount/experiment.py``).

The reference trains one model per ``train_one`` call (99-163) and fans the
(series x kind) tasks out over GIL-bound threads (385-401).  Here
``train_many`` is the core: it prepares every series on the host (split,
train-only normaliser — the L2 semantics), packs all training rows into one
CSR block in HBM, launches ONE fused PNN kernel and ONE LM kernel per call
on two CUDA streams (models are independent; seeds are derived on the
device from the ``series_seed`` entropy), then one batched prediction on the
test rows.  ``train_one``, ``learning_curve`` and ``run_experiment`` are
thin wrappers with the reference's signatures, results and artifacts.
"""

from __future__ import annotations

import hashlib
import json
import math
import time
import zlib
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence, Union

import numpy as np

from . import __version__, _lib, brbpnn, engine, metrics, pnn, prep
from .persist import SavedModel, save_model
from .traces import (BbSeries, Normalizer, SplitError, SplitMode, SplitSpec, classify,
                     fit_normalizer, split, trace_header)

MODEL_KINDS = ("pnn", "brbpnn")


def series_seed(base_seed: int, key: tuple, kind: str) -> int:
    """Stable per-(series, model) seed (experiment.py:38-50), via the C-ABI
    SeedSequence (the device derives the same value from the entropy)."""
    app, kernel_id, bb_id = key
    return _lib.seedseq_u64([int(base_seed) & _lib.M64, zlib.crc32(app.encode("utf-8")),
                             int(kernel_id), int(bb_id), zlib.crc32(kind.encode("utf-8"))])


@dataclass
class ExperimentConfig:
    split_mode: SplitMode = SplitMode.HIGH_LOW
    fraction: float = 0.7
    seed: int = 0
    models: tuple = MODEL_KINDS
    pnn_epochs: int = 300
    pnn_batch_size: int = 10
    pnn_learning_rate: float = 1e-4
    pnn_hidden: int = 10
    br_hidden: int = 1
    br_max_epochs: int = 1000
    workers: int = 1
    heatmap_bins: int = 32

    def split_spec(self) -> SplitSpec:
        return SplitSpec(self.split_mode, self.fraction, self.seed)

    def to_manifest(self) -> dict:
        doc = dict(self.__dict__)
        doc["split_mode"] = self.split_mode.value
        doc["models"] = list(self.models)
        return doc


@dataclass
class SeriesResult:
    key: tuple
    kind: str
    error: Optional[str] = None
    n_train: int = 0
    n_test: int = 0
    mse: Optional[float] = None
    pearson: Optional[float] = None
    spearman: Optional[float] = None
    constant_target: bool = False
    pinned_hyperparams: bool = False
    pred_raw: Optional[np.ndarray] = None
    actual_raw: Optional[np.ndarray] = None
    saved: Optional[SavedModel] = None

    @property
    def accuracy(self) -> Optional[float]:
        return None if self.mse is None else metrics.accuracy_percent(self.mse)


# ---------------------------------------------------------------------------
# host preparation (traces.py semantics)
# ---------------------------------------------------------------------------

@dataclass
class Prepared:
    series: BbSeries
    error: Optional[str] = None
    norm: Optional[Normalizer] = None
    Xtr: Optional[np.ndarray] = None
    ytr: Optional[np.ndarray] = None
    Xte: Optional[np.ndarray] = None
    yte: Optional[np.ndarray] = None
    yte_raw: Optional[np.ndarray] = None


def prepare(series: BbSeries, spec: SplitSpec) -> Prepared:
    """experiment.py:105-116 for one series: split, fit the normaliser on
    train, transform (one-series case of ``prepare_many``)."""
    return prepare_many([series], spec)[0]


def prepare_many(series_list: Sequence[BbSeries], spec: SplitSpec) -> list:
    """Split + normalise many series in whole-array passes (``prep.prepare``)
    and hand back per-series views."""
    table = prep.SeriesTable.from_series(series_list)
    P = prep.prepare(table, spec.mode.value, spec.fraction, spec.seed)
    out = []
    for i, s in enumerate(series_list):
        if i in P.errors:
            out.append(Prepared(s, error=P.errors[i]))
            continue
        d = int(table.d[i])
        a, b = int(P.tr_off[i]), int(P.tr_off[i + 1])
        c, e = int(P.te_off[i]), int(P.te_off[i + 1])
        norm = Normalizer(P.x_min[i, :d].copy(), P.x_max[i, :d].copy(), float(P.y_min[i]),
                          float(P.y_max[i]))
        out.append(Prepared(s, None, norm, P.Xtr[a:b, :d], P.ytr[a:b], P.Xte[c:e, :d], P.yte[c:e],
                            P.yte_raw[c:e]))
    return out


@dataclass
class Task:
    prep: Prepared
    kind: str
    hidden: int


def _config_error(kind: str, config: ExperimentConfig) -> Optional[str]:
    if kind == "pnn":
        try:
            pnn.TrainConfig(epochs=config.pnn_epochs, batch_size=config.pnn_batch_size,
                            learning_rate=config.pnn_learning_rate, hidden=config.pnn_hidden)
        except Exception as exc:  # same message the reference's try block records
            return f"{type(exc).__name__}: {exc}"
        return None
    if kind == "brbpnn":
        return None
    return f"ValueError: unknown model kind {kind!r}"


def _envelope_error(kind: str, d: int, h: int) -> Optional[str]:
    """Shapes the device kernels do not cover (d <= 16; PNN hidden <= 64;
    BR-BPNN P = h (d + 2) + 1 <= 512) fail this one series instead of the
    whole batched launch."""
    if d > _lib.MAX_INPUTS:
        return f"UnsupportedShape: {d} inputs exceed the device limit {_lib.MAX_INPUTS}"
    if kind == "pnn" and h > _lib.PNN_MAX_HIDDEN:
        return f"UnsupportedShape: PNN hidden {h} exceeds the device limit {_lib.PNN_MAX_HIDDEN}"
    if kind == "brbpnn" and h * (d + 2) + 1 > _lib.LM_MAX_PARAMS:
        return (f"UnsupportedShape: BR-BPNN with {h * (d + 2) + 1} parameters exceeds the device "
                f"limit {_lib.LM_MAX_PARAMS}")
    return None


@dataclass
class BatchOutput:
    results: list
    device_seconds: float = 0.0
    kernel_launches: int = 0
    extra: dict = field(default_factory=dict)


def _launch_group(kind: str, tasks: list, data: engine.DeviceData, rows: dict, config,
                  base_seed: int, precision: int):
    """Enqueue one fused training launch for all tasks of ``kind``."""
    keys = [t.prep.series.key for t in tasks]
    seeds = engine.series_seed_table(
        base_seed, np.array([zlib.crc32(k[0].encode("utf-8")) for k in keys], dtype=np.uint64),
        np.array([k[1] for k in keys], dtype=np.uint64), np.array([k[2] for k in keys], dtype=np.uint64),
        np.full(len(keys), zlib.crc32(kind.encode("utf-8")), dtype=np.uint64))
    rb = np.array([rows[id(t.prep)][0] for t in tasks], dtype=np.int64)
    n = np.array([rows[id(t.prep)][1] for t in tasks], dtype=np.int32)
    d = np.array([t.prep.Xtr.shape[1] for t in tasks], dtype=np.int32)
    h = np.array([t.hidden for t in tasks], dtype=np.int32)
    if kind == "pnn":
        tab, P = engine.pnn_tasks(rb, n, d, h, config.pnn_epochs, config.pnn_batch_size,
                                  config.pnn_learning_rate, pnn.DEFAULT_EPS, seeds, False)
        return engine.launch_pnn(data, tab, P, precision), seeds
    tab, P = engine.lm_tasks(rb, n, d, h, config.br_max_epochs, seeds, False)
    return engine.launch_lm(data, tab, P), seeds


def train_many(pairs: Sequence[tuple], config: ExperimentConfig, *, precision: Optional[int] = None,
               br_hidden_of=None, prepared: Optional[dict] = None) -> BatchOutput:
    """Train and evaluate every (series, kind) pair with batched kernels.

    A pair may carry its own split as a third element, ``(series, kind,
    SplitSpec)`` (learning curves: one split per training fraction, all in
    the same launch); otherwise ``config.split_spec()`` applies.
    ``br_hidden_of(series) -> int`` optionally overrides ``config.br_hidden``
    per series (e.g. hidden 10 for gramschmit).
    Returns SeriesResult objects in input order, identical in meaning to
    calling the reference ``train_one`` on each pair.
    """
    torch = engine.torch_cuda()
    precision = pnn.PRECISION if precision is None else precision
    spec = config.split_spec()
    cache = {} if prepared is None else prepared
    results: list = [None] * len(pairs)
    tasks: dict = {"pnn": [], "brbpnn": []}
    order: dict = {"pnn": [], "brbpnn": []}
    def cache_key(series, sp):
        return id(series) if sp is spec else (id(series), sp.mode, sp.fraction, sp.seed)

    # batched split + normalise of every (series, split) not prepared yet
    todo: dict = {}
    for pair in pairs:
        sp = pair[2] if len(pair) > 2 else spec
        ck = cache_key(pair[0], sp)
        if ck not in cache:
            todo.setdefault((sp.mode, sp.fraction, sp.seed), {})[ck] = pair[0]
    for (mode, fraction, seed), group in todo.items():
        for ck, p in zip(group, prepare_many(list(group.values()), SplitSpec(mode, fraction, seed))):
            cache[ck] = p
    for i, pair in enumerate(pairs):
        series, kind = pair[0], pair[1]
        sp = pair[2] if len(pair) > 2 else spec
        res = SeriesResult(series.key, kind)
        results[i] = res
        p = cache[cache_key(series, sp)]
        if p.error is not None:
            res.error = p.error
            continue
        res.n_train, res.n_test = len(p.ytr), len(p.yte)
        res.constant_target = p.norm.constant_target
        err = _config_error(kind, config)
        if err is not None:
            res.error = err
            continue
        hidden = config.pnn_hidden if kind == "pnn" else (
            br_hidden_of(series) if br_hidden_of else config.br_hidden)
        err = _envelope_error(kind, series.arity, int(hidden))
        if err is not None:  # isolated per series, like any other failure
            res.error = err
            continue
        tasks[kind].append(Task(p, kind, int(hidden)))
        order[kind].append(i)

    # one CSR block with every prepared series' training rows
    preps = {}
    for kind in tasks:
        for t in tasks[kind]:
            preps[id(t.prep)] = t.prep
    plist = list(preps.values())
    if not plist:
        return BatchOutput(results)
    packed = engine.pack([p.Xtr for p in plist], [p.ytr for p in plist])
    rows = {id(p): (int(packed.row_begin[j]), int(packed.n[j])) for j, p in enumerate(plist)}
    data = engine.DeviceData(packed)

    t0 = time.perf_counter()
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(main)
    runs = {}
    launches = 0
    for kind, stream in (("pnn", main), ("brbpnn", side)):
        if tasks[kind]:
            with torch.cuda.stream(stream):
                runs[kind] = _launch_group(kind, tasks[kind], data, rows, config, config.seed,
                                           precision)
                launches += 1
    main.wait_stream(side)

    # batched prediction on the (normalised) test rows of every trained model
    all_tasks, all_idx, w_parts, kinds = [], [], [], []
    fetched = {}
    for kind, (run, seeds) in runs.items():
        fetched[kind] = (run.fetch(), seeds)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    for kind, (res_k, seeds) in fetched.items():
        for j, t in enumerate(tasks[kind]):
            all_tasks.append((kind, j, t))
    if all_tasks:
        q = engine.pack([t.prep.Xte for _, _, t in all_tasks])
        dd = np.array([t.prep.Xte.shape[1] for _, _, t in all_tasks])
        hh = np.array([t.hidden for _, _, t in all_tasks])
        kk = np.array([0 if k == "pnn" else 1 for k, _, _ in all_tasks])
        W = np.concatenate([fetched[k][0].w(j) for k, j, _ in all_tasks])
        woff = engine.offsets(engine.n_params(dd, hh))
        pred_flat = engine.predict(W, woff, dd, hh, kk, q, None, eps=pnn.DEFAULT_EPS)
        # per-model test metrics on the device (bbml_metrics): MSE in the
        # normalised space, Pearson / Spearman of the de-normalised predictions
        yq = np.concatenate([t.prep.yte for _, _, t in all_tasks])
        yq_raw = np.concatenate([t.prep.yte_raw for _, _, t in all_tasks])
        Dq = max(1, int(dd.max()))
        norm_rows = np.stack([t.prep.norm.row(Dq) for _, _, t in all_tasks])
        met = engine.metrics(pred_flat, yq, yq_raw, q.row_begin, q.row_begin, q.n, dd, norm_rows)
        launches += 2
    for a, (kind, j, t) in enumerate(all_tasks):
        i = order[kind][j]
        res = results[i]
        rk = fetched[kind][0]
        st = rk.status[j]
        seed_rec = fetched[kind][1][j]
        try:
            if kind == "pnn":
                pnn.raise_for_status(st)
            else:
                brbpnn.raise_for_status(st)
        except Exception as exc:
            res.error = f"{type(exc).__name__}: {exc}"
            continue
        d = t.prep.Xtr.shape[1]
        w = rk.w(j)
        pred = pred_flat[int(q.row_begin[a]):int(q.row_begin[a]) + int(q.n[a])]
        res.mse = float(met[a, 0])
        res.pred_raw = t.prep.norm.inverse_targets(pred)
        res.actual_raw = t.prep.yte_raw
        if len(pred) >= 2:
            res.pearson = None if math.isnan(met[a, 1]) else float(met[a, 1])
            res.spearman = None if math.isnan(met[a, 2]) else float(met[a, 2])
        seed = _lib.seedseq_u64(list(_seed_entropy(seed_rec)))
        if kind == "pnn":
            model = pnn.PnnModel.from_packed(w, d, t.hidden)
            meta = {"epochs": config.pnn_epochs, "batch_size": config.pnn_batch_size,
                    "learning_rate": config.pnn_learning_rate, "hidden": config.pnn_hidden}
        else:
            hd = t.hidden * d
            model = brbpnn.BrbpnnModel(w[:hd].reshape(t.hidden, d).copy(), w[hd:hd + t.hidden].copy(),
                                       w[hd + t.hidden:hd + 2 * t.hidden].copy(), float(w[-1]),
                                       float(st["alpha"]), float(st["beta"]))
            ran = int(st["epochs"])
            res.pinned_hyperparams = bool(st["detail"])
            meta = {"hidden": t.hidden, "max_epochs": config.br_max_epochs, "epochs_run": ran,
                    "gamma": float(st["gamma"]) if ran else None,
                    "mu": float(st["mu"]) if ran else None}
        res.saved = SavedModel(kind, model, t.prep.norm, t.prep.series.key, seed, meta)
        res.saved._packed = w  # pack-order weights (columnar writer)
    return BatchOutput(results, dev_s, launches)


def _seed_entropy(rec) -> list:
    """Reassemble the entropy word list of a mode-1 seed record as one int list
    whose SeedSequence is identical (words are already 32-bit)."""
    return [int(w) for w in rec["words"][:int(rec["n_words"])]]


def train_one(series: BbSeries, kind: str, config: ExperimentConfig) -> SeriesResult:
    """Split, normalise, train one model on the device, evaluate (experiment.py:99-163)."""
    return train_many([(series, kind)], config).results[0]


@dataclass
class AppSummary:
    app: str
    kind: str
    n_series: int
    n_failed: int
    avg_mse: Optional[float]
    accuracy: Optional[float]
    pearson_pooled: Optional[float]
    spearman_pooled: Optional[float]
    any_constant_target: bool
    any_pinned: bool


def summarize(rows: Sequence[SeriesResult], split_mode: SplitMode) -> list:
    """Per (app, kind) summary (experiment.py:180-206): mean test MSE of the
    successful fits and the pooled Pearson / Spearman of all their
    de-normalised predictions vs raw counts -- every group's correlations in
    one device call (bbml_pooled_metrics, counting ranks)."""
    groups: dict = {}
    for r in rows:
        groups.setdefault((r.key[0], r.kind), []).append(r)
    keys = sorted(groups)
    seg, preds, acts = [], [], []
    for g, k in enumerate(keys):
        for r in groups[k]:
            if r.error is None:
                seg.append(g)
                preds.append(np.asarray(r.pred_raw, dtype=float))
                acts.append(np.asarray(r.actual_raw, dtype=float))
    pooled = np.full((len(keys), 2), np.nan)
    if seg:
        n = np.array([len(p) for p in preds], dtype=np.int32)
        off = engine.offsets(n.astype(np.int64))
        ident = np.tile([0.0, 1.0, 0.0, 1.0], (len(n), 1))  # predictions already de-normalised
        res = engine.pooled_metrics(np.array(seg, np.int32), np.concatenate(preds), np.concatenate(acts),
                                    off, off, n, np.ones(len(n), np.int32), ident)
        pooled[:len(res)] = res
    out = []
    for g, (app, kind) in enumerate(keys):
        grp = groups[(app, kind)]
        ok = [r for r in grp if r.error is None]
        avg = float(np.mean([r.mse for r in ok])) if ok else None
        total = sum(len(r.pred_raw) for r in ok)
        pear = None if total < 2 or math.isnan(pooled[g, 0]) else float(pooled[g, 0])
        spear = None if total < 2 or math.isnan(pooled[g, 1]) else float(pooled[g, 1])
        out.append(AppSummary(app, kind, len(grp), len(grp) - len(ok), avg,
                              None if avg is None else metrics.accuracy_percent(avg), pear, spear,
                              any(r.constant_target for r in ok), any(r.pinned_hyperparams for r in ok)))
    return out


@dataclass(frozen=True)
class CurvePoint:
    fraction: float
    accuracy: Optional[float]
    skipped: bool = False


def learning_curves(series_list: Sequence[BbSeries], kinds: Sequence[str],
                    fractions: Sequence[float], seed: int,
                    config: Optional[ExperimentConfig] = None, *, br_hidden_of=None) -> dict:
    """Batched learning curves (the reference's ``cmd_sweep``
    loop, cli.py:232-237, over ``learning_curve``, experiment.py:221-253):
    every (series, kind, fraction) fit of the sweep is one task of ONE
    ``train_many`` call -- a PNN launch and an LM launch for the whole sweep.
    Returns ``{(series.key, kind): [CurvePoint per fraction]}``; points are
    identical in meaning to calling ``learning_curve`` per series and kind
    (random split at each fraction under the shared seed; degenerate splits
    and failed fits are skipped, not fatal)."""
    config = ExperimentConfig() if config is None else config
    cfg = ExperimentConfig(**{**config.__dict__, "split_mode": SplitMode.RANDOM, "seed": seed})
    specs = [SplitSpec(SplitMode.RANDOM, float(f), seed) for f in fractions]
    triples = [(s, k, sp) for s in series_list for k in kinds for sp in specs]
    out = train_many(triples, cfg, br_hidden_of=br_hidden_of).results if triples else []
    curves: dict = {}
    for (s, k, sp), r in zip(triples, out):
        pt = (CurvePoint(sp.fraction, None, skipped=True) if r.error is not None
              else CurvePoint(sp.fraction, r.accuracy))
        curves.setdefault((s.key, k), []).append(pt)
    return curves


def learning_curve(series: BbSeries, kind: str, fractions: Sequence[float], seed: int,
                   config: Optional[ExperimentConfig] = None) -> list:
    """Random-split accuracy per training fraction (experiment.py:221-253),
    all fractions in one batched device call."""
    return learning_curves([series], [kind], fractions, seed, config)[(series.key, kind)]


def run_sweep(series_list: Sequence[BbSeries], config: ExperimentConfig, out_dir,
              fractions: Sequence[float], seed: int, input_digests=None) -> int:
    """``bbcount sweep`` (cli.py:217-248) minus argument parsing: every curve of
    the sweep from one batched call, written as ``curve_<slug>.csv`` plus
    ``sweep_manifest.json``.  Returns the number of curves."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    fractions = sorted(float(f) for f in fractions)
    curves = learning_curves(series_list, config.models, fractions, seed, config)
    for s in series_list:
        for kind in config.models:
            write_curve_csv(curves[(s.key, kind)], out_dir / f"curve_{series_slug(s.key, kind)}.csv")
    manifest = {"config": config.to_manifest(), "fractions": fractions,
                "inputs": dict(input_digests or {}), "curves": len(curves)}
    with open(out_dir / "sweep_manifest.json", "w", encoding="utf-8", newline="\n") as fh:
        json.dump(manifest, fh, indent=2)
        fh.write("\n")
    return len(curves)


# ---------------------------------------------------------------------------
# artifacts (experiment.py:261-370)
# ---------------------------------------------------------------------------

def _fmt(v) -> str:
    if v is None:
        return "undefined"
    if isinstance(v, bool):
        return str(v).lower()
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    return str(v)


def series_slug(key: tuple, kind: Optional[str] = None) -> str:
    s = f"{key[0]}_k{key[1]}_b{key[2]}"
    return f"{s}_{kind}" if kind else s


def write_report_csv(rows: Sequence[SeriesResult], path: Path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("app,kernel_id,bb_id,model,n_train,n_test,mse,accuracy,"
                 "pearson,spearman,constant_target,pinned_hyperparams,error\n")
        for r in sorted(rows, key=lambda r: (r.key, r.kind)):
            err = (r.error or "").replace(",", ";")
            fh.write(f"{r.key[0]},{r.key[1]},{r.key[2]},{r.kind},{r.n_train},{r.n_test},"
                     f"{_fmt(r.mse)},{_fmt(r.accuracy)},{_fmt(r.pearson)},{_fmt(r.spearman)},"
                     f"{_fmt(r.constant_target)},{_fmt(r.pinned_hyperparams)},{err}\n")


def write_summary_csv(summaries: Sequence[AppSummary], split_mode: SplitMode, path: Path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("app,split,model,n_series,n_failed,avg_mse,accuracy_percent,"
                 "pearson_pooled,spearman_pooled,constant_target,pinned_hyperparams\n")
        for s in summaries:
            fh.write(f"{s.app},{split_mode.value},{s.kind},{s.n_series},{s.n_failed},"
                     f"{_fmt(s.avg_mse)},{_fmt(s.accuracy)},{_fmt(s.pearson_pooled)},"
                     f"{_fmt(s.spearman_pooled)},{_fmt(s.any_constant_target)},{_fmt(s.any_pinned)}\n")


def write_heatmap_csv(data: metrics.HeatmapData, path: Path) -> None:
    e = data.edges
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("pred_bin,actual_bin,pred_low,pred_high,actual_low,actual_high,count,on_identity\n")
        for i in range(data.bins):
            for j in range(data.bins):
                fh.write(f"{i},{j},{_fmt(float(e[i]))},{_fmt(float(e[i + 1]))},{_fmt(float(e[j]))},"
                         f"{_fmt(float(e[j + 1]))},{int(data.counts[i, j])},{_fmt(i == j)}\n")


def write_kde_csv(curve: metrics.KdeCurve, path: Path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("x,density\n")
        for x, dv in zip(curve.grid, curve.density):
            fh.write(f"{_fmt(float(x))},{_fmt(float(dv))}\n")


def write_curve_csv(points: Sequence[CurvePoint], path: Path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("fraction,accuracy,skipped\n")
        for p in points:
            fh.write(f"{_fmt(p.fraction)},{_fmt(p.accuracy)},{_fmt(p.skipped)}\n")


def write_split_manifests(series_list: Sequence[BbSeries], spec: SplitSpec, out_dir: Path) -> None:
    """splits_<app>.csv: every trace row with its partition (experiment.py:
    344-362); the labels of all series come from one batched prep pass."""
    table = prep.SeriesTable.from_series(series_list)
    labels, errors = prep.split_labels(table, spec.mode.value, spec.fraction, spec.seed)
    names = np.array(["discarded", "train", "test"], dtype=object)
    by_app: dict = {}
    for i, s in enumerate(series_list):
        by_app.setdefault(s.key[0], []).append(i)
    for app, idx in sorted(by_app.items()):
        lines = [",".join(trace_header(series_list[idx[0]].arity) + ["partition"])]
        for i in idx:
            s = series_list[i]
            a, b = int(table.offsets[i]), int(table.offsets[i + 1])
            # a constant-feature range split labels the whole series "error"
            bad = i in errors and "are constant" in errors[i]
            lab = ["error"] * (b - a) if bad else names[labels[a:b]]
            head = f"{s.key[0]},{s.key[1]},{s.key[2]},"
            for row, count, l in zip(s.X, s.y, lab):
                lines.append(head + ",".join(str(int(v)) for v in row) + f",{int(count)},{l}")
        with open(out_dir / f"splits_{app}.csv", "w", encoding="utf-8", newline="\n") as fh:
            fh.write("\n".join(lines) + "\n")


def write_splits_columnar(series_list: Sequence[BbSeries], spec: SplitSpec, path: Path) -> None:
    """The splits manifest as arrays (columnar layout): per series its key
    and row range (CSR offsets into the input trace rows, in input order),
    per row its partition code (0 discarded, 1 train, 2 test, -1 the
    series' range split failed: the reference's ``error`` label)."""
    table = prep.SeriesTable.from_series(series_list)
    labels, errors = prep.split_labels(table, spec.mode.value, spec.fraction, spec.seed)
    lab = labels.astype(np.int8)
    for i, msg in errors.items():
        if "are constant" in msg:
            lab[table.offsets[i]:table.offsets[i + 1]] = -1
    np.savez(path, app=np.array([k[0] for k in table.keys]).astype(str),
             kernel_id=np.array([k[1] for k in table.keys], dtype=np.int64),
             bb_id=np.array([k[2] for k in table.keys], dtype=np.int64), offsets=table.offsets,
             partition=lab)


def device_heatmaps(rows: Sequence[SeriesResult], bins: int):
    """Heatmap edges / counts of every successful row in one device call
    (bbml_heatmaps); returns (row indices, edges (M, bins+1), counts (M, bins, bins))."""
    idx = [i for i, r in enumerate(rows)
           if r.error is None and r.pred_raw is not None and len(r.pred_raw)]
    if not idx:
        return idx, np.zeros((0, bins + 1)), np.zeros((0, bins, bins), np.int32)
    preds = [np.asarray(rows[i].pred_raw, dtype=float) for i in idx]
    n = np.array([len(p) for p in preds], dtype=np.int32)
    off = engine.offsets(n.astype(np.int64))
    ident = np.tile([0.0, 1.0, 0.0, 1.0], (len(idx), 1))  # predictions already de-normalised
    edges, counts = engine.heatmaps(np.concatenate(preds),
                                    np.concatenate([np.asarray(rows[i].actual_raw, float) for i in idx]),
                                    off, off, n, np.ones(len(idx), np.int32), ident, bins)
    return idx, edges, counts


_CFG_NUMERIC = ("epochs_run", "gamma", "mu")  # per-model BR values, kept as columns


def write_models_columnar(rows: Sequence[SeriesResult], path: Path) -> int:
    """Every saved model of a run in ONE columnar file (numpy .npz): keys,
    kinds, shapes, seeds, flat pack-order weights + offsets, normalisers,
    BR hyperparameters, the per-model config as a shared JSON template plus
    numeric columns.  ``export_models_json`` turns it into the reference's
    per-model JSON (schema v1) files."""
    saved = [r.saved for r in rows if r.saved is not None]
    M = len(saved)
    models = [m.model for m in saved]
    d = np.fromiter((m.n_inputs for m in models), dtype=np.int32, count=M)
    h = np.fromiter((m.hidden for m in models), dtype=np.int32, count=M)
    w = [getattr(m, "_packed", None) for m in saved]
    w = [x if x is not None else np.concatenate([np.ravel(mm.W1), mm.b1, mm.W2, [mm.b2]])
         for x, mm in zip(w, models)]
    D = max(1, int(d.max())) if M else 1
    norm = np.zeros((M, 2 * D + 2))
    for i, m in enumerate(saved):  # [x_min(d), x_max(d), y_min, y_max]
        nm, di = m.normalizer, int(d[i])
        norm[i, :di] = nm.x_min
        norm[i, di:2 * di] = nm.x_max
        norm[i, 2 * di] = nm.y_min
        norm[i, 2 * di + 1] = nm.y_max
    templates: dict = {}
    tpl = np.zeros(M, dtype=np.int32)
    num = np.full((M, len(_CFG_NUMERIC)), np.nan)
    isnone = np.zeros((M, len(_CFG_NUMERIC)), dtype=bool)
    for i, m in enumerate(saved):
        cfg = m.config
        key = tuple((k, None if k in _CFG_NUMERIC else v) for k, v in cfg.items())
        tpl[i] = templates.setdefault(key, len(templates))
        for c, k in enumerate(_CFG_NUMERIC):
            if k in cfg:
                v = cfg[k]
                if v is None:
                    isnone[i, c] = True
                else:
                    num[i, c] = v
    tpl_json = [json.dumps(dict(k)) for k in sorted(templates, key=templates.get)]
    np.savez(path,
             app=np.array([m.key[0] for m in saved]).astype(str),
             kernel_id=np.fromiter((m.key[1] for m in saved), dtype=np.int64, count=M),
             bb_id=np.fromiter((m.key[2] for m in saved), dtype=np.int64, count=M),
             kind=np.array([m.kind for m in saved]).astype(str), d=d, h=h,
             seed=np.array([str(m.seed) for m in saved]).astype(str),
             weights=np.concatenate(w) if w else np.zeros(0),
             w_offset=engine.offsets(np.array([len(x) for x in w], dtype=np.int64)) if M else np.zeros(0, np.int64),
             norm=norm,
             eps=np.fromiter((getattr(m, "eps", np.nan) for m in models), dtype=np.float64, count=M),
             alpha=np.fromiter((getattr(m, "alpha", np.nan) for m in models), dtype=np.float64, count=M),
             beta=np.fromiter((getattr(m, "beta", np.nan) for m in models), dtype=np.float64, count=M),
             config_template=np.array(tpl_json).astype(str), config_index=tpl,
             config_numeric=num, config_none=isnone,
             config_int=np.array([k in ("epochs_run",) for k in _CFG_NUMERIC]))
    return M


def read_kde_columnar(path: Union[str, Path]) -> dict:
    """{slug: KdeCurve} from kde.npz (grid rebuilt as linspace(lo, hi, G))."""
    z = np.load(path, allow_pickle=False)
    G = z["density"].shape[1] if z["density"].ndim == 2 else 256
    return {str(s): metrics.KdeCurve(np.linspace(z["lo"][i], z["hi"][i], G), z["density"][i],
                                     float(z["bandwidth"][i])) for i, s in enumerate(z["slug"])}


def read_heatmaps_columnar(path: Union[str, Path]) -> dict:
    """{slug: HeatmapData} from heatmaps.npz (sparse counts back to bins x bins)."""
    z = np.load(path, allow_pickle=False)
    B = int(z["bins"])
    counts = np.zeros((len(z["slug"]), B * B), dtype=np.int64)
    counts[z["model"], z["bin"]] = z["count"]
    return {str(s): metrics.HeatmapData(z["edges"][i], counts[i].reshape(B, B))
            for i, s in enumerate(z["slug"])}


def read_models_columnar(path: Union[str, Path]) -> list:
    """SavedModel objects back from ``models.npz``."""
    z = np.load(path, allow_pickle=False)
    out = []
    for i in range(len(z["d"])):
        d, h = int(z["d"][i]), int(z["h"][i])
        w = z["weights"][int(z["w_offset"][i]):int(z["w_offset"][i]) + h * (d + 2) + 1]
        hd = h * d
        W1, b1, W2, b2 = w[:hd].reshape(h, d).copy(), w[hd:hd + h].copy(), w[hd + h:hd + 2 * h].copy(), float(w[-1])
        kind = str(z["kind"][i])
        model = (pnn.PnnModel(W1, b1, W2, b2, eps=float(z["eps"][i])) if kind == "pnn" else
                 brbpnn.BrbpnnModel(W1, b1, W2, b2, alpha=float(z["alpha"][i]), beta=float(z["beta"][i])))
        row = z["norm"][i]
        norm = Normalizer(row[:d].copy(), row[d:2 * d].copy(), float(row[2 * d]), float(row[2 * d + 1]))
        key = (str(z["app"][i]), int(z["kernel_id"][i]), int(z["bb_id"][i]))
        cfg = json.loads(str(z["config_template"][int(z["config_index"][i])]))
        for c, k in enumerate(_CFG_NUMERIC):
            if k in cfg:
                v = z["config_numeric"][i, c]
                cfg[k] = None if z["config_none"][i, c] else (int(v) if z["config_int"][c] else float(v))
        out.append(SavedModel(kind, model, norm, key, int(z["seed"][i]), cfg))
    return out


def export_models_json(columnar: Union[str, Path], out_dir: Union[str, Path]) -> int:
    """The reference layout (models/<slug>.json, schema v1) from models.npz."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    models = read_models_columnar(columnar)
    for m in models:
        save_model(m, out_dir / f"{series_slug(m.key, m.kind)}.json")
    return len(models)


def digest_file(path: Union[str, Path]) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(65536), b""):
            h.update(chunk)
    return h.hexdigest()


@dataclass
class ExperimentOutput:
    rows: list
    summaries: list
    out_dir: Path


def run_experiment(series_list: Sequence[BbSeries], config: ExperimentConfig,
                   out_dir: Union[str, Path], input_digests: Optional[dict] = None,
                   br_hidden_of=None, layout: str = "files") -> ExperimentOutput:
    """experiment.py:385-451 with ONE batched device call for all tasks
    (``workers`` is accepted for compatibility; results never depend on it).

    ``layout="files"`` writes the reference's artifact tree (report.csv,
    summary.csv, splits_<app>.csv, models/<slug>.json, heatmap_<slug>.csv,
    kde_<slug>.csv, manifest.json).  ``layout="columnar"`` keeps report /
    summary / manifest and replaces the per-model / per-series files with
    models.npz, heatmaps.npz and kde.npz (one file each however many models:
    cfg 4 has 320k of them) and splits_<app>.csv with splits.npz (per-row
    partition codes); ``export_models_json`` recovers the JSON files.
    Heatmaps and the summary correlations come from the device in one call
    each."""
    if layout not in ("files", "columnar"):
        raise ValueError(f"layout must be 'files' or 'columnar', got {layout!r}")
    started = time.time()
    clock = {}
    t0 = time.perf_counter()
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    pairs = [(s, k) for s in series_list for k in config.models]
    rows = train_many(pairs, config, br_hidden_of=br_hidden_of).results
    clock["train_predict_metrics_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rows.sort(key=lambda r: (r.key, r.kind))
    if rows and all(r.error is not None for r in rows):
        raise RuntimeError("all series failed; first error: " + str(rows[0].error))
    last = [time.perf_counter()]

    def mark(name):  # per-stage wall clock into ExperimentOutput.timing
        now = time.perf_counter()
        clock[name] = now - last[0]
        last[0] = now

    summaries = summarize(rows, config.split_mode)
    mark("summarize_s")
    write_report_csv(rows, out_dir / "report.csv")
    write_summary_csv(summaries, config.split_mode, out_dir / "summary.csv")
    if layout == "files":
        write_split_manifests(series_list, config.split_spec(), out_dir)
    else:
        write_splits_columnar(series_list, config.split_spec(), out_dir / "splits.npz")
    mark("report_summary_splits_s")
    hm_idx, hm_edges, hm_counts = device_heatmaps(rows, config.heatmap_bins)
    mark("heatmaps_s")
    kdes = []
    if layout == "files":  # host numpy: the reference's kde_*.csv byte for byte
        for s in series_list:
            try:
                kdes.append((s.key, metrics.kde(s.y)))
            except (metrics.BandwidthError, metrics.MetricShapeError):
                continue
    else:  # one device call for every series (bbml_kde; within 1e-12 of numpy)
        grid, dens, bw = engine.kde([s.y for s in series_list])
        kdes = [(s.key, metrics.KdeCurve(grid[i], dens[i], float(bw[i])))
                for i, s in enumerate(series_list) if bw[i] > 0.0]
    mark("kde_s")
    if layout == "files":
        models_dir = out_dir / "models"
        models_dir.mkdir(exist_ok=True)
        for r in rows:
            if r.saved is not None:
                save_model(r.saved, models_dir / f"{series_slug(r.key, r.kind)}.json")
        for j, i in enumerate(hm_idx):
            r = rows[i]
            write_heatmap_csv(metrics.HeatmapData(hm_edges[j], hm_counts[j]),
                              out_dir / f"heatmap_{series_slug(r.key, r.kind)}.csv")
        for key, curve in kdes:
            write_kde_csv(curve, out_dir / f"kde_{series_slug(key)}.csv")
    else:
        write_models_columnar(rows, out_dir / "models.npz")
        mark("models_npz_s")
        flat = hm_counts.reshape(len(hm_idx), -1)  # sparse: most bins are empty
        mi, bi = np.nonzero(flat)
        np.savez(out_dir / "heatmaps.npz",
                 slug=np.array([series_slug(rows[i].key, rows[i].kind) for i in hm_idx]).astype(str),
                 edges=hm_edges, bins=np.array(config.heatmap_bins), model=mi.astype(np.int32),
                 bin=bi.astype(np.int32), count=flat[mi, bi].astype(np.int32))
        # the grid is linspace(lo, hi, 256): stored as its two ends
        np.savez(out_dir / "kde.npz", slug=np.array([series_slug(k) for k, _ in kdes]).astype(str),
                 lo=np.array([c.grid[0] for _, c in kdes]), hi=np.array([c.grid[-1] for _, c in kdes]),
                 density=np.stack([c.density for _, c in kdes]) if kdes else np.zeros((0, 256)),
                 bandwidth=np.array([c.bandwidth for _, c in kdes]))
        mark("heatmaps_kde_npz_s")
    clock["artifacts_s"] = time.perf_counter() - t0
    manifest = {
        "config": config.to_manifest(),
        "inputs": input_digests or {},
        "series": [{"app": s.key[0], "kernel_id": s.key[1], "bb_id": s.key[2], "n": len(s)}
                   for s in series_list],
        "errors": {series_slug(r.key, r.kind): r.error for r in rows if r.error is not None},
        "versions": {"bbcount": __version__, "numpy": np.__version__},
        "wall_time_seconds": time.time() - started,
    }
    with open(out_dir / "manifest.json", "w", encoding="utf-8", newline="\n") as fh:
        json.dump(manifest, fh, indent=2)
        fh.write("\n")
    out = ExperimentOutput(rows, summaries, out_dir)
    out.timing = clock  # not in the manifest: it would break byte-identical reruns
    return out
