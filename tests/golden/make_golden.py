"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (needs ``/root/reference``):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Writes small ``.npz`` files next to this script.  The GPU box never reads
``/root/reference``; tests compare against these committed files.
Each file records the NumPy version that produced it.
"""

from __future__ import annotations

import dataclasses
import io
import os
import sys
import zlib

import numpy as np

REF = os.environ.get("BBML_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from bbcount import brbpnn, pnn  # noqa: E402  (reference)
from bbcount.experiment import ExperimentConfig, series_seed, train_one  # noqa: E402
from bbcount.families import GridSpec, family_by_name, generate_dataset  # noqa: E402
from bbcount.persist import SavedModel  # noqa: E402
from bbcount.traces import BbSeries, Normalizer, SplitMode, ingest  # noqa: E402

from paper_2202_07798_b200 import synth  # noqa: E402  (input generator only)

OUT = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


def words(x: int, n: int) -> list[int]:
    return [(x >> (64 * i)) & M64 for i in range(n)]


def save(name: str, d: dict) -> None:
    d["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(os.path.join(OUT, name), **d)
    print(name, os.path.getsize(os.path.join(OUT, name + ".npz")), "bytes")


def gen_rng():
    d = {}
    seeds = [0, 1, 123, 2**63 + 5, 2**64 + 7, 2**96 + 11]
    d["seeds_lo"] = np.array([s & M64 for s in seeds], dtype=np.uint64)
    d["seeds_hi"] = np.array([s >> 64 for s in seeds], dtype=np.uint64)
    for i, s in enumerate(seeds):
        r = np.random.default_rng(s)
        st = r.bit_generator.state["state"]
        d[f"s{i}_state"] = np.array(words(st["state"], 2) + words(st["inc"], 2), dtype=np.uint64)
        d[f"s{i}_uniform"] = r.uniform(-0.7, 0.7, size=(10, 2)).ravel()
        d[f"s{i}_scalar"] = np.array(float(r.uniform(-1.0, 1.0)))
        for n in (1, 2, 3, 7, 100, 1000):
            d[f"s{i}_perm{n}"] = r.permutation(n)
        d[f"s{i}_tail_uniform"] = r.uniform(0.0, 1.0, size=5)
    keys = [("app", 0, 1), ("app", 0, 2), ("linear", 0, 2), ("2mm", 0, 20), ("x", 3, 99999)]
    ss = []
    for base in (0, 7, 2**40, M64):
        for key in keys:
            for kind in ("pnn", "brbpnn"):
                ss.append((base, zlib.crc32(key[0].encode()), key[1], key[2],
                           zlib.crc32(kind.encode()), series_seed(base, key, kind)))
    d["series_seed"] = np.array(ss, dtype=np.uint64)
    save("rng", d)


PNN_CASES = [
    # d, h, n, epochs, batch, lr, seed
    (2, 10, 100, 30, 10, 1e-4, 7),
    (1, 10, 37, 12, 10, 1e-4, 123),
    (3, 5, 23, 9, 4, 1e-3, 5),
    (4, 10, 1, 4, 10, 1e-4, 9),
    (2, 1, 17, 6, 1, 1e-2, 11),
    (1, 3, 40, 20, 32, 1e-4, 2**63 + 3),
    (2, 10, 64, 15, 10, 5e-2, 42),
    (4, 7, 55, 5, 6, 1e-4, 0),
]


def gen_pnn():
    d = {}
    rng = np.random.default_rng(2024)
    for i, (di, h, n, ep, bs, lr, seed) in enumerate(PNN_CASES):
        X = rng.uniform(0.0, 1.0, size=(n, di))
        y = rng.uniform(0.0, 1.0, size=n)
        cfg = pnn.TrainConfig(epochs=ep, batch_size=bs, learning_rate=lr, seed=seed, hidden=h)
        m, hist = pnn.train(X, y, cfg)
        Xt = rng.uniform(-0.5, 1.5, size=(13, di))
        d[f"c{i}_cfg"] = np.array([di, h, n, ep, bs], dtype=np.int64)
        d[f"c{i}_lr"] = np.array(lr)
        d[f"c{i}_seed"] = np.array(words(seed, 2), dtype=np.uint64)
        d[f"c{i}_X"], d[f"c{i}_y"] = X, y
        d[f"c{i}_w"] = np.concatenate([m.W1.ravel(), m.b1, m.W2, [m.b2]])
        d[f"c{i}_hist"] = np.array(hist)
        d[f"c{i}_Xt"] = Xt
        d[f"c{i}_pred"] = np.atleast_1d(pnn.forward(m, Xt))
    d["n_cases"] = np.array(len(PNN_CASES))
    # unit level: loss_and_grads, forward
    for i in range(12):
        di = int(rng.integers(1, 5))
        h = int(rng.integers(1, 11))
        m = pnn.init_model(di, hidden=h, rng=rng)
        X = rng.uniform(-1.0, 1.5, size=(int(rng.integers(1, 11)), di))
        y = rng.uniform(0.0, 1.5, size=len(X))
        loss, g = pnn.loss_and_grads(m, X, y)
        d[f"u{i}_dh"] = np.array([di, h])
        d[f"u{i}_w"] = np.concatenate([m.W1.ravel(), m.b1, m.W2, [m.b2]])
        d[f"u{i}_X"], d[f"u{i}_y"] = X, y
        d[f"u{i}_loss"] = np.array(loss)
        d[f"u{i}_g"] = np.concatenate([g["W1"].ravel(), g["b1"], g["W2"], np.atleast_1d(g["b2"])])
        Xf = rng.normal(scale=50.0, size=(20, di))
        d[f"u{i}_Xf"] = Xf
        d[f"u{i}_f"] = pnn.forward(m, Xf)
    d["n_units"] = np.array(12)
    save("pnn", d)


BR_CASES = [
    # d, h, n, seed, estimate, alpha0, beta0, max_epochs, target
    (2, 1, 50, 5, True, 1e-12, 1.0, 1000, "sin"),
    (1, 1, 25, 0, True, 1e-12, 1.0, 1000, "lin"),
    (2, 2, 30, 1, True, 1e-12, 1.0, 1000, "prod"),
    (1, 1, 40, 2, True, 1e-12, 1.0, 1000, "noise"),
    (1, 1, 30, 3, False, 0.01, 1.0, 1000, "lin_noise"),
    (1, 1, 30, 3, False, 100.0, 1.0, 1000, "lin_noise"),
    (1, 1, 20, 1, False, 0.0, 1.0, 200, "lin_noise"),
    (2, 3, 30, 2, True, 1e-12, 1.0, 1000, "prod"),
    (1, 10, 40, 0, True, 1e-12, 1.0, 60, "sin"),
    (3, 1, 60, 9, True, 1e-12, 1.0, 1000, "sin"),
    (2, 1, 30, 4, True, 1e-12, 1.0, 1000, "const"),
    (4, 2, 45, 6, True, 1e-12, 1.0, 300, "sin"),
]


def _target(kind, X, rng):
    if kind == "sin":
        return np.sin(3.0 * X.sum(axis=1))
    if kind == "lin":
        return 2.0 * X[:, 0]
    if kind == "prod":
        return X[:, 0] * X[:, -1] + rng.normal(0.0, 0.05, len(X))
    if kind == "noise":
        return rng.normal(0.0, 1.0, len(X))
    if kind == "lin_noise":
        return 1.5 * X[:, 0] + rng.normal(0.0, 0.05, len(X))
    return np.full(len(X), 0.5)


def gen_br():
    d = {}
    rng = np.random.default_rng(77)
    for i, (di, h, n, seed, est, a0, b0, mx, tgt) in enumerate(BR_CASES):
        X = rng.uniform(0.0, 1.0, size=(n, di))
        y = _target(tgt, X, rng)
        m, hist = brbpnn.train(X, y, hidden=h, seed=seed, config=brbpnn.LmConfig(max_epochs=mx),
                               estimate_hyperparams=est, alpha0=a0, beta0=b0)
        d[f"c{i}_cfg"] = np.array([di, h, n, seed, int(est), mx], dtype=np.int64)
        d[f"c{i}_ab"] = np.array([a0, b0])
        d[f"c{i}_X"], d[f"c{i}_y"] = X, y
        d[f"c{i}_w"] = brbpnn.pack(m)
        d[f"c{i}_final_ab"] = np.array([m.alpha, m.beta])
        d[f"c{i}_hist"] = np.array([dataclasses.astuple(r) for r in hist], dtype=float).reshape(-1, 10)
        Xt = rng.uniform(-0.5, 1.5, size=(11, di))
        d[f"c{i}_Xt"] = Xt
        d[f"c{i}_pred"] = np.atleast_1d(brbpnn.forward(m, Xt))
    d["n_cases"] = np.array(len(BR_CASES))
    for i in range(10):
        di = int(rng.integers(1, 5))
        h = int(rng.integers(1, 5))
        m = brbpnn.init_model(di, hidden=h, rng=rng)
        m.alpha, m.beta = float(rng.uniform(1e-3, 1.0)), float(rng.uniform(0.5, 5.0))
        X = rng.uniform(-1.0, 1.5, size=(int(rng.integers(2, 12)), di))
        y = rng.uniform(-1.0, 1.0, size=len(X))
        J = brbpnn.jacobian(m, X)
        w = brbpnn.pack(m)
        r = brbpnn.forward(m, X) - y
        mu = float(10.0 ** rng.uniform(-4, 1))
        d[f"u{i}_dh"] = np.array([di, h])
        d[f"u{i}_w"], d[f"u{i}_X"], d[f"u{i}_y"] = w, X, y
        d[f"u{i}_ab_mu"] = np.array([m.alpha, m.beta, mu])
        d[f"u{i}_J"] = J
        d[f"u{i}_obj"] = np.array(brbpnn.objective(m, X, y))
        d[f"u{i}_delta"] = brbpnn.solve_damped(J, r, w, m.alpha, m.beta, mu)
        f, e_d, e_w = brbpnn.objective(m, X, y)
        up = brbpnn.evidence_update(e_d, e_w, J.T @ J, m.alpha, m.beta, len(y))
        d[f"u{i}_evid"] = np.array([up.alpha, up.beta, up.gamma, float(up.pinned)])
        d[f"u{i}_eig"] = np.linalg.eigvalsh(J.T @ J)
    d["n_units"] = np.array(10)
    save("brbpnn", d)


def _ref_series(key, X, y):
    return BbSeries(tuple(key), np.asarray(X, dtype=float), np.asarray(y, dtype=float))


def _family(name, axes):
    buf = io.StringIO()
    generate_dataset(family_by_name(name).program, GridSpec(axes), buf)
    buf.seek(0)
    return [(s.key, s.X, s.y) for s in ingest(buf)]


def gen_train_one():
    d = {}
    runs = []
    app = synth.app20()
    runs += [(s, "high-low", 0, 300, 1000) for s in app]
    runs += [(s, "random", 3, 40, 100) for s in app[:6]]
    runs += [(s, "mixed-high-low", 1, 25, 1000) for s in app[5:9]]
    lin = _family("linear", (tuple(range(1, 61)),))
    runs += [(s, "random", 0, 50, 1000) for s in lin]
    tri = _family("trilinear", (tuple(range(12, 19, 2)),) * 3)
    runs += [(s, "high-low", 0, 60, 1000) for s in tri[:3]]
    flat = (("flat", 0, 0), np.ones((6, 1)), np.arange(6, dtype=float))
    runs += [(flat, "high-low", 0, 10, 10)]
    mode_of = {"high-low": SplitMode.HIGH_LOW, "random": SplitMode.RANDOM,
               "mixed-high-low": SplitMode.MIXED_HIGH_LOW}
    i = 0
    for (key, X, y), mode, seed, pe, be in runs:
        for kind in ("pnn", "brbpnn"):
            cfg = ExperimentConfig(split_mode=mode_of[mode], seed=seed, pnn_epochs=pe,
                                   br_max_epochs=be)
            r = train_one(_ref_series(key, X, y), kind, cfg)
            p = f"r{i}_"
            d[p + "key"] = np.array([key[0], str(key[1]), str(key[2]), kind, mode])
            d[p + "cfg"] = np.array([seed, pe, be], dtype=np.int64)
            d[p + "X"], d[p + "y"] = X, y
            d[p + "error"] = np.array(r.error or "")
            d[p + "nn"] = np.array([r.n_train, r.n_test], dtype=np.int64)
            d[p + "flags"] = np.array([r.constant_target, r.pinned_hyperparams])
            if r.error is None:
                d[p + "mse"] = np.array(r.mse)
                d[p + "pred_raw"] = r.pred_raw
                sm = r.saved.model
                d[p + "w"] = np.concatenate([sm.W1.ravel(), sm.b1, sm.W2, [sm.b2]])
                d[p + "seed"] = np.array(words(r.saved.seed, 1), dtype=np.uint64)
                d[p + "corr"] = np.array([np.nan if r.pearson is None else r.pearson,
                                          np.nan if r.spearman is None else r.spearman])
                if kind == "brbpnn":
                    d[p + "br_meta"] = np.array([r.saved.config["epochs_run"],
                                                 r.saved.config["gamma"] or np.nan,
                                                 r.saved.config["mu"] or np.nan,
                                                 sm.alpha, sm.beta])
                # extrapolation through the persisted model
                raw = np.array(X, dtype=float)[::7] * 1.5
                d[p + "raw_q"] = raw
                d[p + "counts_q"] = r.saved.predict_counts(raw)
            i += 1
    d["n_runs"] = np.array(i)
    save("train_one", d)


def gen_experiment():
    """The reference's run_experiment artifacts (acceptance criterion 8's
    configuration -- linear family, grid n=1:60, high-low, both models, 60
    PNN / 100 BR epochs, seed 17 -- plus three more apps so the summary has
    several groups): summary.csv, report.csv, one model JSON / heatmap / kde
    file per kind, the splits manifest."""
    import tempfile
    from pathlib import Path

    from bbcount.experiment import run_experiment

    series = _family("linear", (tuple(range(1, 61)),))
    series += [(k, X, y) for k, X, y in synth.app20()[:4]]
    series += _family("trilinear", (tuple(range(12, 19, 2)),) * 3)[:2]
    ref_series = [_ref_series(k, X, y) for k, X, y in series]
    cfg = ExperimentConfig(split_mode=SplitMode.HIGH_LOW, fraction=0.7, seed=17, pnn_epochs=60,
                           br_max_epochs=100)
    d = {"n_series": np.array(len(series))}
    for i, (k, X, y) in enumerate(series):
        d[f"s{i}_key"] = np.array([k[0], str(k[1]), str(k[2])])
        d[f"s{i}_X"], d[f"s{i}_y"] = np.asarray(X, float), np.asarray(y, float)
    with tempfile.TemporaryDirectory() as tmp:
        run_experiment(ref_series, cfg, tmp)
        out = Path(tmp)
        files = ["summary.csv", "report.csv"]
        files += sorted(p.name for p in out.glob("splits_*.csv"))[:2]
        files += sorted(p.name for p in out.glob("heatmap_*.csv"))[:3]
        files += sorted(p.name for p in out.glob("kde_*.csv"))[:2]
        files += ["models/" + p.name for p in sorted((out / "models").glob("*.json"))[:4]]
        d["files"] = np.array(files)
        for j, f in enumerate(files):
            d[f"f{j}"] = np.array((out / f).read_text())
        d["all_files"] = np.array(sorted(str(p.relative_to(out)) for p in out.rglob("*") if p.is_file()))
    save("experiment", d)


def gen_families():
    """The reference's generate_dataset (CFG interpreter) on small grids of
    each builtin family, and on the app20 grid for the four families app20
    is made of: trace CSV text and the ingested series."""
    d = {}
    grids = {"linear": ((1, 2, 3, 7, 60),), "bilinear": ((1, 2, 5), (3, 4)),
             "trilinear": ((1, 3), (2, 5), (1, 4)), "triangular": ((1, 2, 9, 20),),
             "branchy": ((1, 7, 8, 9, 10, 33),)}
    for name, axes in grids.items():
        buf = io.StringIO()
        generate_dataset(family_by_name(name).program, GridSpec(axes), buf)
        d[f"{name}_csv"] = np.array(buf.getvalue())
    ax = tuple(range(2, 31, 2))
    for name, axes in (("bilinear", (ax, ax)), ("triangular", (ax,)), ("linear", (ax,)),
                       ("branchy", (ax,))):
        for key, X, y in _family(name, axes):
            d[f"app_{name}_{key[2]}_X"], d[f"app_{name}_{key[2]}_y"] = X, y
    save("families", d)


def gen_pnn_long():
    """Long-series PNN case (the bench's longest sequential chain): the first
    suite16 pathfinder series, random split 0.7 / seed 0 and the reference's
    normaliser, 4 epochs of pnn.train (761 minibatches each) with the
    series_seed the bench gives restart 0."""
    from bbcount.traces import SplitSpec, fit_normalizer, split

    key, X, y = next(s for s in synth.suite16(seed=0) if s[0][0] == "pathfinder")
    tr, te = split(_ref_series(key, X, y), SplitSpec(SplitMode.RANDOM, 0.7, 0))
    nm = fit_normalizer(tr)
    Xn, yn = nm.transform_features(tr.X), nm.transform_targets(tr.y)
    Xt = nm.transform_features(te.X)
    seed = series_seed(0, key, "pnn")
    d = {"X": Xn, "y": yn, "Xt": Xt, "seed": np.array(words(seed, 2), dtype=np.uint64),
         "epochs": np.array(4)}
    m, hist = pnn.train(Xn, yn, pnn.TrainConfig(epochs=4, seed=seed))
    d["w"] = np.concatenate([m.W1.ravel(), m.b1, m.W2, [m.b2]])
    d["hist"] = np.array(hist)
    d["pred"] = np.atleast_1d(pnn.forward(m, Xt))
    save("pnn_long", d)


if __name__ == "__main__":
    if sys.argv[1:] == ["pnn_long"]:
        gen_pnn_long()
        sys.exit(0)
    if sys.argv[1:] == ["experiment"]:
        gen_experiment()
        sys.exit(0)
    if sys.argv[1:] == ["families"]:
        gen_families()
        sys.exit(0)
    gen_families()
    gen_experiment()
    gen_pnn_long()
    gen_rng()
    gen_pnn()
    gen_br()
    gen_train_one()
