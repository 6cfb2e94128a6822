"""Device parity: CUDA kernels (through the drop-in API / C-ABI) against the
golden fixtures produced by the reference and against the CPU oracle.

Tolerances:
  PNN FP64 kernel  : weights and predictions <= 1e-12 relative (1e-15 abs floor)
  PNN FP32 kernel  : predictions <= 1e-3 relative (north-star gate)
  BR h <= 3        : predictions <= 1e-6 relative, same history length +-2 epochs
  initial weights  : bit-identical (device PCG64 == NumPy PCG64)
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2202_07798_b200 import brbpnn, engine, pnn  # noqa: E402
from oracle import bbml_oracle as O  # noqa: E402


def _seed(words):
    return int(words[0]) | (int(words[1]) << 64)


def _rel(a, b, floor=1e-15):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def test_device_init_bit_identical_to_numpy():
    # BR with max_epochs = 0 returns the initial weights untouched (all paths:
    # hidden-1 warp, P <= 32 warp, P <= 8, wide CTA kernel at P = 321)
    for seed in (0, 5, 2**63 + 3):
        for d, h in ((2, 10), (1, 1), (4, 7), (3, 64)):
            rng = np.random.default_rng(seed)
            want = O.init_flat(rng, d, h)
            X = np.random.default_rng(1).uniform(size=(5, d))
            y = np.zeros(5)
            model, hist = brbpnn.train(X, y, hidden=h, seed=seed, config=brbpnn.LmConfig(max_epochs=0))
            assert hist == []
            np.testing.assert_array_equal(brbpnn.pack(model), want)


def test_pnn_fp64_matches_reference_golden(golden):
    g = golden("pnn")
    for i in range(int(g["n_cases"])):
        d, h, n, ep, bs = (int(v) for v in g[f"c{i}_cfg"])
        cfg = pnn.TrainConfig(epochs=ep, batch_size=bs, learning_rate=float(g[f"c{i}_lr"]),
                              seed=_seed(g[f"c{i}_seed"]), hidden=h)
        model, hist = pnn.train(g[f"c{i}_X"], g[f"c{i}_y"], cfg)
        w = model.packed()
        assert _rel(w, g[f"c{i}_w"]) <= 1e-11, (i, _rel(w, g[f"c{i}_w"]))
        assert _rel(hist, g[f"c{i}_hist"]) <= 1e-12, i
        pred = pnn.forward(model, g[f"c{i}_Xt"])
        assert _rel(pred, g[f"c{i}_pred"]) <= 1e-11, i


def test_pnn_fp32_predictions_within_gate(golden):
    g = golden("pnn")
    old = pnn.PRECISION
    pnn.PRECISION = 32
    try:
        for i in range(int(g["n_cases"])):
            d, h, n, ep, bs = (int(v) for v in g[f"c{i}_cfg"])
            cfg = pnn.TrainConfig(epochs=ep, batch_size=bs, learning_rate=float(g[f"c{i}_lr"]),
                                  seed=_seed(g[f"c{i}_seed"]), hidden=h)
            model, _ = pnn.train(g[f"c{i}_X"], g[f"c{i}_y"], cfg)
            pred = pnn.forward(model, g[f"c{i}_Xt"])
            assert _rel(pred, g[f"c{i}_pred"]) <= 1e-3, (i, _rel(pred, g[f"c{i}_pred"]))
    finally:
        pnn.PRECISION = old


def test_pnn_long_series_matches_reference_golden(golden):
    """Pathfinder-size PNN (7,604 rows: the long-series kernel with one
    producer warp per model, the uint16 permutation double buffer at its
    largest and the epoch-boundary stream rewind) against the reference's own
    run: FP64 history <= 1e-12, weights <= 1e-11; FP32 predictions <= 1e-3."""
    g = golden("pnn_long")
    cfg = pnn.TrainConfig(epochs=int(g["epochs"]), seed=_seed(g["seed"]))
    model, hist = pnn.train(g["X"], g["y"], cfg)
    assert _rel(hist, g["hist"]) <= 1e-12, _rel(hist, g["hist"])
    assert _rel(model.packed(), g["w"]) <= 1e-11, _rel(model.packed(), g["w"])
    assert _rel(pnn.forward(model, g["Xt"]), g["pred"]) <= 1e-11
    old = pnn.PRECISION
    pnn.PRECISION = 32
    try:
        m32, _ = pnn.train(g["X"], g["y"], cfg)
    finally:
        pnn.PRECISION = old
    assert _rel(pnn.forward(m32, g["Xt"]), g["pred"]) <= 1e-3


def test_br_matches_reference_golden(golden):
    g = golden("brbpnn")
    worst = {}
    for i in range(int(g["n_cases"])):
        d, h, n, seed, est, mx = (int(v) for v in g[f"c{i}_cfg"])
        a0, b0 = (float(v) for v in g[f"c{i}_ab"])
        model, hist = brbpnn.train(g[f"c{i}_X"], g[f"c{i}_y"], hidden=h, seed=seed,
                                   config=brbpnn.LmConfig(max_epochs=mx), estimate_hyperparams=bool(est),
                                   alpha0=a0, beta0=b0)
        want = g[f"c{i}_hist"]
        pred = brbpnn.forward(model, g[f"c{i}_Xt"])
        worst[i] = (_rel(pred, g[f"c{i}_pred"], 1e-12), len(hist), len(want))
    print(worst)
    for i, (err, nh, nw) in worst.items():
        h = int(g[f"c{i}_cfg"][1])
        if h <= 3:
            assert err <= 1e-6, (i, err)
            # early stop = 5 epochs with (gamma, E_D, E_W) all within 1e-7
            # relative: a knife edge (the reference's own 1-ulp
            # spread shifts it by up to 2 epochs for h = 1)
            assert abs(nh - nw) <= (2 if h == 1 else 5), (i, nh, nw)
        else:
            # hidden >= 10 (P = 31 here: the tridiagonal-form warp path):
            # predictions within max(1e-3, 25 x the reference's own 1-ulp
            # spread, measured by the oracle on its inputs moved by one ulp)
            d, _, n, seed, est, mx = (int(v) for v in g[f"c{i}_cfg"])
            X, y, Xt = g[f"c{i}_X"], g[f"c{i}_y"], g[f"c{i}_Xt"]
            spread = 0.0
            if err > 1e-3:
                for Xp, yp in ((X, np.nextafter(y, np.inf)), (X, np.nextafter(y, -np.inf)),
                               (np.nextafter(X, np.inf), y)):
                    f = O.br_fit(Xp, yp, d, h, seed=seed, max_epochs=mx)
                    spread = max(spread, _rel(O.br_out(f.w, Xt, d, h), g[f"c{i}_pred"], 1e-12))
                print(f"golden BR case {i} (h={h}): device {err:.2e}, reference 1-ulp spread {spread:.2e}")
            assert err <= max(1e-3, 25 * spread), (i, err, spread)
            assert nh == nw or (nh < mx and nw < mx), (i, nh, nw)


def test_forward_matches_golden(golden):
    g = golden("pnn")
    for i in range(int(g["n_units"])):
        d, h = (int(v) for v in g[f"u{i}_dh"])
        m = pnn.PnnModel.from_packed(g[f"u{i}_w"], d, h)
        assert _rel(pnn.forward(m, g[f"u{i}_Xf"]), g[f"u{i}_f"]) <= 1e-13


def test_loss_and_grads_match_golden(golden):
    g = golden("pnn")
    for i in range(int(g["n_units"])):
        d, h = (int(v) for v in g[f"u{i}_dh"])
        m = pnn.PnnModel.from_packed(g[f"u{i}_w"], d, h)
        loss, gr = pnn.loss_and_grads(m, g[f"u{i}_X"], g[f"u{i}_y"])
        flat = np.concatenate([gr["W1"].ravel(), gr["b1"], gr["W2"], np.atleast_1d(gr["b2"])])
        assert loss == pytest.approx(float(g[f"u{i}_loss"]), rel=1e-12)
        np.testing.assert_allclose(flat, g[f"u{i}_g"], rtol=1e-10, atol=1e-14)


def test_br_units_match_golden(golden):
    g = golden("brbpnn")
    for i in range(int(g["n_units"])):
        d, h = (int(v) for v in g[f"u{i}_dh"])
        w, X, y = g[f"u{i}_w"], g[f"u{i}_X"], g[f"u{i}_y"]
        alpha, beta, mu = (float(v) for v in g[f"u{i}_ab_mu"])
        m = brbpnn.BrbpnnModel(*[None] * 4, alpha=alpha, beta=beta)
        m.W1 = np.zeros((h, d))
        brbpnn.unpack(m, w.copy())
        J = brbpnn.jacobian(m, X)
        np.testing.assert_allclose(J, g[f"u{i}_J"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(brbpnn.objective(m, X, y), g[f"u{i}_obj"], rtol=1e-12)
        r = brbpnn.forward(m, X) - y
        delta = brbpnn.solve_damped(J, r, w, alpha, beta, mu)
        np.testing.assert_allclose(delta, g[f"u{i}_delta"], rtol=1e-8, atol=1e-12)
        f, e_d, e_w = brbpnn.objective(m, X, y)
        up = brbpnn.evidence_update(e_d, e_w, J.T @ J, alpha, beta, len(y))
        np.testing.assert_allclose([up.alpha, up.beta, up.gamma], g[f"u{i}_evid"][:3], rtol=1e-9,
                                   atol=1e-12)


def test_br_wide_first_epoch_and_gamma_within_reference_self_spread():
    """P > 32 (wide CTA kernel) and the P <= 32 tridiagonal path.  The LM step
    of epoch 0 is deterministic and must match; gamma depends on the
    eps*||J'J|| noise of near-null eigenvalues (rank-deficient J'J, alpha0 =
    1e-12), so it is gated by the reference's OWN 1-ulp spread (SURVEY §8c:
    the reference moves by >1e-3 under 1-ulp target perturbations at h >= 10)."""
    for d, h, n in ((2, 12, 40), (2, 10, 40), (1, 40, 30), (2, 64, 300), (2, 64, 60)):
        X = np.random.default_rng(n + d).uniform(0, 1, size=(n, d))
        y = np.sin(3 * X.sum(axis=1))
        fit = O.br_fit(X, y, d, h, seed=3, max_epochs=1)
        ulp = O.br_fit(X, np.nextafter(y, np.inf), d, h, seed=3, max_epochs=1)
        _, hist = brbpnn.train(X, y, hidden=h, seed=3, config=brbpnn.LmConfig(max_epochs=1))
        r_o, r_d = fit.records[0], hist[0]
        assert _rel([r_d.f_before, r_d.f_after, r_d.e_d, r_d.e_w], r_o[1:5]) <= 1e-9, (d, h, n)
        # noise envelope of equally valid eigen-solvers on the same J'J (LAPACK
        # syevd / syevr, squared singular values of J, einsum-formed J'J)
        import scipy.linalg as sl

        J = O.br_jac(fit.w, X, d, h)
        P = J.shape[1]

        def gam(lam):
            s = np.clip(lam, 0, None)
            return float(np.sum(s / (s + 1e-12)))

        sv = np.linalg.svd(J, compute_uv=False)
        env = [r_o[7], gam(sl.eigh(J.T @ J, eigvals_only=True, driver="evr")),
               gam(np.concatenate([sv ** 2, np.zeros(max(0, P - len(sv)))])),
               gam(np.linalg.eigvalsh(np.einsum("ki,kj->ij", J, J)))]
        spread = abs(r_o[7] - ulp.records[0][7])
        lo, hi = min(env) - 25 * spread - 1e-9 * P, max(env) + 25 * spread + 1e-9 * P
        assert lo <= r_d.gamma <= hi, (d, h, n, r_d.gamma, env, spread)


def _spread_gate(label, items, data, kw, oracle_pred, floors):
    """For fits beyond 1e-3: device error <= 25 x the oracle's own 1-ulp
    spread (oracle.pool.self_spread), which must itself exceed 1e-3 / 25."""
    from oracle.pool import self_spread

    for key, e in items:
        X, y = data[key]
        spread = self_spread(key, X, y, "brbpnn", kw, oracle_pred[key], floors[key])
        print(f"{label} {key}: device {e:.2e}, oracle 1-ulp spread {spread:.2e}")
        assert spread * 25 >= 1e-3 and e <= 25 * spread, (key, e, spread)


def test_br_hidden10_parity_gramschmit_1000_epochs():
    """The near-chaotic hidden-10 fits (the 83 gramschmit series of suite16,
    random split, the bench's 1000 epochs) through the drop-in
    experiment.train_many: predicted counts <= max(1e-3, 25 x the oracle's
    own 1-ulp spread) per series, accuracy within +-0.5 pp."""
    from paper_2202_07798_b200 import synth
    from paper_2202_07798_b200.experiment import ExperimentConfig, train_many
    from paper_2202_07798_b200.traces import BbSeries, SplitMode
    from oracle.pool import oracle_map, rel

    raw = [s for s in synth.suite16(seed=0) if s[0][0] == "gramschmit"]
    series = [BbSeries(k, X, y) for k, X, y in raw]
    cfg = ExperimentConfig(split_mode=SplitMode.RANDOM, seed=0, br_hidden=10, br_max_epochs=1000,
                           models=("brbpnn",))
    res = train_many([(s, "brbpnn") for s in series], cfg).results
    kw = dict(mode="random", base_seed=0, br_hidden=10, br_max_epochs=1000)
    ora = oracle_map([(k, X, y, "brbpnn", kw, None) for k, X, y in raw])
    floors = {k: 1e-6 * max(1.0, float(np.max(np.abs(y)))) for k, X, y in raw}
    beyond = []
    for (k, X, y), r, o in zip(raw, res, ora):
        assert r.error is None and o.error is None, (k, r.error, o.error)
        e = rel(r.pred_raw, o.pred_raw, floors[k])
        if e > 1e-3:
            beyond.append((k, e))
    by = {k: (X, y) for k, X, y in raw}
    _spread_gate("gramschmit h=10", beyond, by, kw, {k: o.pred_raw for (k, _, _), o in zip(raw, ora)},
                 floors)
    acc_dev = 100 * (1 - float(np.mean([r.mse for r in res])))
    acc_ora = 100 * (1 - float(np.mean([o.mse for o in ora])))
    print("gramschmit h=10 accuracy device %.3f oracle %.3f, beyond 1e-3: %d" % (acc_dev, acc_ora, len(beyond)))
    assert abs(acc_dev - acc_ora) <= 0.5


def test_train_one_matches_reference_golden(golden):
    """experiment.train_one / train_many (batched device path) against the
    reference's own train_one on the same series: errors, flags, split sizes,
    MSE and raw predictions (PNN FP64 <= 1e-9; BR hidden 1 <= 1e-6), seeds and
    predict_counts extrapolation through the saved model."""
    from paper_2202_07798_b200.experiment import ExperimentConfig, train_many
    from paper_2202_07798_b200.traces import BbSeries, SplitMode

    g = golden("train_one")
    modes = {"high-low": SplitMode.HIGH_LOW, "random": SplitMode.RANDOM,
             "mixed-high-low": SplitMode.MIXED_HIGH_LOW}
    groups = {}
    for i in range(int(g["n_runs"])):
        p = f"r{i}_"
        app, k, b, kind, mode = (str(v) for v in g[p + "key"])
        seed, pe, be = (int(v) for v in g[p + "cfg"])
        groups.setdefault((mode, seed, pe, be), []).append((i, (app, int(k), int(b)), kind))
    checked = 0
    for (mode, seed, pe, be), items in groups.items():
        cfg = ExperimentConfig(split_mode=modes[mode], seed=seed, pnn_epochs=pe, br_max_epochs=be)
        series = {}
        pairs = []
        for i, key, kind in items:
            p = f"r{i}_"
            s = series.setdefault(key, BbSeries(key, g[p + "X"], g[p + "y"]))
            pairs.append((s, kind))
        results = train_many(pairs, cfg).results
        for (i, key, kind), r in zip(items, results):
            p = f"r{i}_"
            want_err = str(g[p + "error"])
            assert (r.error or "") == want_err or (r.error and want_err), (key, kind, r.error, want_err)
            if want_err:
                assert r.error is not None
                continue
            assert r.error is None, (key, kind, r.error)
            assert [r.n_train, r.n_test] == list(g[p + "nn"])
            assert [r.constant_target, r.pinned_hyperparams] == list(g[p + "flags"]), (key, kind)
            assert r.saved.seed == int(g[p + "seed"][0])
            tol = 1e-9 if kind == "pnn" else 1e-6
            # relative error with a floor at 1e-6 of the series' count scale
            # (predictions of a count that is 0 on the test side are ~1e-9)
            floor = 1e-6 * max(1.0, float(np.max(np.abs(g[p + "y"]))))
            e = _rel(r.pred_raw, g[p + "pred_raw"], floor)
            if kind == "brbpnn" and float(g[p + "br_meta"][4]) >= 1e12 and e > tol:
                # degenerate fit: E_D -> 0 drives beta to its 1e12 clamp and the
                # damped system to condition ~1e24, so late epochs amplify
                # rounding (a step target fitted by a saturating tanh).  Gate
                # at max(1e-3, 25 x the reference's own 1-ulp spread), the
                # spread measured here by re-running the oracle (bit-identical
                # to the reference) on its normalised training data moved by
                # one ulp (oracle.PERTURBATIONS).
                from oracle.pool import self_spread

                spread = self_spread(key, g[p + "X"], g[p + "y"], kind,
                                     dict(mode=mode, base_seed=seed, pnn_epochs=pe, br_max_epochs=be),
                                     g[p + "pred_raw"], floor)
                print(f"beta-clamped {key}: device {e:.2e}, reference 1-ulp spread {spread:.2e}")
                assert e <= max(1e-3, 25 * spread), (key, kind, e, spread)
                checked += 1
                continue
            assert _rel(r.pred_raw, g[p + "pred_raw"], floor) <= tol, (key, kind)
            assert abs(r.mse - float(g[p + "mse"])) <= tol * max(1.0, abs(float(g[p + "mse"]))), (key, kind)
            got = r.saved.predict_counts(g[p + "raw_q"])
            assert _rel(got, g[p + "counts_q"], floor) <= tol, (key, kind)
            # device Pearson / Spearman (experiment.py:150-152): Pearson against
            # the reference's value; Spearman against the oracle on the device's
            # own predictions (saturated fits predict exactly tied values, so
            # 1e-16 prediction differences move ranks by 1/2) and against the
            # reference's value when its predictions have no ties
            pw, sw = (float(v) for v in g[p + "corr"])
            assert (r.pearson is None) == np.isnan(pw), (key, kind, r.pearson, pw)
            if r.pearson is not None:
                assert abs(r.pearson - pw) <= 1e-6, (key, kind, r.pearson, pw)
            so = O.spearman(r.pred_raw, r.actual_raw)
            assert (r.spearman is None) == (so is None), (key, kind, r.spearman, so)
            if so is not None:
                assert abs(r.spearman - so) <= 1e-12, (key, kind, r.spearman, so)
                if len(np.unique(g[p + "pred_raw"])) == len(g[p + "pred_raw"]):
                    assert abs(r.spearman - sw) <= 1e-6, (key, kind, r.spearman, sw)
            checked += 1
    assert checked >= 60


def test_learning_curves_batched_match_oracle(tmp_path):
    """a whole learning-curve sweep (series x kinds x
    fractions) in one batched call.  Every point equals the single-task
    device result bit for bit (models are independent), matches the oracle's
    train_one on the same random split (PNN FP64 / BR hidden 1: accuracy
    within 1e-6 pp), and skipped points (degenerate splits) agree."""
    import json

    from paper_2202_07798_b200 import synth
    from paper_2202_07798_b200.experiment import (ExperimentConfig, learning_curves, run_sweep,
                                                   train_one)
    from paper_2202_07798_b200.metrics import accuracy_percent
    from paper_2202_07798_b200.traces import BbSeries, SplitMode

    raw = synth.app20()[:3]
    series = [BbSeries(k, X, y) for k, X, y in raw]
    fr = (0.02, 0.1, 0.3, 0.5, 0.7, 0.9)
    seed = 5
    cfg = ExperimentConfig(pnn_epochs=40, br_max_epochs=60)
    curves = learning_curves(series, ("pnn", "brbpnn"), fr, seed, cfg)
    assert len(curves) == 6
    n_pts = 0
    for s in series:
        for kind in ("pnn", "brbpnn"):
            pts = curves[(s.key, kind)]
            assert [p.fraction for p in pts] == list(fr)
            for p in pts:
                o = O.train_one(s.key, s.X, s.y, kind, mode="random", fraction=p.fraction,
                                base_seed=seed, pnn_epochs=40, br_max_epochs=60)
                if o.error is not None:
                    assert p.skipped, (s.key, kind, p.fraction, o.error)
                    continue
                assert not p.skipped, (s.key, kind, p.fraction)
                assert abs(p.accuracy - accuracy_percent(o.mse)) <= 1e-6, (s.key, kind, p.fraction)
                n_pts += 1
            single = train_one(s, kind, ExperimentConfig(**{**cfg.__dict__, "split_mode": SplitMode.RANDOM,
                                                            "fraction": 0.7, "seed": seed}))
            assert single.accuracy == pts[fr.index(0.7)].accuracy
    assert n_pts >= 24
    n = run_sweep(series, cfg, tmp_path, fr, seed)
    assert n == 6
    man = json.loads((tmp_path / "sweep_manifest.json").read_text())
    assert man["curves"] == 6 and man["fractions"] == sorted(fr)
    assert len(list(tmp_path.glob("curve_*.csv"))) == 6


def test_br_wide_parity_hidden64_1000_epochs():
    """BASELINE cfg 5 (hidden 64, P = 257) on the device's wide path at the
    bench's 1000 epochs, ten app20 series (HighLow split, 100 training rows):
    predicted counts <= max(1e-3, 25 x the oracle's own 1-ulp spread) per
    series, accuracy within the north-star +-0.5 pp."""
    from paper_2202_07798_b200 import synth
    from paper_2202_07798_b200.experiment import ExperimentConfig, train_many
    from paper_2202_07798_b200.traces import BbSeries, SplitMode
    from oracle.pool import oracle_map, rel

    raw = synth.app20()[:10]
    series = [BbSeries(k, X, y) for k, X, y in raw]
    cfg = ExperimentConfig(split_mode=SplitMode.HIGH_LOW, seed=0, br_hidden=64, br_max_epochs=1000,
                           models=("brbpnn",))
    res = train_many([(s, "brbpnn") for s in series], cfg).results
    kw = dict(mode="high-low", base_seed=0, br_hidden=64, br_max_epochs=1000)
    ora = oracle_map([(k, X, y, "brbpnn", kw, None) for k, X, y in raw])
    floors = {k: 1e-6 * max(1.0, float(np.max(np.abs(y)))) for k, X, y in raw}
    dev, orc, beyond = [], [], []
    for (k, X, y), r, o in zip(raw, res, ora):
        assert (r.error is None) == (o.error is None), (k, r.error, o.error)
        if r.error is None:
            dev.append(r.mse)
            orc.append(o.mse)
            e = rel(r.pred_raw, o.pred_raw, floors[k])
            if e > 1e-3:
                beyond.append((k, e))
    assert len(dev) >= 8
    by = {k: (X, y) for k, X, y in raw}
    _spread_gate("hidden 64", beyond, by, kw, {k: o.pred_raw for (k, _, _), o in zip(raw, ora)}, floors)
    acc_dev = 100 * (1 - float(np.mean(dev)))
    acc_ora = 100 * (1 - float(np.mean(orc)))
    print("hidden-64 accuracy device %.3f oracle %.3f, beyond 1e-3: %d" % (acc_dev, acc_ora, len(beyond)))
    assert abs(acc_dev - acc_ora) <= 0.5


def test_br_hidden1_long_series_multiwarp():
    """Hidden-1 fits with n >= 2048 training rows run one model per CTA of 4
    warps (sample passes split over warps, reduced in warp order); against
    the oracle's train_one on the same random split: predictions <= 1e-6
    relative, or max(1e-3, 25 x the oracle's own 1-ulp spread) for a
    beta-clamped degenerate fit (as in test_train_one_matches_reference_golden)."""
    from paper_2202_07798_b200 import synth
    from paper_2202_07798_b200.experiment import ExperimentConfig, train_many
    from paper_2202_07798_b200.traces import BbSeries, SplitMode

    raw = synth.app20(axis=tuple(range(1, 65)))[:4]
    series = [BbSeries(k, X, y) for k, X, y in raw]
    cfg = ExperimentConfig(split_mode=SplitMode.RANDOM, seed=1, br_max_epochs=300,
                           models=("brbpnn",))
    res = train_many([(s, "brbpnn") for s in series], cfg).results
    for (k, X, y), r in zip(raw, res):
        o = O.train_one(k, X, y, "brbpnn", mode="random", base_seed=1, br_max_epochs=300)
        assert r.error is None and o.error is None, (k, r.error, o.error)
        assert r.n_train == o.n_train and r.n_train >= 2048
        floor = 1e-6 * max(1.0, float(np.max(np.abs(y))))
        e = _rel(r.pred_raw, o.pred_raw, floor)
        if e <= 1e-6:
            continue
        # beyond 1e-6: max(1e-3, 25 x the oracle's own 1-ulp spread)
        from oracle.pool import self_spread

        spread = self_spread(k, X, y, "brbpnn", dict(mode="random", base_seed=1, br_max_epochs=300),
                             o.pred_raw, floor)
        print(f"multi-warp {k}: device {e:.2e}, oracle 1-ulp spread {spread:.2e}")
        assert e <= max(1e-3, 25 * spread), (k, e, spread)


def test_device_metrics_match_oracle():
    """bbml_metrics / bbml_pooled_metrics / bbml_heatmaps
    against the oracle's restatement of metrics.py (bit-identical to the
    reference, tests/test_oracle_golden.py): MSE in the normalised space,
    Pearson / Spearman (tie-averaged ranks) of de-normalised predictions,
    undefined -> NaN; random and tie-heavy vectors, constants, n = 1, and test
    sets beyond the shared-memory sort (counting-rank path); pooled groups;
    heatmap edges bit-identical and counts equal."""
    from paper_2202_07798_b200 import engine

    rng = np.random.default_rng(4)
    sizes = [1, 2, 3, 7, 50, 333, 1000, 4096, 5000, 9000]
    preds, an, ar, norms = [], [], [], []
    for k, n in enumerate(sizes):
        p = rng.normal(size=n)
        a = rng.normal(size=n)
        if k % 3 == 1:
            p = np.round(p, 1)  # ties
            a = np.round(a * 2) / 2
        if k == 2:
            a = np.full(n, 0.25)  # constant actual -> undefined correlations
        lo, hi = rng.uniform(-5, 5), rng.uniform(6, 50)
        preds.append(p)
        an.append(a)
        ar.append(np.round(a * (hi - lo) + lo, 3))
        norms.append([0.0, 1.0, lo, hi])
    off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    nn = np.array(sizes, np.int32)
    ones = np.ones(len(sizes), np.int32)
    out = engine.metrics(np.concatenate(preds), np.concatenate(an), np.concatenate(ar), off, off, nn,
                         ones, np.array(norms))
    for k, n in enumerate(sizes):
        p, a, raw = preds[k], an[k], ar[k]
        lo, hi = norms[k][2], norms[k][3]
        want_mse = float(np.mean((p - a) ** 2))
        assert abs(out[k, 0] - want_mse) <= 1e-12 * max(1.0, want_mse)
        assert out[k, 3] == 1.0
        if n < 2:
            assert np.isnan(out[k, 1]) and np.isnan(out[k, 2])
            continue
        pr = p * (hi - lo) + lo
        for col, ref in ((1, O.pearson(pr, raw)), (2, O.spearman(pr, raw))):
            if ref is None:
                assert np.isnan(out[k, col]), (n, col)
            else:
                assert abs(out[k, col] - ref) <= 1e-12, (n, col, out[k, col], ref)
    # pooled groups (experiment.summarize): groups 0 = sizes[3:6], 1 = sizes[6:], 2 = sizes[:3]
    grp = np.array([2, 2, 2, 0, 0, 0, 1, 1, 1, 1], np.int32)
    pooled = engine.pooled_metrics(grp, np.concatenate(preds), np.concatenate(ar), off, off, nn, ones,
                                   np.array(norms))
    for gi in range(3):
        ks = [k for k in range(len(sizes)) if grp[k] == gi]
        pr = np.concatenate([preds[k] * (norms[k][3] - norms[k][2]) + norms[k][2] for k in ks])
        raw = np.concatenate([ar[k] for k in ks])
        for col, ref in ((0, O.pearson(pr, raw)), (1, O.spearman(pr, raw))):
            assert (np.isnan(pooled[gi, col]) if ref is None else abs(pooled[gi, col] - ref) <= 1e-12), \
                (gi, col, pooled[gi, col], ref)
    # heatmaps of |de-normalised prediction| vs |raw|: edges bit-identical, counts equal
    P = [np.abs(p) for p in preds]
    A = [np.abs(r) for r in ar]
    edges, counts = engine.heatmaps(np.concatenate(P), np.concatenate(A), off, off, nn, ones,
                                    np.tile([0.0, 1.0, 0.0, 1.0], (len(sizes), 1)), 32)
    for k in range(len(sizes)):
        e, c = O.heatmap(P[k], A[k], 32)
        assert edges[k].tobytes() == e.tobytes(), k
        np.testing.assert_array_equal(counts[k], c)


def test_br_units_wide_hidden64():
    """solve_damped / evidence_update at P = 257 (hidden 64, the wide unit
    kernel: J'J and the workspace in a global slab) against the oracle's
    numpy restatement (LAPACK dgesv / dsyevd)."""
    rng = np.random.default_rng(11)
    d, h, n = 2, 64, 300
    P = h * (d + 2) + 1
    m = brbpnn.init_model(d, hidden=h, rng=rng)
    m.alpha, m.beta = 0.01, 2.0
    X = rng.uniform(0, 1, size=(n, d))
    y = np.sin(3 * X.sum(axis=1))
    J = brbpnn.jacobian(m, X)
    w = brbpnn.pack(m)
    r = brbpnn.forward(m, X) - y
    delta = brbpnn.solve_damped(J, r, w, m.alpha, m.beta, 0.5)
    want = O.br_step(J, r, w, m.alpha, m.beta, 0.5)
    np.testing.assert_allclose(delta, want, rtol=1e-8, atol=1e-12)
    f, e_d, e_w = brbpnn.objective(m, X, y)
    up = brbpnn.evidence_update(e_d, e_w, J.T @ J, m.alpha, m.beta, n)
    ref = O.br_evidence(e_d, e_w, J.T @ J, m.alpha, m.beta, n)
    assert abs(up.gamma - ref[2]) <= 1e-6 * P, (up.gamma, ref[2])
