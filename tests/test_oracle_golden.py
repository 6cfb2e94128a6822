"""Pin the CPU oracle against fixtures produced by running the reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import bbml_oracle as O
from oracle.rng import Pcg64, generate_u64

M64 = (1 << 64) - 1


def _seed(words):
    return int(words[0]) | (int(words[1]) << 64) if len(words) > 1 else int(words[0])


def test_pcg64_streams_match_reference(golden):
    g = golden("rng")
    for i, (lo, hi) in enumerate(zip(g["seeds_lo"], g["seeds_hi"])):
        seed = int(lo) | (int(hi) << 64)
        p = Pcg64(seed)
        st = g[f"s{i}_state"]
        assert p.state == int(st[0]) | (int(st[1]) << 64)
        assert p.inc == int(st[2]) | (int(st[3]) << 64)
        assert [p.uniform(-0.7, 0.7) for _ in range(20)] == list(g[f"s{i}_uniform"])
        assert p.uniform(-1.0, 1.0) == float(g[f"s{i}_scalar"])
        for n in (1, 2, 3, 7, 100, 1000):
            assert p.permutation(n) == list(g[f"s{i}_perm{n}"]), (seed, n)
        assert [p.uniform(0.0, 1.0) for _ in range(5)] == list(g[f"s{i}_tail_uniform"])


def test_series_seed_matches_reference(golden):
    for base, app_crc, k, b, kind_crc, want in golden("rng")["series_seed"]:
        got = generate_u64([int(base), int(app_crc), int(k), int(b), int(kind_crc)], 1)[0]
        assert got == int(want)


def test_numpy_generator_still_matches_fixture(golden):
    # guards the oracle's own use of numpy.random against a numpy upgrade
    g = golden("rng")
    r = np.random.default_rng(123)
    assert list(r.uniform(-0.7, 0.7, size=(10, 2)).ravel()) == list(g["s2_uniform"])


def test_pnn_oracle_matches_reference(golden):
    g = golden("pnn")
    for i in range(int(g["n_cases"])):
        d, h, n, ep, bs = (int(v) for v in g[f"c{i}_cfg"])
        w, hist = O.pnn_fit(g[f"c{i}_X"], g[f"c{i}_y"], d, h, ep, bs, float(g[f"c{i}_lr"]),
                            _seed(g[f"c{i}_seed"]))
        np.testing.assert_allclose(w, g[f"c{i}_w"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(hist, g[f"c{i}_hist"], rtol=1e-12)
        pred = O.pnn_rate(w, g[f"c{i}_Xt"], d, h)
        np.testing.assert_allclose(pred, g[f"c{i}_pred"], rtol=1e-12)


def test_pnn_units_match_reference(golden):
    g = golden("pnn")
    for i in range(int(g["n_units"])):
        d, h = (int(v) for v in g[f"u{i}_dh"])
        loss, grad = O.pnn_batch_grad(g[f"u{i}_w"], g[f"u{i}_X"], g[f"u{i}_y"], d, h)
        assert loss == pytest.approx(float(g[f"u{i}_loss"]), rel=1e-13)
        np.testing.assert_allclose(grad, g[f"u{i}_g"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(O.pnn_rate(g[f"u{i}_w"], g[f"u{i}_Xf"], d, h), g[f"u{i}_f"],
                                   rtol=1e-13)


def test_br_oracle_matches_reference(golden):
    g = golden("brbpnn")
    for i in range(int(g["n_cases"])):
        d, h, n, seed, est, mx = (int(v) for v in g[f"c{i}_cfg"])
        a0, b0 = (float(v) for v in g[f"c{i}_ab"])
        fit = O.br_fit(g[f"c{i}_X"], g[f"c{i}_y"], d, h, seed=seed, max_epochs=mx,
                       estimate=bool(est), alpha0=a0, beta0=b0)
        hist = np.array(fit.records, dtype=float).reshape(-1, 10)
        want = g[f"c{i}_hist"]
        assert hist.shape == want.shape, i
        np.testing.assert_allclose(fit.w, g[f"c{i}_w"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(hist, want, rtol=1e-9, atol=1e-12, equal_nan=True)
        np.testing.assert_allclose(O.br_out(fit.w, g[f"c{i}_Xt"], d, h), g[f"c{i}_pred"],
                                   rtol=1e-9, atol=1e-12)


def test_br_units_match_reference(golden):
    g = golden("brbpnn")
    for i in range(int(g["n_units"])):
        d, h = (int(v) for v in g[f"u{i}_dh"])
        w, X, y = g[f"u{i}_w"], g[f"u{i}_X"], g[f"u{i}_y"]
        alpha, beta, mu = (float(v) for v in g[f"u{i}_ab_mu"])
        J = O.br_jac(w, X, d, h)
        np.testing.assert_allclose(J, g[f"u{i}_J"], rtol=1e-14, atol=1e-15)
        e_d, e_w = O.br_energies(w, X, y, d, h)
        np.testing.assert_allclose([beta * e_d + alpha * e_w, e_d, e_w], g[f"u{i}_obj"], rtol=1e-13)
        r = O.br_out(w, X, d, h) - y
        np.testing.assert_allclose(O.br_step(J, r, w, alpha, beta, mu), g[f"u{i}_delta"],
                                   rtol=1e-10, atol=1e-13)
        ev = O.br_evidence(e_d, e_w, J.T @ J, alpha, beta, len(y))
        np.testing.assert_allclose(ev[:3], g[f"u{i}_evid"][:3], rtol=1e-10, atol=1e-13)


def test_train_one_oracle_matches_reference(golden):
    g = golden("train_one")
    for i in range(int(g["n_runs"])):
        p = f"r{i}_"
        app, k, b, kind, mode = (str(v) for v in g[p + "key"])
        seed, pe, be = (int(v) for v in g[p + "cfg"])
        if kind == "pnn" and pe > 100:
            continue  # long PNN runs are covered on the GPU side
        res = O.train_one((app, int(k), int(b)), g[p + "X"], g[p + "y"], kind, mode=mode,
                          base_seed=seed, pnn_epochs=pe, br_max_epochs=be)
        want_err = str(g[p + "error"])
        assert (res.error is not None) == bool(want_err), (i, res.error, want_err)
        if res.error is None:
            assert res.mse == pytest.approx(float(g[p + "mse"]), rel=1e-9, abs=1e-14)
            np.testing.assert_allclose(res.pred_raw, g[p + "pred_raw"], rtol=1e-9)
            assert res.seed == int(g[p + "seed"][0])


def test_pnn_oracle_matches_reference_long_series(golden):
    """The pathfinder-size case (7,604 training rows, 4 epochs = 3,044
    sequential Adam steps, the bench's longest chain) — pins the oracle's
    permutation stream and Adam at the long-series size."""
    g = golden("pnn_long")
    X, y = g["X"], g["y"]
    w, hist = O.pnn_fit(X, y, X.shape[1], 10, int(g["epochs"]), 10, 1e-4, _seed(g["seed"]))
    np.testing.assert_allclose(w, g["w"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(hist, g["hist"], rtol=1e-12, atol=0)


def test_oracle_metrics_reproduce_reference_correlations(golden):
    """Pearson / Spearman of the reference's own test predictions (golden
    pred_raw) vs the raw test counts give the reference's r*_corr exactly."""
    g = golden("train_one")
    checked = 0
    for i in range(int(g["n_runs"])):
        p = f"r{i}_"
        if str(g[p + "error"]) or len(g[p + "pred_raw"]) < 2:
            continue
        app, k, b, kind, mode = (str(v) for v in g[p + "key"])
        seed = int(g[p + "cfg"][0])
        lab = O.split_labels(g[p + "X"], mode, 0.7, seed)
        actual = g[p + "y"][lab == 2]
        for got, want in ((O.pearson(g[p + "pred_raw"], actual), g[p + "corr"][0]),
                          (O.spearman(g[p + "pred_raw"], actual), g[p + "corr"][1])):
            assert (got is None and np.isnan(want)) or got == float(want), (app, k, b, kind)
        checked += 1
    assert checked >= 60
