"""The reference's own unit-level known answers, asked of the drop-in API.

Each case restates one assertion from the reference suite
(`pkg/tests/test_pnn.py`, `pkg/tests/test_brbpnn.py`, cited per test) against
`paper_2202_07798_b200.pnn` / `.brbpnn`, whose unit functions run on the
device through `libbbml.so` (`units.cu`).  Host-only checks (input
validation, the scalar Poisson helpers) run on CPU; everything that reaches a
kernel is marked `gpu`.
"""
import math

import numpy as np
import pytest

from paper_2202_07798_b200 import brbpnn, pnn

gpu = pytest.mark.gpu


# ---------------------------------------------------------------- host side

def test_poisson_pmf_known_values_and_domain():
    # test_pnn.py:16-35
    assert pnn.poisson_pmf(1.0, 0) == pytest.approx(math.exp(-1.0), abs=1e-15)
    assert pnn.poisson_pmf(2.0, 2) == pytest.approx(2.0 * math.exp(-2.0), abs=1e-15)
    for lam in (0.5, 5.0, 20.0):
        assert sum(pnn.poisson_pmf(lam, j) for j in range(201)) == pytest.approx(1.0, abs=1e-9)
    assert 0.0 < pnn.poisson_pmf(150.0, 150) < 1.0
    for lam, j in ((0.0, 1), (-1.0, 1), (1.0, -2)):
        with pytest.raises(pnn.DomainError):
            pnn.poisson_pmf(lam, j)


def test_poisson_nll_known_values():
    # test_pnn.py:38-64
    assert pnn.poisson_nll(1.0, 0.0) == pytest.approx(1.0, abs=1e-12)
    assert pnn.poisson_nll(2.0, 3.0, eps=0.0) == pytest.approx(2.0 - 3.0 * math.log(2.0), abs=1e-15)
    got = pnn.poisson_nll(np.array([1.0, 2.0]), np.array([0.0, 3.0]), eps=0.0)
    assert got == pytest.approx((3.0 - 3.0 * math.log(2.0)) / 2.0, abs=1e-13)
    with pytest.raises(pnn.NumericError):
        pnn.poisson_nll(float("nan"), 1.0)
    with pytest.raises(pnn.NumericError):
        pnn.poisson_nll(1.0, float("inf"))


def test_shape_errors_raised_before_any_launch():
    # test_pnn.py:85-88 (arity); pnn.py:222-225 (empty / mismatched series)
    model = pnn.init_model(3, rng=np.random.default_rng(2))
    with pytest.raises(pnn.ShapeError):
        pnn.forward(model, np.zeros(2))
    with pytest.raises(pnn.ShapeError):
        pnn.train(np.zeros((0, 2)), np.zeros(0))
    with pytest.raises(pnn.ShapeError):
        pnn.train(np.zeros((4, 2)), np.zeros(3))


def test_init_draw_order_matches_reference_generator():
    # pnn.py:87-105 / brbpnn.py:63-82: W1, b1, W2 then the scalar b2
    m = pnn.init_model(2, hidden=10, rng=np.random.default_rng(11))
    rng = np.random.default_rng(11)
    a, c = 1 / math.sqrt(2), 1 / math.sqrt(10)
    np.testing.assert_array_equal(m.W1, rng.uniform(-a, a, size=(10, 2)))
    np.testing.assert_array_equal(m.b1, rng.uniform(-a, a, size=10))
    np.testing.assert_array_equal(m.W2, rng.uniform(-c, c, size=10))
    assert m.b2 == float(rng.uniform(-c, c))


# ---------------------------------------------------------------- PNN units

@gpu
def test_pnn_forward_zero_weights_give_log_two():
    # test_pnn.py:67-72
    model = pnn.PnnModel(W1=np.zeros((10, 2)), b1=np.zeros(10), W2=np.zeros(10), b2=0.0)
    assert pnn.forward(model, np.zeros(2)) == pytest.approx(math.log(2.0) + model.eps, abs=1e-12)


@gpu
def test_pnn_forward_positive_and_deterministic():
    # test_pnn.py:74-86
    rng = np.random.default_rng(0)
    model = pnn.init_model(2, rng=rng)
    X = rng.normal(scale=50.0, size=(200, 2))
    out = pnn.forward(model, X)
    assert np.all(np.isfinite(out)) and np.all(out > 0.0)
    x = np.array([0.3, -0.7])
    assert pnn.forward(model, x) == pnn.forward(model, x)


@gpu
def test_adam_first_step_zero_grad_and_nonfinite_block():
    # test_pnn.py:91-112
    params = {"w": np.array(0.0)}
    state = pnn.init_adam(params, learning_rate=1e-4)
    pnn.adam_step(state, params, {"w": np.array(1.0)})
    assert float(params["w"]) == pytest.approx(-1e-4 / (1.0 + 1e-8), rel=1e-9)

    params = {"w": np.array([1.0, -2.0])}
    state = pnn.init_adam(params)
    for _ in range(5):
        pnn.adam_step(state, params, {"w": np.zeros(2)})
    np.testing.assert_array_equal(params["w"], [1.0, -2.0])

    params = {"W1": np.array([0.0])}
    state = pnn.init_adam(params)
    with pytest.raises(pnn.NumericError) as err:
        pnn.adam_step(state, params, {"W1": np.array([float("nan")])})
    assert "W1" in str(err.value)


@gpu
def test_pnn_backprop_matches_finite_differences():
    # test_pnn.py:116-152 (central differences, rel 1e-4)
    rng = np.random.default_rng(42)
    step = 1e-5
    for _ in range(8):
        d = int(rng.integers(1, 4))
        model = pnn.init_model(d, hidden=5, rng=rng)
        X = rng.uniform(-1, 1.5, size=(int(rng.integers(2, 9)), d))
        y = rng.uniform(0, 1.5, size=len(X))
        _, grads = pnn.loss_and_grads(model, X, y)
        analytic = np.concatenate([np.ravel(grads[k]) for k in ("W1", "b1", "W2", "b2")])
        w = model.packed()
        numeric = np.empty_like(w)
        for i in range(w.size):
            wp, wm = w.copy(), w.copy()
            wp[i] += step
            wm[i] -= step
            lp, _ = pnn.loss_and_grads(pnn.PnnModel.from_packed(wp, d, 5), X, y)
            lm, _ = pnn.loss_and_grads(pnn.PnnModel.from_packed(wm, d, 5), X, y)
            numeric[i] = (lp - lm) / (2 * step)
        scale = np.maximum(np.abs(numeric), 1e-6)
        assert (np.abs(analytic - numeric) / scale).max() <= 1e-4


@gpu
def test_pnn_loss_identity_for_zero_targets():
    # test_pnn.py:154-159
    rng = np.random.default_rng(5)
    model = pnn.init_model(2, rng=rng)
    X = rng.uniform(0, 1, size=(9, 2))
    loss, _ = pnn.loss_and_grads(model, X, np.zeros(9))
    assert loss == pytest.approx(float(np.mean(pnn.forward(model, X))), rel=1e-12)


@gpu
def test_pnn_train_seeded_determinism_bit_identical():
    # test_pnn.py:163-172
    rng = np.random.default_rng(6)
    X = rng.uniform(0, 1, size=(40, 1))
    y = rng.uniform(0, 1, size=40)
    cfg = pnn.TrainConfig(epochs=20, seed=123)
    a, ha = pnn.train(X, y, cfg)
    b, hb = pnn.train(X, y, cfg)
    assert ha == hb
    np.testing.assert_array_equal(a.packed(), b.packed())


# ---------------------------------------------------------------- BR units

@gpu
def test_tansig_known_values():
    # test_brbpnn.py:15-33
    assert brbpnn.tansig(0.0) == 0.0
    assert brbpnn.tansig(1.0) == pytest.approx(2.0 / (1.0 + math.exp(-2.0)) - 1.0, abs=1e-15)
    assert brbpnn.tansig(1.0) == pytest.approx(0.761594, abs=1e-6)
    x = np.random.default_rng(7).uniform(-20, 20, size=1000)
    np.testing.assert_allclose(brbpnn.tansig(x), np.tanh(x), atol=1e-12)
    assert brbpnn.tansig(1e6) == 1.0 and brbpnn.tansig(-1e6) == -1.0


def _br(W1, W2, b2, alpha, beta):
    W1 = np.asarray(W1, dtype=float)
    return brbpnn.BrbpnnModel(W1=W1, b1=np.zeros(W1.shape[0]), W2=np.asarray(W2, dtype=float),
                              b2=b2, alpha=alpha, beta=beta)


@gpu
def test_objective_known_values():
    # test_brbpnn.py:36-65
    f, e_d, _ = brbpnn.objective(_br([[0.0]], [0.0], 0.5, 0.0, 1.0), np.array([[1.0], [2.0]]),
                                 np.array([0.5, 0.5]))
    assert f == 0.0 and e_d == 0.0
    f, _, e_w = brbpnn.objective(_br(np.zeros((1, 2)), [0.0], 0.0, 1.0, 0.0), np.ones((3, 2)),
                                 np.ones(3))
    assert e_w == 0.0 and f == 0.0
    model = _br([[0.3]], [-0.4], 0.0, 1.0, 2.0)
    X = np.array([[0.0]])
    y = np.array([brbpnn.forward(model, X)[0] + 0.5])
    f, e_d, e_w = brbpnn.objective(model, X, y)
    assert e_d == pytest.approx(0.25, abs=1e-15)
    assert e_w == pytest.approx(0.25, abs=1e-15)
    assert f == pytest.approx(0.75, abs=1e-14)


@gpu
def test_jacobian_matches_finite_differences():
    # test_brbpnn.py:68-93
    rng = np.random.default_rng(21)
    step = 1e-6
    for _ in range(10):
        d, h = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        model = brbpnn.init_model(d, hidden=h, rng=rng)
        X = rng.uniform(-1, 1.5, size=(int(rng.integers(2, 7)), d))
        J = brbpnn.jacobian(model, X)
        w = brbpnn.pack(model)
        numeric = np.empty_like(J)
        for i in range(w.size):
            wp, wm = w.copy(), w.copy()
            wp[i] += step
            wm[i] -= step
            brbpnn.unpack(model, wp)
            plus = brbpnn.forward(model, X)
            brbpnn.unpack(model, wm)
            minus = brbpnn.forward(model, X)
            numeric[:, i] = (plus - minus) / (2 * step)
        brbpnn.unpack(model, w)
        scale = np.maximum(np.abs(numeric), 1e-6)
        assert (np.abs(J - numeric) / scale).max() <= 1e-4


@gpu
def test_gauss_newton_step_exact_for_linear_residuals():
    # test_brbpnn.py:97-106
    rng = np.random.default_rng(3)
    X = np.column_stack([np.ones(12), rng.uniform(0, 5, 12)])
    y = 3.0 - 2.0 * X[:, 1] + rng.normal(0, 0.3, 12)
    w = np.zeros(2)
    delta = brbpnn.solve_damped(X, X @ w - y, w, alpha=0.0, beta=1.0, mu=1e-12)
    optimum, *_ = np.linalg.lstsq(X, y, rcond=None)
    np.testing.assert_allclose(w + delta, optimum, rtol=1e-8, atol=1e-9)


@gpu
def test_rejected_trial_keeps_weights_and_grows_mu():
    # test_brbpnn.py:108-121
    model = _br([[0.0]], [0.0], 0.25, 0.0, 1.0)
    X, y = np.array([[0.0], [1.0]]), np.array([0.25, 0.25])
    state = brbpnn.LmState(mu=0.005)
    before = brbpnn.pack(model).copy()
    assert not brbpnn.lm_trial(model, state, X, y, brbpnn.LmConfig())
    np.testing.assert_array_equal(brbpnn.pack(model), before)
    assert state.mu == pytest.approx(0.05)


@gpu
def test_accepted_trial_strictly_decreases_objective():
    # test_brbpnn.py:123-133
    model = brbpnn.init_model(1, hidden=1, rng=np.random.default_rng(5))
    X = np.linspace(0, 1, 15).reshape(-1, 1)
    y = 1.5 * X.ravel() + 0.25
    state = brbpnn.LmState(mu=0.005)
    f_before, _, _ = brbpnn.objective(model, X, y)
    assert brbpnn.lm_step(model, state, X, y, brbpnn.LmConfig())
    f_after, _, _ = brbpnn.objective(model, X, y)
    assert f_after < f_before


@gpu
def test_stall_returns_false_past_mu_max():
    # test_brbpnn.py:135-145
    model = _br([[0.0]], [0.0], 0.0, 0.0, 1.0)
    state = brbpnn.LmState(mu=0.005)
    assert not brbpnn.lm_step(model, state, np.array([[0.0], [1.0]]), np.zeros(2),
                              brbpnn.LmConfig())
    assert state.mu > brbpnn.LmConfig().mu_max


@gpu
def test_evidence_gamma_bounds_and_pinning():
    # test_brbpnn.py:149-174
    rng = np.random.default_rng(6)
    for _ in range(40):
        n, p = int(rng.integers(2, 20)), int(rng.integers(1, 8))
        J = rng.normal(size=(n, p))
        upd = brbpnn.evidence_update(float(rng.uniform(0.01, 5)), float(rng.uniform(0.01, 5)),
                                     J.T @ J, float(rng.uniform(1e-6, 10)),
                                     float(rng.uniform(1e-6, 10)), n)
        assert 0.0 <= upd.gamma <= p
    J = np.ones((4, 2))
    upd = brbpnn.evidence_update(1.0, 0.0, J.T @ J, 1.0, 1.0, 4)
    assert upd.pinned and upd.alpha == brbpnn.HYPER_MAX
    upd = brbpnn.evidence_update(0.0, 1.0, J.T @ J, 1.0, 1.0, 4)
    assert upd.pinned and upd.beta == brbpnn.HYPER_MAX
