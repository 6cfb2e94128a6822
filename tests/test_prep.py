"""Batched split / normalise (prep.py) against the oracle's per-series
restatement of the reference's traces.py (CPU): labels, error texts and
normalised rows bit for bit, on many series at once and on the edge cases
the reference handles (empty series, one row, constant features, constant
targets, extreme fractions, negative parameters)."""

import numpy as np
import pytest

from oracle import bbml_oracle as O
from paper_2202_07798_b200 import prep, synth
from paper_2202_07798_b200.traces import (BbSeries, ConstantFeatureError, DegenerateSplitError,
                                          SplitMode, SplitSpec, classify, split)


def _series():
    out = [BbSeries(k, X, y) for k, X, y in synth.app20()]
    rng = np.random.default_rng(3)
    for i, n in enumerate((1, 2, 3, 7, 40)):
        d = 1 + i % 3
        out.append(BbSeries(("rnd", i, 0), rng.integers(-5, 9, size=(n, d)).astype(float),
                            rng.integers(0, 50, size=n).astype(float)))
    out.append(BbSeries(("flat", 0, 0), np.ones((6, 1)), np.arange(6.0)))
    out.append(BbSeries(("flat2", 0, 0), np.array([[1.0, 2.0], [3.0, 2.0], [5.0, 2.0]]), np.ones(3)))
    out.append(BbSeries(("const_y", 0, 0), np.arange(8.0).reshape(-1, 1), np.full(8, 4.0)))
    out.append(BbSeries(("empty", 0, 0), np.zeros((0, 2)), np.zeros(0)))
    return out


def _oracle(series, mode, fraction, seed):
    """Per-series reference semantics via the oracle restatement."""
    X, y = series.X, series.y
    if len(y) == 0:
        return "empty", None
    try:
        lab = O.split_labels(X, mode, fraction, seed)
    except ValueError:
        return "constant", None
    tr, te = np.flatnonzero(lab == 1), np.flatnonzero(lab == 2)
    if tr.size == 0 or te.size == 0:
        return ("empty train" if tr.size == 0 else "empty test"), lab
    nm = O.Norm.fit(X[tr], y[tr])
    return None, (lab, nm.fx(X[tr]), nm.fy(y[tr]), nm.fx(X[te]), nm.fy(y[te]), y[te])


@pytest.mark.parametrize("mode", ["random", "high-low", "mixed-high-low"])
@pytest.mark.parametrize("fraction", [0.02, 0.3, 0.7, 0.95])
def test_batched_prepare_matches_per_series_reference(mode, fraction):
    series = _series()
    t = prep.SeriesTable.from_series(series)
    P = prep.prepare(t, mode, fraction, 5)
    for i, s in enumerate(series):
        err, want = _oracle(s, mode, fraction, 5)
        if err is not None:
            assert i in P.errors, (s.key, err)
            text = P.errors[i]
            assert {"empty": "empty train partition (series is empty)"}.get(err, err) in text or \
                (err == "constant" and "are constant" in text), (s.key, err, text)
            continue
        assert i not in P.errors, (s.key, P.errors.get(i))
        lab, Xtr, ytr, Xte, yte, yraw = want
        a, b = P.tr_off[i], P.tr_off[i + 1]
        c, e = P.te_off[i], P.te_off[i + 1]
        d = s.X.shape[1]
        np.testing.assert_array_equal(P.labels[t.offsets[i]:t.offsets[i + 1]], lab)
        assert P.Xtr[a:b, :d].tobytes() == np.ascontiguousarray(Xtr).tobytes(), s.key
        assert P.ytr[a:b].tobytes() == ytr.tobytes(), s.key
        assert P.Xte[c:e, :d].tobytes() == np.ascontiguousarray(Xte).tobytes(), s.key
        assert P.yte[c:e].tobytes() == yte.tobytes(), s.key
        np.testing.assert_array_equal(P.yte_raw[c:e], yraw)
        assert not P.Xtr[a:b, d:].any() and not P.Xte[c:e, d:].any()


def test_single_series_api_raises_reference_errors():
    spec = SplitSpec(SplitMode.HIGH_LOW, 0.7, 0)
    with pytest.raises(ConstantFeatureError, match="are constant; range split undefined"):
        classify(BbSeries(("f", 0, 0), np.ones((4, 1)), np.arange(4.0)), spec)
    with pytest.raises(DegenerateSplitError, match=r"empty train partition \(series is empty\)"):
        split(BbSeries(("e", 0, 0), np.zeros((0, 1)), np.zeros(0)), spec)
    with pytest.raises(DegenerateSplitError) as ei:
        split(BbSeries(("one", 1, 2), np.array([[3.0]]), np.array([1.0])), SplitSpec(SplitMode.RANDOM, 0.7, 0))
    assert ei.value.partition == "test"
    assert str(ei.value) == "empty test partition (('one', 1, 2) under random)"
    s = BbSeries(("ok", 0, 0), np.arange(10.0).reshape(-1, 1), np.arange(10.0) ** 2)
    tr, te = split(s, spec)
    lab = classify(s, spec)
    assert list(lab).count("train") == len(tr) and list(lab).count("test") == len(te)
