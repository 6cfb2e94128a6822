"""Batched data preparation: split, train-only min-max normalisation and CSR
packing of EVERY series of a run in a handful of whole-array NumPy passes.

This is the host stage in front of the kernels (the
reference's ``traces.classify`` / ``split`` 218-263 and ``Normalizer`` /
``fit_normalizer`` 271-324, applied per series inside ``train_one``,
experiment.py:105-116).  Instead of one Python call chain per series, the raw
rows of all series live in one CSR table (``SeriesTable``) and each step is
a segmented array operation:

* random split: the reference shuffles each series with
  ``default_rng(spec.seed).permutation(n)`` — the same seed for every
  series, so the permutation depends only on ``n``: one draw per distinct
  length, scattered into all series of that length;
* range splits: per-series feature min / max by ``minimum.reduceat``,
  thresholds ``min + fraction * (max - min)`` broadcast back to the rows,
  LOW / HIGH as row-wise all() over the series' own columns;
* normaliser: min / max of the train rows per series (``reduceat`` over the
  train-packed block), then the reference's elementwise maps
  ``(x - min) / span`` (constant dimension -> 0) on every row at once —
  the same IEEE operations per element, so values are bit-identical to the
  per-series path.

Row order inside a series is preserved (the reference takes
``flatnonzero(labels == ...)``, i.e. ascending row index), which fixes the
minibatch contents the permutation stream indexes into.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

TRAIN, TEST, DISCARD = 1, 2, 0


@dataclass
class SeriesTable:
    """Raw rows of many series: ``X (N, dmax)`` (columns >= d[s] are 0),
    ``y (N,)``, series s owns rows ``offsets[s]:offsets[s+1]``."""

    keys: list
    X: np.ndarray
    y: np.ndarray
    offsets: np.ndarray
    d: np.ndarray

    @classmethod
    def from_series(cls, series: Sequence) -> "SeriesTable":
        n = np.array([len(s.y) for s in series], dtype=np.int64)
        d = np.array([s.X.shape[1] for s in series], dtype=np.int32)
        off = np.zeros(len(series) + 1, dtype=np.int64)
        np.cumsum(n, out=off[1:])
        dmax = int(d.max(initial=1))
        if len(series) and (d == dmax).all():  # one arity: a single concatenation
            X = np.concatenate([np.asarray(s.X, dtype=float) for s in series]).reshape(-1, dmax)
        else:
            X = np.zeros((int(off[-1]), dmax))
            for s, (a, b) in zip(series, zip(off[:-1], off[1:])):
                X[a:b, :s.X.shape[1]] = s.X
        y = np.concatenate([np.asarray(s.y, dtype=float) for s in series]) if len(series) else np.zeros(0)
        return cls([s.key for s in series], X, y, off, d)

    @property
    def n(self) -> np.ndarray:
        return np.diff(self.offsets)

    def row_series(self) -> np.ndarray:
        return np.repeat(np.arange(len(self.keys)), self.n)


def _seg_reduce(ufunc, A: np.ndarray, starts: np.ndarray, counts: np.ndarray, fill: float) -> np.ndarray:
    """ufunc.reduceat over row segments; empty segments get ``fill``."""
    out = np.full((len(starts),) + A.shape[1:], fill)
    nz = counts > 0
    if nz.any() and len(A):
        out[nz] = ufunc.reduceat(A, starts[nz], axis=0)
    return out


def split_labels(t: SeriesTable, mode: str, fraction: float, seed: int):
    """Label every row TRAIN / TEST / DISCARD; returns ``(labels, errors)``
    with ``errors[s]`` the reference's error text for series that cannot be
    split (empty series, constant feature in a range mode, empty side)."""
    if not 0.0 < fraction < 1.0:
        raise ValueError(f"fraction must be in (0, 1), got {fraction}")
    n = t.n
    labels = np.zeros(len(t.y), dtype=np.int8)
    errors: dict = {}
    for s in np.flatnonzero(n == 0):
        errors[int(s)] = "empty train partition (series is empty)"
    if mode == "random":
        for length in np.unique(n[n > 0]):
            perm = np.random.default_rng(seed).permutation(int(length))
            cut = math.ceil(fraction * int(length))
            local = np.empty(int(length), dtype=np.int8)
            local[perm[:cut]] = TRAIN
            local[perm[cut:]] = TEST
            starts = t.offsets[:-1][n == length]
            labels[(starts[:, None] + np.arange(length)[None, :]).ravel()] = np.tile(local, len(starts))
    else:
        starts = t.offsets[:-1]
        lo = _seg_reduce(np.minimum, t.X, starts, n, 0.0)
        hi = _seg_reduce(np.maximum, t.X, starts, n, 0.0)
        own = np.arange(t.X.shape[1])[None, :] < t.d[:, None]          # (S, dmax)
        const = (hi <= lo) & own
        for s in np.flatnonzero(const.any(axis=1) & (n > 0)):
            errors[int(s)] = (f"features {np.flatnonzero(const[s]).tolist()} are constant; "
                              f"range split undefined for {t.keys[s]}")
        # padded columns get theta = +inf for LOW (x <= inf) and -inf for
        # HIGH (x > -inf), so the row-wise all() only sees the series' own
        theta = lo + fraction * (hi - lo)
        tlo = np.repeat(np.where(own, theta, np.inf), n, axis=0)
        thi = np.repeat(np.where(own, theta, -np.inf), n, axis=0)
        low = t.X[:, 0] <= tlo[:, 0]
        high = t.X[:, 0] > thi[:, 0]
        for k in range(1, t.X.shape[1]):  # column-wise all(): D <= 16 passes
            low &= t.X[:, k] <= tlo[:, k]
            high &= t.X[:, k] > thi[:, k]
        labels[high] = TEST
        if mode == "high-low":
            labels[low & ~high] = TRAIN
        elif mode == "mixed-high-low":
            labels[~high] = TRAIN
        else:
            raise ValueError(f"unknown split mode {mode!r}")
    S = len(t.keys)
    # per-series label counts: prefix sums of the train / test indicators at the segment ends
    ends = t.offsets
    ctr = np.concatenate([[0], np.cumsum(labels == TRAIN)])[ends]
    cte = np.concatenate([[0], np.cumsum(labels == TEST)])[ends]
    counts = np.zeros((S, 3), dtype=np.int64)
    counts[:, TRAIN] = np.diff(ctr)
    counts[:, TEST] = np.diff(cte)
    for s in np.flatnonzero((counts[:, TRAIN] == 0) | (counts[:, TEST] == 0)):
        s = int(s)
        if s not in errors:
            side = "train" if counts[s, TRAIN] == 0 else "test"
            errors[s] = f"empty {side} partition ({t.keys[s]} under {mode})"
    return labels, errors


@dataclass
class Prepared:
    """Split + normalised rows of every series, train and test packed in
    series order; ``ok`` lists the series that prepared without error."""

    table: SeriesTable
    labels: np.ndarray
    errors: dict
    ok: np.ndarray
    x_min: np.ndarray           # (S, dmax) train-split statistics
    x_max: np.ndarray
    y_min: np.ndarray           # (S,)
    y_max: np.ndarray
    tr_off: np.ndarray          # (S+1,) train rows of series s: tr_off[s]:tr_off[s+1]
    te_off: np.ndarray
    Xtr: np.ndarray             # normalised (N_train, dmax)
    ytr: np.ndarray
    Xte: np.ndarray
    yte: np.ndarray
    yte_raw: np.ndarray
    Xte_raw: np.ndarray = field(default=None)

    def norm_rows(self, dmax: Optional[int] = None) -> np.ndarray:
        """(S, 2 dmax + 2) rows [x_min(d), x_max(d), y_min, y_max] (device layout)."""
        D = self.table.X.shape[1] if dmax is None else dmax
        S = len(self.table.keys)
        out = np.zeros((S, 2 * D + 2))
        d = self.table.d.astype(np.int64)
        W = self.x_min.shape[1]
        col = np.arange(W)[None, :]
        own = col < d[:, None]
        rows = np.repeat(np.arange(S), W).reshape(S, W)
        out[rows[own], col.repeat(S, 0)[own]] = self.x_min[own]
        out[rows[own], (col + d[:, None])[own]] = self.x_max[own]
        out[np.arange(S), 2 * d] = self.y_min
        out[np.arange(S), 2 * d + 1] = self.y_max
        return out


def _normalise(X, y, counts, x_min, x_max, y_min, y_max, own):
    """Traces.py Normalizer.transform_* on every row: (v - min) / span with
    span -> 1 then 0 output for constant (and padded) dimensions.  Per-series
    constants are expanded once (np.repeat over the segment lengths)."""
    span = x_max - x_min
    live = (span > 0) & own
    safe = np.where(live, span, 1.0)
    lo = np.where(live, x_min, 0.0)
    Xn = X - np.repeat(lo, counts, axis=0)
    Xn /= np.repeat(safe, counts, axis=0)
    np.copyto(Xn, 0.0, where=~np.repeat(live, counts, axis=0))
    ys = y_max - y_min
    ylive = ys > 0
    yn = y - np.repeat(np.where(ylive, y_min, 0.0), counts)
    yn /= np.repeat(np.where(ylive, ys, 1.0), counts)
    np.copyto(yn, 0.0, where=~np.repeat(ylive, counts))
    return Xn, yn


def prepare(t: SeriesTable, mode: str, fraction: float, seed: int) -> Prepared:
    """Split every series, fit each normaliser on its train rows, normalise
    train and test rows (experiment.py:105-116 for all series at once)."""
    labels, errors = split_labels(t, mode, fraction, seed)
    S = len(t.keys)
    bad = np.zeros(S, dtype=bool)
    bad[list(errors)] = True
    rs = np.repeat(np.arange(S), t.n)
    use = ~bad[rs]
    tr_rows = np.flatnonzero(use & (labels == TRAIN))
    te_rows = np.flatnonzero(use & (labels == TEST))
    ntr = np.bincount(rs[tr_rows], minlength=S) if S else np.zeros(0, np.int64)
    nte = np.bincount(rs[te_rows], minlength=S) if S else np.zeros(0, np.int64)
    tr_off = np.zeros(S + 1, dtype=np.int64)
    te_off = np.zeros(S + 1, dtype=np.int64)
    np.cumsum(ntr, out=tr_off[1:])
    np.cumsum(nte, out=te_off[1:])
    Xtr_raw, ytr_raw = t.X[tr_rows], t.y[tr_rows]
    x_min = _seg_reduce(np.minimum, Xtr_raw, tr_off[:-1], ntr, 0.0)
    x_max = _seg_reduce(np.maximum, Xtr_raw, tr_off[:-1], ntr, 0.0)
    y_min = _seg_reduce(np.minimum, ytr_raw, tr_off[:-1], ntr, 0.0)
    y_max = _seg_reduce(np.maximum, ytr_raw, tr_off[:-1], ntr, 0.0)
    own = np.arange(t.X.shape[1])[None, :] < t.d[:, None]
    Xtr, ytr = _normalise(Xtr_raw, ytr_raw, ntr, x_min, x_max, y_min, y_max, own)
    Xte_raw, yte_raw = t.X[te_rows], t.y[te_rows]
    Xte, yte = _normalise(Xte_raw, yte_raw, nte, x_min, x_max, y_min, y_max, own)
    ok = np.flatnonzero(~bad)
    return Prepared(t, labels, errors, ok, x_min, x_max, y_min, y_max, tr_off, te_off,
                    Xtr, ytr, Xte, yte, yte_raw, Xte_raw)
