"""Synthetic basic-block count workloads (bench and test inputs).

The reference generates counts by interpreting parametric CFGs
(``cfg.py:271-313``) whose closed-form oracles are exact
(``families.py:75-165``, acceptance criterion 1).  Trace generation is out of
the hot-path scope, so the workloads here are built
directly from closed-form count formulas:

* ``app20``   — SURVEY §8d config 1/2: one 2-input app with five kernels
  (bilinear, triangular, linear, branchy, straight-line) = 20 BB series over
  the grid n, m in 2..30 step 2 (225 samples per series).
* ``suite16`` — config 3: 16 apps shaped like PAPER.md Table 1 (inputs, BBs,
  samples/series = samples / BBs), polynomial count surfaces.
* ``sweep``   — config 4: many app20-shaped apps with varied coefficients.

Series are returned as ``(key, X, y)`` with ``X`` float64 (n, d) raw
parameters and ``y`` float64 raw counts, ordered by key like
``traces.group_series`` (traces.py:182-188).
"""

from __future__ import annotations

import itertools
from typing import Iterator

import numpy as np

BRANCHY_THRESHOLD = 8

# (name, #inputs, #BBs, #BB samples)
TABLE1 = (
    ("2mm", 4, 21, 11505),
    ("atax", 2, 21, 25865),
    ("bicg", 2, 21, 27281),
    ("covariance", 2, 54, 9595),
    ("correlation", 2, 135, 5020),
    ("doitgen", 3, 13, 6009),
    ("gemm", 3, 10, 81219),
    ("gesummv", 1, 10, 9998),
    ("lu", 1, 31, 4347),
    ("gramschmit", 1, 83, 3117),
    ("syrk", 2, 15, 9900),
    ("mvt", 1, 21, 8189),
    ("gaussian", 1, 36, 2070),
    ("lud", 1, 11, 2052),
    ("nw", 1, 21, 3357),
    ("pathfinder", 3, 6, 65171),
)


def _app20_counts(n: np.ndarray, m: np.ndarray, coef=(1, 1, 1, 1)) -> list[np.ndarray]:
    """Per-BB counts of the five-kernel app; ``coef`` scales the loops."""
    a, b, c, e = coef
    one = np.ones_like(n)
    nn, mm = a * n, b * m
    tri = c * n
    br = e * n
    bigger = br > BRANCHY_THRESHOLD
    return [
        # kernel 0: bilinear nest over (n, m)
        one, nn * (mm + 1), nn * mm, nn, one,
        # kernel 1: triangular nest over n
        one, tri * (tri + 3) // 2, tri * (tri + 1) // 2, tri, one,
        # kernel 2: linear loop over m
        one, mm + 1, mm, one,
        # kernel 3: branchy loop guarded by n > threshold
        one, np.where(bigger, br + 1, 0), np.where(bigger, br, 0), np.where(bigger, 0, 1), one,
        # kernel 4: straight-line block
        one,
    ]


_APP20_KEYS = [(0, b) for b in range(5)] + [(1, b) for b in range(5)] + \
              [(2, b) for b in range(4)] + [(3, b) for b in range(5)] + [(4, 0)]


def app20(name: str = "app20", axis=tuple(range(2, 31, 2)), coef=(1, 1, 1, 1)):
    grid = np.array(list(itertools.product(axis, axis)), dtype=np.int64)
    counts = _app20_counts(grid[:, 0], grid[:, 1], coef)
    X = grid.astype(float)
    return [((name, k, b), X, np.asarray(c, dtype=float)) for (k, b), c in zip(_APP20_KEYS, counts)]


def _unique_points(rng: np.random.Generator, d: int, count: int) -> np.ndarray:
    """``count`` distinct integer parameter vectors in a d-dim box."""
    side = max(2, int(np.ceil(count ** (1.0 / d) * 1.6)))
    pts: set = set()
    out = []
    while len(out) < count:
        cand = rng.integers(1, side + 1, size=(count, d))
        for row in map(tuple, cand):
            if row not in pts:
                pts.add(row)
                out.append(row)
                if len(out) == count:
                    break
    arr = np.array(sorted(out), dtype=np.int64)
    return arr


def _poly_counts(rng: np.random.Generator, P: np.ndarray) -> np.ndarray:
    """A random non-negative integer count surface over the parameters."""
    n, d = P.shape
    shape = rng.integers(0, 6)
    if shape == 0:
        return np.ones(n, dtype=np.int64)  # entry/exit-like constant block
    terms = np.full(n, int(rng.integers(0, 4)), dtype=np.int64)
    dims = rng.permutation(d)
    if shape in (1, 2):  # linear
        terms += int(rng.integers(1, 4)) * P[:, dims[0]]
    elif shape == 3:  # product of two (or square)
        j = dims[1] if d > 1 else dims[0]
        terms += int(rng.integers(1, 3)) * P[:, dims[0]] * P[:, j]
    elif shape == 4:  # triangular
        q = P[:, dims[0]]
        terms += q * (q + 1) // 2
    else:  # branchy: zero below a threshold
        q = P[:, dims[0]]
        thr = int(np.median(q))
        terms = np.where(q > thr, terms + q, 0)
    if d > 2 and shape == 3 and rng.integers(0, 2):
        terms *= P[:, dims[2]]
    return terms


def suite16(seed: int = 0, scale: float = 1.0):
    """Config 3: 509 series over 16 Table-1-shaped apps."""
    rng = np.random.default_rng(seed)
    series = []
    for name, d, bbs, samples in TABLE1:
        per = max(8, int(round(samples * scale / bbs)))
        P = _unique_points(rng, d, per)
        X = P.astype(float)
        for b in range(bbs):
            y = _poly_counts(rng, P).astype(float)
            series.append(((name, 0, b), X, y))
    series.sort(key=lambda s: s[0])
    return series


def suite16_hidden(app: str) -> int:
    """BR hidden size per app: 10 for gramschmit, else 1."""
    return 10 if app == "gramschmit" else 1


def sweep(n_apps: int, seed: int = 0) -> Iterator:
    """Config 4: ``n_apps`` app20-shaped apps with varied loop scales."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_apps):
        coef = tuple(int(c) for c in rng.integers(1, 4, size=4))
        out.extend(app20(f"sweep{i:05d}", coef=coef))
    return out


# ---------------------------------------------------------------------------
# The reference's five builtin families (families.py:64-165) as vectorised
# closed-form counts, and its trace-CSV dataset format (families.py:330-362,
# traces.py header): SURVEY §8f f4.  The reference interprets each family's
# CFG program once per grid point (3.3 s for a 343-point trilinear grid); the
# counts below are the same integers for every grid point at once, and the
# writer emits the reference's file byte for byte.
# ---------------------------------------------------------------------------

# name -> (parameter names, blocks of kernel 0)
FAMILIES = {
    "linear": (("n",), 4),
    "bilinear": (("n", "m"), 5),
    "trilinear": (("n", "m", "kk"), 5),
    "triangular": (("n",), 5),
    "branchy": (("n",), 5),
}


def family_counts(name: str, P: np.ndarray) -> np.ndarray:
    """(points, blocks) int64 execution counts of kernel 0's blocks at the
    parameter rows ``P`` (points, arity)."""
    P = np.asarray(P, dtype=np.int64)
    one = np.ones(len(P), dtype=np.int64)
    if name == "linear":
        n = P[:, 0]
        cols = [one, n + 1, n, one]
    elif name == "bilinear":
        n, m = P[:, 0], P[:, 1]
        cols = [one, n * (m + 1), n * m, n, one]
    elif name == "trilinear":
        n, m, k = P[:, 0], P[:, 1], P[:, 2]
        cols = [one, n * m * (k + 1), n * m * k, n * m, one]
    elif name == "triangular":
        n = P[:, 0]
        cols = [one, n * (n + 3) // 2, n * (n + 1) // 2, n, one]
    elif name == "branchy":
        n = P[:, 0]
        big = n > BRANCHY_THRESHOLD
        cols = [one, np.where(big, n + 1, 0), np.where(big, n, 0), np.where(big, 0, 1), one]
    else:
        raise KeyError(f"unknown family {name!r}")
    return np.stack(cols, axis=1)


def grid_points(axes) -> np.ndarray:
    """itertools.product order of the per-parameter value tuples (GridSpec)."""
    return np.array(list(itertools.product(*axes)), dtype=np.int64).reshape(-1, len(axes))


def generate_dataset(name: str, axes, out) -> int:
    """Write the family's trace CSV over the grid (the reference's
    ``generate_dataset`` format: header app,kernel_id,bb_id,p0..,count, one
    row per (grid point, block) in grid order, blocks ascending).  ``out``:
    path or text stream.  Returns the number of rows."""
    P = grid_points(axes)
    C = family_counts(name, P)
    nb = C.shape[1]
    params = [",".join(map(str, row)) for row in P.tolist()]
    head = "app,kernel_id,bb_id," + ",".join(f"p{i}" for i in range(P.shape[1])) + ",count\n"
    lines = [f"{name},0,{b},{params[i]},{C[i, b]}\n" for i in range(len(P)) for b in range(nb)]
    text = head + "".join(lines)
    if isinstance(out, (str, bytes)) or hasattr(out, "__fspath__"):
        with open(out, "w", encoding="utf-8", newline="") as fh:
            fh.write(text)
    else:
        out.write(text)
    return len(lines)


def family_series(name: str, axes):
    """The series the reference's ingest of that dataset yields: one per
    block, key (name, 0, b), X = grid points, y = counts (key order)."""
    P = grid_points(axes)
    C = family_counts(name, P).astype(float)
    X = P.astype(float)
    return [((name, 0, b), X, C[:, b].copy()) for b in range(C.shape[1])]
