"""Synthetic workloads against the reference's CFG interpreter (CPU):
the vectorised closed-form family counts and the trace-CSV writer reproduce
the reference's ``generate_dataset`` byte for byte, and app20 (SURVEY §8d
config 1 / 2) is exactly bilinear(n, m) + triangular(n) + linear(m) +
branchy(n) + a straight-line block on the n, m = 2..30 step 2 grid
(tests/golden/families.npz, made by running the reference)."""

import io

import numpy as np
import pytest

from paper_2202_07798_b200 import synth

GRIDS = {"linear": ((1, 2, 3, 7, 60),), "bilinear": ((1, 2, 5), (3, 4)),
         "trilinear": ((1, 3), (2, 5), (1, 4)), "triangular": ((1, 2, 9, 20),),
         "branchy": ((1, 7, 8, 9, 10, 33),)}


@pytest.mark.parametrize("name", sorted(GRIDS))
def test_generate_dataset_byte_identical_to_reference(golden, name):
    buf = io.StringIO()
    rows = synth.generate_dataset(name, GRIDS[name], buf)
    want = str(golden("families")[f"{name}_csv"])
    assert buf.getvalue() == want
    assert rows == want.count("\n") - 1


def test_app20_is_the_reference_families_on_its_grid(golden):
    g = golden("families")
    app = {key[1:]: (X, y) for key, X, y in synth.app20()}
    parts = [("bilinear", 0, 5, slice(0, 2)), ("triangular", 1, 5, slice(0, 1)),
             ("linear", 2, 4, slice(1, 2)), ("branchy", 3, 5, slice(0, 1))]
    for name, kernel, blocks, cols in parts:
        for b in range(blocks):
            X, y = app[(kernel, b)]
            Xf, yf = g[f"app_{name}_{b}_X"], g[f"app_{name}_{b}_y"]
            # app20 rows are the (n, m) product; the family row for (n, m) is
            # the one with the same value(s) on the family's own parameters
            lut = {tuple(r): v for r, v in zip(Xf.tolist(), yf.tolist())}
            for row, v in zip(X[:, cols].tolist(), y.tolist()):
                assert lut[tuple(row)] == v, (name, b, row)
    np.testing.assert_array_equal(app[(4, 0)][1], 1.0)
    assert len(app) == 20


def test_family_series_match_reference_ingest(golden):
    g = golden("families")
    ax = tuple(range(2, 31, 2))
    for name, axes in (("bilinear", (ax, ax)), ("linear", (ax,)), ("branchy", (ax,))):
        for key, X, y in synth.family_series(name, axes):
            np.testing.assert_array_equal(X, g[f"app_{name}_{key[2]}_X"])
            np.testing.assert_array_equal(y, g[f"app_{name}_{key[2]}_y"])
