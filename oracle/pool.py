"""TEST INFRASTRUCTURE ONLY — run the CPU oracle's train_one over many tasks in a
infrastructure: the checker for the GPU parity tests, never the product).
One BLAS thread per worker; longest tasks first."""

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def _task(job):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import bbml_oracle as O

    key, X, y, kind, kw, perturb = job
    return O.train_one(key, X, y, kind, perturb=perturb or None, **kw)


def oracle_map(jobs):
    """jobs: (key, X, y, kind, train_one kwargs, perturbation or None)."""
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    cost = [len(j[1]) * (30 if j[3] == "pnn" else (j[4].get("br_hidden", 1) ** 2)) for j in jobs]
    order = sorted(range(len(jobs)), key=lambda i: -cost[i])
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
        res = dict(zip(order, pool.map(_task, [jobs[i] for i in order], chunksize=1)))
    return [res[i] for i in range(len(jobs))]


def rel(a, b, floor):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def self_spread(key, X, y, kind, kw, base_pred, floor):
    """The oracle's own 1-ulp spread for one fit: max relative change of its
    predicted counts over the PERTURBATIONS of its normalised training data."""
    from oracle import bbml_oracle as O

    runs = oracle_map([(key, X, y, kind, kw, p) for p in O.PERTURBATIONS])
    return max(rel(r.pred_raw, base_pred, floor) for r in runs)
