"""Batched device engine: packs many independent models into task tables,
moves the CSR training data to HBM and calls the C-ABI kernels.

All compute happens in ``libbbml.so``; PyTorch is used only for device
memory and the current CUDA stream.  There is no CPU fallback: without a
CUDA device every entry point raises ``DeviceUnavailable``.

Data layout in HBM:
  X  float64 [N_rows, x_stride]  row-major, x_stride = max inputs in the batch
  y  float64 [N_rows]
  each model = a contiguous row range [row_begin, row_begin + n)
  weights float64, pack order W1|b1|W2|b2 per model at w_offset
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import LM_TASK, PNN_TASK, PRED_TASK, STATUS, check, lib, ptr


def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise _lib.DeviceUnavailable(
            "no CUDA device: paper_2202_07798_b200 runs only on the GPU (no CPU fallback)")
    lib()
    return torch


def n_params(d, h):
    return np.asarray(h) * (np.asarray(d) + 2) + 1


@dataclass
class Packed:
    """CSR pack of per-model row blocks (host side)."""
    X: np.ndarray            # (N, stride) float64
    y: np.ndarray            # (N,) float64
    row_begin: np.ndarray    # (M,) int64
    n: np.ndarray            # (M,) int32
    d: np.ndarray            # (M,) int32

    @property
    def stride(self) -> int:
        return int(self.X.shape[1])


def pack(Xs: Sequence[np.ndarray], ys: Optional[Sequence[np.ndarray]] = None) -> Packed:
    d = np.array([np.atleast_2d(x).shape[1] for x in Xs], dtype=np.int32)
    n = np.array([len(np.atleast_2d(x)) for x in Xs], dtype=np.int32)
    stride = max(1, int(d.max(initial=1)))
    rb = np.zeros(len(Xs), dtype=np.int64)
    if len(Xs):
        rb[1:] = np.cumsum(n[:-1], dtype=np.int64)
    N = int(n.sum())
    X = np.zeros((max(N, 1), stride), dtype=np.float64)
    y = np.zeros(max(N, 1), dtype=np.float64)
    for i, x in enumerate(Xs):
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        X[rb[i]:rb[i] + n[i], :d[i]] = x
        if ys is not None:
            y[rb[i]:rb[i] + n[i]] = np.asarray(ys[i], dtype=np.float64)
    return Packed(X, y, rb, n, d)


def offsets(sizes: np.ndarray) -> np.ndarray:
    off = np.zeros(len(sizes), dtype=np.int64)
    if len(sizes):
        off[1:] = np.cumsum(np.asarray(sizes, dtype=np.int64)[:-1])
    return off


def seeds_table(entropies, mode: int) -> np.ndarray:
    out = np.zeros(len(entropies), dtype=_lib.SEED)
    for i, e in enumerate(entropies):
        out[i] = _lib.seed_record(e, mode)
    return out


def series_seed_table(base_seed: int, app_crc: np.ndarray, kernel: np.ndarray, bb: np.ndarray,
                      kind_crc: np.ndarray) -> np.ndarray:
    """Vectorised bbml_seed records (mode 1) for experiment.series_seed
    entropy [base & 2^64-1, crc32(app), kernel, bb, crc32(kind)]."""
    M = len(app_crc)
    out = np.zeros(M, dtype=_lib.SEED)
    base_words = _lib.int_words(int(base_seed) & _lib.M64)
    cols = [np.asarray(app_crc, dtype=np.uint64), np.asarray(kernel, dtype=np.uint64),
            np.asarray(bb, dtype=np.uint64), np.asarray(kind_crc, dtype=np.uint64)]
    nw = np.full(M, len(base_words), dtype=np.int32)
    words = out["words"]
    for j, w in enumerate(base_words):
        words[:, j] = w
    for c in cols:
        big = c > _lib.M32
        rows = np.arange(M)
        lo = (c & np.uint64(_lib.M32)).astype(np.uint32)
        hi = (c >> np.uint64(32)).astype(np.uint32)
        words[rows, nw] = lo
        nw = nw + 1
        if np.any(big):
            rb = rows[big]
            words[rb, nw[big]] = hi[big]
            nw[big] += 1
        if np.any(nw > _lib.MAX_WORDS):
            raise ValueError("series seed entropy exceeds 8 words")
    out["n_words"] = nw
    out["mode"] = 1
    return out


# ---------------------------------------------------------------------------
# device results
# ---------------------------------------------------------------------------

@dataclass
class TrainResult:
    weights: np.ndarray            # flat float64
    w_offset: np.ndarray           # (M,) int64
    P: np.ndarray                  # (M,) int
    status: np.ndarray             # (M,) STATUS
    history: Optional[np.ndarray]  # flat float64 or None
    hist_offset: Optional[np.ndarray]

    def w(self, i: int) -> np.ndarray:
        o = int(self.w_offset[i])
        return self.weights[o:o + int(self.P[i])]


class DeviceData:
    """Training rows resident in HBM (reused across PNN / BR / restarts)."""

    def __init__(self, packed: Packed, device=None):
        torch = torch_cuda()
        self.packed = packed
        self.device = torch.device("cuda" if device is None else device)
        self.X = torch.from_numpy(np.ascontiguousarray(packed.X)).to(self.device)
        self.y = torch.from_numpy(np.ascontiguousarray(packed.y)).to(self.device)

    @property
    def stride(self) -> int:
        return self.packed.stride


def _stream(torch):
    return torch.cuda.current_stream().cuda_stream


def pnn_tasks(row_begin, n, d, h, epochs, batch, lr, eps, seeds, want_history) -> tuple:
    M = len(n)
    t = np.zeros(M, dtype=PNN_TASK)
    t["row_begin"] = row_begin
    t["n"], t["d"], t["h"] = n, d, h
    t["epochs"], t["batch"] = epochs, batch
    t["lr"], t["eps"] = lr, eps
    t["seed"] = seeds
    P = n_params(t["d"], t["h"]).astype(np.int64)
    t["w_offset"] = offsets(P)
    if want_history:
        t["hist_offset"] = offsets(t["epochs"].astype(np.int64))
    else:
        t["hist_offset"] = -1
    return t, P


def lm_tasks(row_begin, n, d, h, max_epochs, seeds, want_history, estimate=1, mu0=0.005,
             mu_inc=10.0, mu_dec=0.1, mu_max=1e10, alpha0=1e-12, beta0=1.0) -> tuple:
    M = len(n)
    t = np.zeros(M, dtype=LM_TASK)
    t["row_begin"] = row_begin
    t["n"], t["d"], t["h"] = n, d, h
    t["max_epochs"], t["estimate"] = max_epochs, estimate
    t["mu0"], t["mu_inc"], t["mu_dec"], t["mu_max"] = mu0, mu_inc, mu_dec, mu_max
    t["alpha0"], t["beta0"] = alpha0, beta0
    t["seed"] = seeds
    P = n_params(t["d"], t["h"]).astype(np.int64)
    t["w_offset"] = offsets(P)
    if want_history:
        t["hist_offset"] = offsets(t["max_epochs"].astype(np.int64) * 10)
    else:
        t["hist_offset"] = -1
    return t, P


class Run:
    """Device buffers of one training launch (results stay in HBM until fetched)."""

    def __init__(self, torch, tasks, P, hist_len, device):
        M = len(tasks)
        self.tasks, self.P = tasks, P
        self.weights = torch.empty(int(P.sum()) if M else 1, dtype=torch.float64, device=device)
        self.status = torch.empty(max(M, 1) * STATUS.itemsize, dtype=torch.uint8, device=device)
        self.history = (torch.empty(max(hist_len, 1), dtype=torch.float64, device=device)
                        if hist_len is not None else None)

    def fetch(self) -> TrainResult:
        M = len(self.tasks)
        st = self.status.cpu().numpy().view(STATUS)[:M].copy()
        hist = self.history.cpu().numpy() if self.history is not None else None
        return TrainResult(self.weights.cpu().numpy(), self.tasks["w_offset"].copy(), self.P, st,
                           hist, self.tasks["hist_offset"].copy() if hist is not None else None)


def launch_pnn(data: DeviceData, tasks: np.ndarray, P: np.ndarray, precision: int = 64) -> Run:
    torch = torch_cuda()
    want = len(tasks) and tasks["hist_offset"][0] >= 0
    hist_len = int(tasks["epochs"].sum()) if want else None
    run = Run(torch, tasks, P, hist_len, data.device)
    tasks = np.ascontiguousarray(tasks)
    check(lib().bbml_pnn_train(ptr(tasks), len(tasks), ptr(data.X), ptr(data.y), data.stride,
                               ptr(run.weights), ptr(run.history), ptr(run.status), precision,
                               _stream(torch)), "bbml_pnn_train")
    return run


def launch_lm(data: DeviceData, tasks: np.ndarray, P: np.ndarray) -> Run:
    torch = torch_cuda()
    want = len(tasks) and tasks["hist_offset"][0] >= 0
    hist_len = int(tasks["max_epochs"].sum()) * 10 if want else None
    run = Run(torch, tasks, P, hist_len, data.device)
    tasks = np.ascontiguousarray(tasks)
    check(lib().bbml_lm_train(ptr(tasks), len(tasks), ptr(data.X), ptr(data.y), data.stride,
                              ptr(run.weights), ptr(run.history), ptr(run.status),
                              _stream(torch)), "bbml_lm_train")
    return run


def predict(weights_dev, w_offset, d, h, kind, Xq: Packed, norms: Optional[np.ndarray] = None,
            eps=1e-8, device=None):
    """Batched forward / predict_counts.  ``weights_dev`` is a device tensor or
    host array of packed weights; ``norms`` is (M, 2*d_max+2) rows of
    [x_min(d), x_max(d), y_min, y_max] (host) or None."""
    torch = torch_cuda()
    dev = torch.device("cuda" if device is None else device)
    M = len(w_offset)
    t = np.zeros(M, dtype=PRED_TASK)
    t["row_begin"] = Xq.row_begin
    t["n"] = Xq.n
    t["w_offset"] = w_offset
    t["d"], t["h"], t["kind"], t["eps"] = d, h, kind, eps
    t["out_offset"] = Xq.row_begin
    if not torch.is_tensor(weights_dev):
        weights_dev = torch.from_numpy(np.ascontiguousarray(weights_dev, dtype=np.float64)).to(dev)
    Xd = torch.from_numpy(np.ascontiguousarray(Xq.X)).to(dev)
    nd = None
    if norms is not None:
        norms = np.ascontiguousarray(norms, dtype=np.float64)
        t["norm_offset"] = np.arange(M, dtype=np.int64) * norms.shape[1]
        nd = torch.from_numpy(norms.ravel()).to(dev)
    else:
        t["norm_offset"] = -1
    out = torch.empty(max(len(Xq.y), 1), dtype=torch.float64, device=dev)
    check(lib().bbml_predict(ptr(t), M, ptr(Xd), Xq.stride, ptr(weights_dev), ptr(nd), ptr(out),
                             _stream(torch)), "bbml_predict")
    return out.cpu().numpy()[:int(Xq.n.sum())]


def metrics(pred, actual_norm, actual_raw, pred_offset, row_begin, n, d, norms, device=None):
    """Per-model test metrics on the device (``bbml_metrics``):
    for model i, predictions pred[pred_offset[i] : +n[i]] (normalised) against
    actual_norm / actual_raw[row_begin[i] : +n[i]]; ``norms`` is (M, 2*d_max+2)
    rows of [x_min(d), x_max(d), y_min, y_max].  Arrays may be host arrays or
    device tensors.  Returns (M, 4) host float64: mse, pearson, spearman (NaN =
    undefined) and a done flag (1.0: every model, any n)."""
    torch = torch_cuda()
    dev = torch.device("cuda" if device is None else device)

    def on_dev(a):
        if torch.is_tensor(a):
            return a
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

    M = len(n)
    norms = np.ascontiguousarray(norms, dtype=np.float64)
    t = np.zeros(M, dtype=PRED_TASK)
    t["row_begin"] = row_begin
    t["n"] = n
    t["w_offset"] = pred_offset
    t["d"] = d
    t["h"] = 1
    t["norm_offset"] = np.arange(M, dtype=np.int64) * norms.shape[1]
    t["out_offset"] = np.arange(M, dtype=np.int64) * 4
    pd, an, ar, nd = on_dev(pred), on_dev(actual_norm), on_dev(actual_raw), on_dev(norms.ravel())
    out = torch.empty(max(4 * M, 1), dtype=torch.float64, device=dev)
    check(lib().bbml_metrics(ptr(t), M, ptr(pd), ptr(an), ptr(ar), ptr(nd), ptr(out),
                             _stream(torch)), "bbml_metrics")
    return out.cpu().numpy()[:4 * M].reshape(M, 4)


def _met_tasks(pred_offset, row_begin, n, d, norm_rows_count, width):
    M = len(n)
    t = np.zeros(M, dtype=PRED_TASK)
    t["row_begin"] = row_begin
    t["n"] = n
    t["w_offset"] = pred_offset
    t["d"] = d
    t["h"] = 1
    t["norm_offset"] = np.arange(M, dtype=np.int64) * width
    return t


def pooled_metrics(groups, pred, actual_raw, pred_offset, row_begin, n, d, norms, device=None):
    """Pooled Pearson / Spearman per group of models on the device
    (``bbml_pooled_metrics``; experiment.summarize, experiment.py:180-206):
    model i (in ``groups[i]``) contributes its de-normalised predictions and
    raw counts; groups concatenate in model order.  Returns (G, 2) host
    float64, NaN = undefined."""
    torch = torch_cuda()
    dev = torch.device("cuda" if device is None else device)
    groups = np.ascontiguousarray(groups, dtype=np.int32)
    G = int(groups.max()) + 1 if len(groups) else 0
    if G == 0:
        return np.zeros((0, 2))
    norms = np.ascontiguousarray(norms, dtype=np.float64)
    t = _met_tasks(pred_offset, row_begin, n, d, len(n), norms.shape[1])
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    pd, ar, nd = up(pred), up(actual_raw), up(norms.ravel())
    out = torch.empty(2 * G, dtype=torch.float64, device=dev)
    check(lib().bbml_pooled_metrics(ptr(t), len(t), ptr(groups), G, ptr(pd), ptr(ar), ptr(nd),
                                    ptr(out), _stream(torch)), "bbml_pooled_metrics")
    return out.cpu().numpy().reshape(G, 2)


def heatmaps(pred, actual_raw, pred_offset, row_begin, n, d, norms, bins, device=None):
    """Per-model heatmap edges (M, bins+1) and counts (M, bins, bins) on the
    device (``bbml_heatmaps``; metrics.heatmap_data)."""
    torch = torch_cuda()
    dev = torch.device("cuda" if device is None else device)
    norms = np.ascontiguousarray(norms, dtype=np.float64)
    t = _met_tasks(pred_offset, row_begin, n, d, len(n), norms.shape[1])
    M = len(t)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    pd, ar, nd = up(pred), up(actual_raw), up(norms.ravel())
    edges = torch.empty(max(M, 1) * (bins + 1), dtype=torch.float64, device=dev)
    counts = torch.empty(max(M, 1) * bins * bins, dtype=torch.int32, device=dev)
    check(lib().bbml_heatmaps(ptr(t), M, ptr(pd), ptr(ar), ptr(nd), int(bins), ptr(edges), ptr(counts),
                              _stream(torch)), "bbml_heatmaps")
    return (edges.cpu().numpy()[:M * (bins + 1)].reshape(M, bins + 1),
            counts.cpu().numpy()[:M * bins * bins].reshape(M, bins, bins))


def kde(values: Sequence[np.ndarray], grid_points: int = 256, device=None):
    """Count KDE of many series on the device (``bbml_kde``): returns
    (grid (S, G), density (S, G), bandwidth (S,)) host arrays; bandwidth 0
    where the series has no spread (no curve)."""
    torch = torch_cuda()
    dev = torch.device("cuda" if device is None else device)
    n = np.array([len(v) for v in values], dtype=np.int64)
    off = np.zeros(len(values) + 1, dtype=np.int64)
    np.cumsum(n, out=off[1:])
    S = len(values)
    if S == 0:
        return np.zeros((0, grid_points)), np.zeros((0, grid_points)), np.zeros(0)
    flat = np.concatenate([np.asarray(v, dtype=np.float64) for v in values]) if off[-1] else np.zeros(1)
    vd = torch.from_numpy(flat).to(dev)
    grid = torch.empty(S * grid_points, dtype=torch.float64, device=dev)
    dens = torch.empty(S * grid_points, dtype=torch.float64, device=dev)
    bw = torch.empty(S, dtype=torch.float64, device=dev)
    check(lib().bbml_kde(ptr(off), S, ptr(vd), int(grid_points), ptr(grid), ptr(dens), ptr(bw),
                         _stream(torch)), "bbml_kde")
    return (grid.cpu().numpy().reshape(S, grid_points), dens.cpu().numpy().reshape(S, grid_points),
            bw.cpu().numpy())
