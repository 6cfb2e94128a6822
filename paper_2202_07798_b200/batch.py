"""Public batched API: train + evaluate thousands of independent PNN and
BR-BPNN models (one per application x basic block x restart) with three
kernel launches per step:

    stream A: bbml_pnn_train  (all PNN models)
    stream B: bbml_lm_train   (all BR-BPNN models)        } concurrent
    join    : bbml_predict    (every model's test rows)

``Workload`` is the host-side description (CSR-packed, already split and
normalised with the reference semantics); ``DeviceWorkload`` keeps it
resident in HBM so repeated steps re-train from scratch without host work.
``fit_predict`` is the end-to-end call: pinned host buffers -> HBM -> kernels
-> host results.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib, engine
from ._lib import PRED_TASK, STATUS, check, lib, ptr
from . import prep
from .traces import BbSeries, Normalizer, SplitSpec


@dataclass
class Workload:
    train: engine.Packed        # normalised training rows of every prepared series
    test: engine.Packed         # normalised test rows (same series order)
    keys: list                  # series keys (prepared series order)
    norms: list                 # Normalizer per prepared series
    pnn: np.ndarray             # PNN_TASK table
    lm: np.ndarray              # LM_TASK table
    pnn_series: np.ndarray      # series index of each PNN task
    lm_series: np.ndarray       # series index of each LM task
    P_pnn: np.ndarray
    P_lm: np.ndarray
    precision: int = 64
    errors: Optional[dict] = None  # series index -> split error text
    test_raw_y: Optional[np.ndarray] = None  # raw test counts, packed like test.y

    @property
    def n_models(self) -> int:
        return len(self.pnn) + len(self.lm)

    def norm_rows(self) -> np.ndarray:
        """(series, 2*d_max+2) rows of [x_min(d), x_max(d), y_min, y_max]."""
        if getattr(self, "_norm_rows", None) is not None:
            return self._norm_rows
        dmax = max([int(self.train.d.max()) if len(self.train.d) else 1, 1])
        rows = np.zeros((len(self.keys), 2 * dmax + 2))
        for i, nm in enumerate(self.norms):
            if nm is None:
                continue
            d = len(nm.x_min)
            rows[i, :d] = nm.x_min
            rows[i, d:2 * d] = nm.x_max
            rows[i, 2 * d] = nm.y_min
            rows[i, 2 * d + 1] = nm.y_max
        return rows

    def pred_tasks(self) -> np.ndarray:
        """Predict table over all models (PNN first), test rows of each model's series,
        weights in one buffer (PNN block then LM block)."""
        M = self.n_models
        t = np.zeros(M, dtype=PRED_TASK)
        sid = np.concatenate([self.pnn_series, self.lm_series]).astype(np.int64)
        t["row_begin"] = self.test.row_begin[sid]
        t["n"] = self.test.n[sid]
        t["d"] = np.concatenate([self.pnn["d"], self.lm["d"]])
        t["h"] = np.concatenate([self.pnn["h"], self.lm["h"]])
        t["kind"] = np.concatenate([np.zeros(len(self.pnn), np.int32), np.ones(len(self.lm), np.int32)])
        t["eps"] = 1e-8
        t["w_offset"] = np.concatenate([self.pnn["w_offset"],
                                        self.lm["w_offset"] + int(self.P_pnn.sum())])
        t["norm_offset"] = -1
        t["out_offset"] = engine.offsets(t["n"].astype(np.int64))
        return t


def build_workload(series: Sequence[BbSeries], spec: SplitSpec, *, kinds=("pnn", "brbpnn"),
                   restarts: Sequence[int] = (0,), pnn_epochs=300, pnn_batch=10, pnn_lr=1e-4,
                   pnn_hidden=10, br_hidden: int | Callable = 1, br_max_epochs=1000,
                   precision=64, table: Optional[prep.SeriesTable] = None,
                   units: Optional[np.ndarray] = None) -> Workload:
    """Split + normalise every series once (``prep.prepare``: whole-array
    passes with the reference's traces.py semantics), then one PNN and/or BR
    task per (series, restart); restart r seeds the model with
    experiment.series_seed(r, key, kind).  ``units``
    ((U, 2) int array of (series index, restart)) replaces the full
    series x restarts product with an explicit list (a strong-scaling shard);
    units whose series failed to split are dropped."""
    t = prep.SeriesTable.from_series(series) if table is None else table
    P = prep.prepare(t, spec.mode.value, spec.fraction, spec.seed)
    keys = list(t.keys)
    S = len(keys)
    dmax = t.X.shape[1]
    ok_mask = np.zeros(S, dtype=bool)
    ok_mask[P.ok] = True
    d_ser = np.where(ok_mask, t.d, 0).astype(np.int32)
    train = engine.Packed(P.Xtr, P.ytr, P.tr_off[:-1].copy(), np.diff(P.tr_off).astype(np.int32), t.d.copy())
    test = engine.Packed(P.Xte, P.yte, P.te_off[:-1].copy(), np.diff(P.te_off).astype(np.int32), t.d.copy())
    norms = _Normalizers(P, ok_mask)
    ok = P.ok.astype(np.int64)
    crc = {}
    app_crc = np.array([crc.setdefault(k[0], zlib.crc32(k[0].encode("utf-8"))) for k in keys],
                       dtype=np.uint64)
    kid = np.array([k[1] for k in keys], dtype=np.uint64)
    bid = np.array([k[2] for k in keys], dtype=np.uint64)
    tabs = {}
    for kind in ("pnn", "brbpnn"):
        if kind not in kinds or not len(ok):
            tabs[kind] = (None, np.zeros(0, np.int64), np.zeros(0, np.int64))
            continue
        kc = zlib.crc32(kind.encode())
        if units is None:
            pairs = [(ok, int(r)) for r in restarts]
        else:
            u = np.asarray(units, dtype=np.int64).reshape(-1, 2)
            u = u[ok_mask[u[:, 0]]]
            pairs = [(u[u[:, 1] == r, 0], int(r)) for r in np.unique(u[:, 1])]
            order = np.concatenate([np.flatnonzero(u[:, 1] == r) for r in np.unique(u[:, 1])]) \
                if len(u) else np.zeros(0, np.int64)
        seeds, sidx = [], []
        for si, r in pairs:
            seeds.append(engine.series_seed_table(r, app_crc[si], kid[si], bid[si],
                                                  np.full(len(si), kc, dtype=np.uint64)))
            sidx.append(si)
        seeds = np.concatenate(seeds) if seeds else np.zeros(0, dtype=_lib.SEED)
        sidx = np.concatenate(sidx) if sidx else np.zeros(0, np.int64)
        if units is not None and len(sidx):  # back to the caller's unit order
            inv = np.empty_like(order)
            inv[order] = np.arange(len(order))
            seeds, sidx = seeds[inv], sidx[inv]
        rb, n, d = train.row_begin[sidx], train.n[sidx], d_ser[sidx]
        if kind == "pnn":
            tab, Pn = engine.pnn_tasks(rb, n, d, pnn_hidden, pnn_epochs, pnn_batch, pnn_lr, 1e-8,
                                       seeds, False)
        else:
            if callable(br_hidden):  # once per series, then gathered per task
                hs = np.array([br_hidden(k) for k in keys], dtype=np.int32)
                h = hs[sidx]
            else:
                h = br_hidden
            tab, Pn = engine.lm_tasks(rb, n, d, h, br_max_epochs, seeds, False)
        tabs[kind] = (tab, Pn, sidx)
    empty_p = np.zeros(0, dtype=_lib.PNN_TASK)
    empty_l = np.zeros(0, dtype=_lib.LM_TASK)
    pt, pP, ps = tabs["pnn"]
    lt, lP, ls = tabs["brbpnn"]
    wl = Workload(train, test, keys, norms, empty_p if pt is None else pt,
                  empty_l if lt is None else lt, ps, ls,
                  np.zeros(0, np.int64) if pt is None else pP,
                  np.zeros(0, np.int64) if lt is None else lP, precision, P.errors, P.yte_raw)
    wl._norm_rows = P.norm_rows(dmax)
    return wl


class _Normalizers:
    """Per-series ``Normalizer`` views of the batched statistics, built on
    access (None for series that failed to split)."""

    def __init__(self, P, ok_mask):
        self._P, self._ok = P, ok_mask

    def __len__(self) -> int:
        return len(self._ok)

    def __getitem__(self, i):
        if not self._ok[i]:
            return None
        P, d = self._P, int(self._P.table.d[i])
        return Normalizer(P.x_min[i, :d].copy(), P.x_max[i, :d].copy(), float(P.y_min[i]),
                          float(P.y_max[i]))

    def __iter__(self):
        return (self[i] for i in range(len(self)))


class DeviceWorkload:
    """A workload resident in HBM plus its output buffers."""

    # enqueue the PNN call before the LM call: it holds the longest chains
    # (A/B on suite16 x32, tools/ab_order.py: step 936-956 -> 907-935 ms)
    pnn_first = True

    def __init__(self, wl: Workload, device=None, pinned_inputs=None):
        torch = engine.torch_cuda()
        self.torch = torch
        self.wl = wl
        dev = torch.device("cuda" if device is None else device)
        self.device = dev
        src = pinned_inputs or HostBuffers(wl)
        self.host = src
        self.X = torch.empty_like(src.X, device=dev)
        self.y = torch.empty_like(src.y, device=dev)
        self.Xq = torch.empty_like(src.Xq, device=dev)
        self.yq = torch.empty_like(src.yq, device=dev)
        self.yq_raw = torch.empty_like(src.yq_raw, device=dev)
        self.norms = torch.empty_like(src.norms, device=dev)
        self.upload()
        self.n_p, self.n_l = len(wl.pnn), len(wl.lm)
        W = int(wl.P_pnn.sum() + wl.P_lm.sum())
        self.weights = torch.empty(max(W, 1), dtype=torch.float64, device=dev)
        self.status = torch.empty(max(wl.n_models, 1) * STATUS.itemsize, dtype=torch.uint8, device=dev)
        self.pred_tab = wl.pred_tasks()
        self.pred = torch.empty(max(int(self.pred_tab["n"].sum()), 1), dtype=torch.float64, device=dev)
        self.side = torch.cuda.Stream(device=dev)
        self.pnn_tab = np.ascontiguousarray(wl.pnn)
        self.lm_tab = np.ascontiguousarray(wl.lm)
        # per-model test metrics (bbml_metrics): predictions at the predict
        # table's out_offset, targets at the series' test rows
        sid = np.concatenate([wl.pnn_series, wl.lm_series]).astype(np.int64)
        width = wl.norm_rows().shape[1]
        mt = np.zeros(wl.n_models, dtype=PRED_TASK)
        mt["row_begin"] = wl.test.row_begin[sid] if len(sid) else 0
        mt["n"] = self.pred_tab["n"]
        mt["w_offset"] = self.pred_tab["out_offset"]
        mt["d"] = self.pred_tab["d"]
        mt["h"] = 1
        mt["norm_offset"] = sid * width
        mt["out_offset"] = np.arange(wl.n_models, dtype=np.int64) * 4
        self.met_tab = mt
        self.metrics = torch.empty(max(4 * wl.n_models, 1), dtype=torch.float64, device=dev)
        self._pinned_out = None

    def _inputs(self):
        return (("X", self.X, self.host.X), ("y", self.y, self.host.y), ("Xq", self.Xq, self.host.Xq),
                ("yq", self.yq, self.host.yq), ("yq_raw", self.yq_raw, self.host.yq_raw),
                ("norms", self.norms, self.host.norms))

    def upload(self):
        for _, dst, src in self._inputs():
            dst.copy_(src, non_blocking=True)

    def refresh(self, wl: Workload) -> None:
        """Load a freshly prepared workload of the same shapes (e.g. the same
        series re-split and re-normalised from raw rows): host arrays into
        the pinned staging buffers, task tables replaced, then H2D."""
        torch = self.torch
        torch.cuda.current_stream(self.device).synchronize()  # staging may still feed the last H2D
        new = {"X": wl.train.X, "y": wl.train.y, "Xq": wl.test.X, "yq": wl.test.y,
               "yq_raw": wl.test_raw_y, "norms": wl.norm_rows().ravel()}
        for name, _, dst in self._inputs():
            a = np.ascontiguousarray(new[name], dtype=np.float64)
            if a.size != dst.numel():
                raise ValueError(f"refresh: {name} has {a.size} values, the resident workload {dst.numel()}")
            dst.numpy().reshape(a.shape)[...] = a
        if len(wl.pnn) != self.n_p or len(wl.lm) != self.n_l:
            raise ValueError("refresh: model count changed")
        self.wl = wl
        self.pnn_tab = np.ascontiguousarray(wl.pnn)
        self.lm_tab = np.ascontiguousarray(wl.lm)
        self.upload()

    @property
    def table_bytes(self) -> int:
        """Task tables the library uploads per step (train, predict, metrics)."""
        return (self.pnn_tab.nbytes + self.lm_tab.nbytes + self.pred_tab.nbytes + self.met_tab.nbytes)

    @property
    def h2d_bytes(self) -> int:
        return sum(src.numel() * src.element_size() for _, _, src in self._inputs())

    def step(self) -> int:
        """Enqueue train (both kinds, concurrently) + predict on the current
        stream; returns the number of kernel launches issued."""
        torch = self.torch
        so = lib()
        main = torch.cuda.current_stream(self.device)
        launches = 0
        stride = self.wl.train.stride

        def lm():
            with torch.cuda.stream(self.side):
                check(so.bbml_lm_train(ptr(self.lm_tab), self.n_l, ptr(self.X), ptr(self.y), stride,
                                       ptr(self.weights) + 8 * int(self.wl.P_pnn.sum()), None,
                                       ptr(self.status) + STATUS.itemsize * self.n_p,
                                       self.side.cuda_stream), "bbml_lm_train")
            return _launches_lm(self.lm_tab)

        if self.n_l:
            self.side.wait_stream(main)
            if not self.pnn_first:
                launches += lm()
        if self.n_p:
            check(so.bbml_pnn_train(ptr(self.pnn_tab), self.n_p, ptr(self.X), ptr(self.y), stride,
                                    ptr(self.weights), None, ptr(self.status), self.wl.precision,
                                    main.cuda_stream), "bbml_pnn_train")
            launches += _launches_pnn(self.pnn_tab)
        if self.n_l:
            if self.pnn_first:
                launches += lm()
            main.wait_stream(self.side)
        if self.wl.n_models:
            check(so.bbml_predict(ptr(self.pred_tab), len(self.pred_tab), ptr(self.Xq),
                                  self.wl.test.stride, ptr(self.weights), None, ptr(self.pred),
                                  main.cuda_stream), "bbml_predict")
            check(so.bbml_metrics(ptr(self.met_tab), len(self.met_tab), ptr(self.pred),
                                  ptr(self.yq), ptr(self.yq_raw), ptr(self.norms), ptr(self.metrics),
                                  main.cuda_stream), "bbml_metrics")
            launches += 2
        return launches

    def fetch(self, predictions: bool = True) -> dict:
        """Weights, status and per-model metrics ((M, 4): mse, pearson,
        spearman, done); with ``predictions`` also every test prediction."""
        torch = self.torch
        names = ("weights", "status", "metrics") + (("pred",) if predictions else ())
        if self._pinned_out is None:
            self._pinned_out = {}
        for k in names:  # pinned staging buffers, allocated once per workload
            if k not in self._pinned_out:
                self._pinned_out[k] = torch.empty_like(getattr(self, k), device="cpu", pin_memory=True)
            self._pinned_out[k].copy_(getattr(self, k), non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        h = {k: self._pinned_out[k].numpy().copy() for k in names}
        out = {
            "weights": h["weights"],
            "status": h["status"].view(STATUS)[: self.wl.n_models].copy(),
            "metrics": h["metrics"][: 4 * self.wl.n_models].reshape(-1, 4),
        }
        if predictions:
            out["pred"] = h["pred"]
        return out

    def d2h_bytes_for(self, predictions: bool = True) -> int:
        return (self.weights.numel() * 8 + self.status.numel() + self.metrics.numel() * 8 +
                (self.pred.numel() * 8 if predictions else 0))

    @property
    def d2h_bytes(self) -> int:
        return self.d2h_bytes_for(True)


def _launches_pnn(tab) -> int:
    """Kernels bbml_pnn_train launches: one row-conversion pass (FP64 TMA
    records / FP32 rows) plus one trainer per (d, hidden) bucket."""
    if not len(tab):
        return 0
    dm = np.where(tab["d"] <= 2, 2, np.where(tab["d"] <= 4, 4, 16))
    hm = np.where(tab["h"] <= 16, 16, 64)
    return 1 + len(set(zip(dm.tolist(), hm.tolist())))


def _launches_lm(tab) -> int:
    """Kernels bbml_lm_train launches: one per shape group (lm_train.cu
    lm_key: hidden-1 warp path per d, hidden-1 long-series CTA path per d,
    P <= 8, P <= 32, wide)."""
    if not len(tab):
        return 0
    P = tab["h"] * (tab["d"] + 2) + 1
    h1 = (tab["h"] == 1) & (tab["d"] <= 4)
    key = np.where(h1, np.where(tab["n"] >= 2048, 100 + tab["d"], tab["d"]),
                   np.where(P <= 8, 8, np.where(P <= 32, 32, 512)))
    return len(set(key.tolist()))


class HostBuffers:
    """Pinned host copies of the workload inputs (the e2e source buffers)."""

    def __init__(self, wl: Workload):
        torch = engine.torch_cuda()
        self.X = torch.from_numpy(np.ascontiguousarray(wl.train.X)).pin_memory()
        self.y = torch.from_numpy(np.ascontiguousarray(wl.train.y)).pin_memory()
        self.Xq = torch.from_numpy(np.ascontiguousarray(wl.test.X)).pin_memory()
        # test targets (normalised + raw) and normaliser rows for the device metrics
        self.yq = torch.from_numpy(np.ascontiguousarray(wl.test.y, dtype=np.float64)).pin_memory()
        raw = wl.test_raw_y if wl.test_raw_y is not None else np.zeros(0)
        self.yq_raw = torch.from_numpy(np.ascontiguousarray(raw, dtype=np.float64)).pin_memory()
        self.norms = torch.from_numpy(np.ascontiguousarray(wl.norm_rows()).ravel()).pin_memory()


def fit_predict(wl: Workload, dev: Optional[DeviceWorkload] = None,
                predictions: bool = True) -> dict:
    """End-to-end: H2D of the inputs, train every model, predict, per-model
    metrics, D2H of weights / status / metrics (+ predictions)."""
    dev = DeviceWorkload(wl) if dev is None else dev
    dev.upload()
    dev.step()
    return dev.fetch(predictions)
