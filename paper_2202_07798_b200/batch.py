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
from .traces import BbSeries, SplitSpec, split, fit_normalizer, SplitError


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

    @property
    def n_models(self) -> int:
        return len(self.pnn) + len(self.lm)

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
                   precision=64) -> Workload:
    """Split + normalise every series once (traces.py semantics), then one
    PNN and/or BR task per (series, restart); restart r seeds the model with
    experiment.series_seed(r, key, kind)."""
    keys, norms, Xtr, ytr, Xte, yte, errors = [], [], [], [], [], [], {}
    for s in series:
        try:
            tr, te = split(s, spec)
        except SplitError as exc:
            errors[len(keys)] = str(exc)
            keys.append(s.key)
            norms.append(None)
            for lst in (Xtr, Xte):
                lst.append(np.zeros((0, s.arity)))
            ytr.append(np.zeros(0))
            yte.append(np.zeros(0))
            continue
        nm = fit_normalizer(tr)
        keys.append(s.key)
        norms.append(nm)
        Xtr.append(nm.transform_features(tr.X))
        ytr.append(nm.transform_targets(tr.y))
        Xte.append(nm.transform_features(te.X))
        yte.append(nm.transform_targets(te.y))
    train = engine.pack(Xtr, ytr)
    test = engine.pack(Xte, yte)
    ok = np.array([i for i in range(len(keys)) if i not in errors], dtype=np.int64)
    app_crc = np.array([zlib.crc32(k[0].encode("utf-8")) for k in keys], dtype=np.uint64)
    kid = np.array([k[1] for k in keys], dtype=np.uint64)
    bid = np.array([k[2] for k in keys], dtype=np.uint64)
    tabs = {}
    for kind in ("pnn", "brbpnn"):
        if kind not in kinds or not len(ok):
            tabs[kind] = (None, np.zeros(0, np.int64), np.zeros(0, np.int64))
            continue
        seeds, sidx = [], []
        for r in restarts:
            seeds.append(engine.series_seed_table(int(r), app_crc[ok], kid[ok], bid[ok],
                                                  np.full(len(ok), zlib.crc32(kind.encode()),
                                                          dtype=np.uint64)))
            sidx.append(ok)
        seeds = np.concatenate(seeds)
        sidx = np.concatenate(sidx)
        rb, n, d = train.row_begin[sidx], train.n[sidx], train.d[sidx]
        if kind == "pnn":
            tab, P = engine.pnn_tasks(rb, n, d, pnn_hidden, pnn_epochs, pnn_batch, pnn_lr, 1e-8,
                                      seeds, False)
        else:
            h = (np.array([br_hidden(keys[i]) for i in sidx], dtype=np.int32)
                 if callable(br_hidden) else br_hidden)
            tab, P = engine.lm_tasks(rb, n, d, h, br_max_epochs, seeds, False)
        tabs[kind] = (tab, P, sidx)
    empty_p = np.zeros(0, dtype=_lib.PNN_TASK)
    empty_l = np.zeros(0, dtype=_lib.LM_TASK)
    pt, pP, ps = tabs["pnn"]
    lt, lP, ls = tabs["brbpnn"]
    return Workload(train, test, keys, norms, empty_p if pt is None else pt,
                    empty_l if lt is None else lt, ps, ls,
                    np.zeros(0, np.int64) if pt is None else pP,
                    np.zeros(0, np.int64) if lt is None else lP, precision, errors)


class DeviceWorkload:
    """A workload resident in HBM plus its output buffers."""

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

    def upload(self):
        self.X.copy_(self.host.X, non_blocking=True)
        self.y.copy_(self.host.y, non_blocking=True)
        self.Xq.copy_(self.host.Xq, non_blocking=True)

    @property
    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.host.X, self.host.y, self.host.Xq))

    def step(self) -> int:
        """Enqueue train (both kinds, concurrently) + predict on the current
        stream; returns the number of kernel launches issued."""
        torch = self.torch
        so = lib()
        main = torch.cuda.current_stream(self.device)
        launches = 0
        stride = self.wl.train.stride
        if self.n_l:
            self.side.wait_stream(main)
            with torch.cuda.stream(self.side):
                check(so.bbml_lm_train(ptr(self.lm_tab), self.n_l, ptr(self.X), ptr(self.y), stride,
                                       ptr(self.weights) + 8 * int(self.wl.P_pnn.sum()), None,
                                       ptr(self.status) + STATUS.itemsize * self.n_p,
                                       self.side.cuda_stream), "bbml_lm_train")
            launches += _launches_lm(self.lm_tab)
        if self.n_p:
            check(so.bbml_pnn_train(ptr(self.pnn_tab), self.n_p, ptr(self.X), ptr(self.y), stride,
                                    ptr(self.weights), None, ptr(self.status), self.wl.precision,
                                    main.cuda_stream), "bbml_pnn_train")
            launches += _launches_pnn(self.pnn_tab)
        if self.n_l:
            main.wait_stream(self.side)
        if self.wl.n_models:
            check(so.bbml_predict(ptr(self.pred_tab), len(self.pred_tab), ptr(self.Xq),
                                  self.wl.test.stride, ptr(self.weights), None, ptr(self.pred),
                                  main.cuda_stream), "bbml_predict")
            launches += 1
        return launches

    def fetch(self) -> dict:
        out = {
            "weights": self.weights.cpu().numpy(),
            "status": self.status.cpu().numpy().view(STATUS)[: self.wl.n_models].copy(),
            "pred": self.pred.cpu().numpy(),
        }
        return out

    @property
    def d2h_bytes(self) -> int:
        return (self.weights.numel() * 8 + self.status.numel() + self.pred.numel() * 8)


def _launches_pnn(tab) -> int:
    if not len(tab):
        return 0
    dm = np.where(tab["d"] <= 2, 2, np.where(tab["d"] <= 4, 4, 16))
    hm = np.where(tab["h"] <= 16, 16, 64)
    return len(set(zip(dm.tolist(), hm.tolist())))


def _launches_lm(tab) -> int:
    if not len(tab):
        return 0
    P = tab["h"] * (tab["d"] + 2) + 1
    b = np.where(P <= 8, 8, np.where(P <= 32, 32, np.where(P <= 64, 64, 96)))
    return len(set(b.tolist()))


class HostBuffers:
    """Pinned host copies of the workload inputs (the e2e source buffers)."""

    def __init__(self, wl: Workload):
        torch = engine.torch_cuda()
        self.X = torch.from_numpy(np.ascontiguousarray(wl.train.X)).pin_memory()
        self.y = torch.from_numpy(np.ascontiguousarray(wl.train.y)).pin_memory()
        self.Xq = torch.from_numpy(np.ascontiguousarray(wl.test.X)).pin_memory()


def fit_predict(wl: Workload, dev: Optional[DeviceWorkload] = None) -> dict:
    """End-to-end: H2D of the inputs, train every model, predict, D2H results."""
    dev = DeviceWorkload(wl) if dev is None else dev
    dev.upload()
    dev.step()
    return dev.fetch()
