"""Drop-in for ``bbcount.brbpnn`` (reference ``pkg/src/bbcount/brbpnn.py``)
backed by the sm_100a kernels in ``libbbml.so``.

``train`` (brbpnn.py:286-346) runs the fused batched LM kernel
(``bbml_lm_train``); ``forward`` (85-91) the device predictor; the unit-level
functions (``tansig``, ``objective``, ``jacobian``, ``solve_damped``,
``lm_trial``, ``lm_step``, ``evidence_update``, ``update_hyperparams``) call
the device unit kernels and keep the reference's scalar control flow.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple, Optional, Union

import numpy as np

from . import _lib, engine, units

HYPER_MIN = 1e-12
HYPER_MAX = 1e12
MU_FLOOR = 1e-20
DEFAULT_HIDDEN = 1
EARLY_STOP_REL = 1e-7
EARLY_STOP_EPOCHS = 5


class BrbpnnError(Exception):
    pass


class NumericError(BrbpnnError, ArithmeticError):
    """The damped normal equations could not be solved."""


def tansig(x):
    """2 / (1 + exp(-2x)) - 1 on the device (brbpnn.py:33-38)."""
    out = units.tansig(np.asarray(x, dtype=float))
    return float(out) if out.ndim == 0 else out


@dataclass
class BrbpnnModel:
    W1: np.ndarray  # (hidden, n_inputs)
    b1: np.ndarray  # (hidden,)
    W2: np.ndarray  # (hidden,)
    b2: float
    alpha: float = HYPER_MIN
    beta: float = 1.0

    @property
    def n_inputs(self) -> int:
        return self.W1.shape[1]

    @property
    def hidden(self) -> int:
        return self.W1.shape[0]

    @property
    def n_params(self) -> int:
        return self.W1.size + self.b1.size + self.W2.size + 1


def init_model(n_inputs: int, hidden: int = DEFAULT_HIDDEN, rng: Optional[np.random.Generator] = None,
               seed: int = 0, alpha: float = HYPER_MIN, beta: float = 1.0) -> BrbpnnModel:
    """brbpnn.py:63-82 — same draw order as pnn.init_model (caller's NumPy rng)."""
    if rng is None:
        rng = np.random.default_rng(seed)
    a = 1.0 / math.sqrt(n_inputs)
    c = 1.0 / math.sqrt(hidden)
    W1 = rng.uniform(-a, a, size=(hidden, n_inputs))
    b1 = rng.uniform(-a, a, size=hidden)
    W2 = rng.uniform(-c, c, size=hidden)
    return BrbpnnModel(W1, b1, W2, float(rng.uniform(-c, c)), alpha, beta)


def pack(model: BrbpnnModel) -> np.ndarray:
    """Flat parameter vector W1 | b1 | W2 | b2 (brbpnn.py:94-99)."""
    return np.concatenate([model.W1.ravel(), model.b1, model.W2, [model.b2]])


def unpack(model: BrbpnnModel, w: np.ndarray) -> None:
    h, d = model.W1.shape
    hd = h * d
    model.W1 = w[:hd].reshape(h, d).copy()
    model.b1 = w[hd:hd + h].copy()
    model.W2 = w[hd + h:hd + 2 * h].copy()
    model.b2 = float(w[-1])


def forward(model: BrbpnnModel, x: np.ndarray) -> Union[float, np.ndarray]:
    x = np.asarray(x, dtype=float)
    single = x.ndim == 1
    X = np.atleast_2d(x)
    if X.shape[1] != model.n_inputs:  # the reference's X @ W1.T raises here
        raise ValueError(f"forward: expected {model.n_inputs} input columns, got {X.shape[1]}")
    out = engine.predict(pack(model), np.array([0]), model.n_inputs, model.hidden, 1,
                         engine.pack([X]))
    return float(out[0]) if single else out


def objective(model: BrbpnnModel, X: np.ndarray, y: np.ndarray) -> tuple[float, float, float]:
    """(F, E_D, E_W) with F = beta E_D + alpha E_W (brbpnn.py:109-115)."""
    X = np.atleast_2d(np.asarray(X, dtype=float))
    y = np.asarray(y, dtype=float)
    _, e_d, e_w, _ = units.br_eval(pack(model), X, y, model.n_inputs, model.hidden, False)
    return model.beta * e_d + model.alpha * e_w, e_d, e_w


def jacobian(model: BrbpnnModel, X: np.ndarray) -> np.ndarray:
    """d prediction / d parameter, rows = samples, pack() column order."""
    X = np.atleast_2d(np.asarray(X, dtype=float))
    _, _, _, J = units.br_eval(pack(model), X, np.zeros(len(X)), model.n_inputs, model.hidden, True)
    return J


@dataclass
class LmConfig:
    mu0: float = 0.005
    mu_inc: float = 10.0
    mu_dec: float = 0.1
    mu_max: float = 1e10
    max_epochs: int = 1000


@dataclass
class LmState:
    mu: float = 0.005
    epoch: int = 0


def solve_damped(J: np.ndarray, residuals: np.ndarray, w: np.ndarray, alpha: float, beta: float,
                 mu: float) -> np.ndarray:
    """(beta J'J + (mu + alpha) I) delta = -(beta J'r + alpha w), LU on the device."""
    delta, singular = units.damped_solve(J, residuals, w, alpha, beta, mu)
    if singular:
        raise NumericError(f"damped system singular at mu={mu}")
    return delta


def lm_trial(model: BrbpnnModel, state: LmState, X: np.ndarray, y: np.ndarray,
             config: LmConfig) -> bool:
    """One damped Gauss-Newton trial; keeps the weights only if F decreases."""
    X = np.atleast_2d(np.asarray(X, dtype=float))
    y = np.asarray(y, dtype=float)
    w = pack(model)
    r, e_d, e_w, J = units.br_eval(w, X, y, model.n_inputs, model.hidden, True)
    f_before = model.beta * e_d + model.alpha * e_w
    delta = solve_damped(J, r, w, model.alpha, model.beta, state.mu)
    unpack(model, w + delta)
    f_after, _, _ = objective(model, X, y)
    if f_after < f_before:
        state.mu = max(state.mu * config.mu_dec, MU_FLOOR)
        return True
    unpack(model, w)
    state.mu *= config.mu_inc
    return False


def lm_step(model: BrbpnnModel, state: LmState, X: np.ndarray, y: np.ndarray,
            config: LmConfig) -> bool:
    """Trials until acceptance, or False once mu exceeds mu_max (a stall)."""
    while True:
        if lm_trial(model, state, X, y, config):
            return True
        if state.mu > config.mu_max:
            return False


class HyperUpdate(NamedTuple):
    alpha: float
    beta: float
    gamma: float
    pinned: bool


def evidence_update(e_d: float, e_w: float, jtj: np.ndarray, alpha: float, beta: float,
                    n_samples: int) -> HyperUpdate:
    """MacKay re-estimation with device Jacobi eigenvalues (brbpnn.py:221-251)."""
    a, b, g, pinned, _ = units.evidence(e_d, e_w, jtj, alpha, beta, n_samples)
    return HyperUpdate(a, b, g, pinned)


def update_hyperparams(model: BrbpnnModel, X: np.ndarray, y: np.ndarray) -> HyperUpdate:
    X = np.atleast_2d(np.asarray(X, dtype=float))
    y = np.asarray(y, dtype=float)
    r, e_d, e_w, J = units.br_eval(pack(model), X, y, model.n_inputs, model.hidden, True)
    jtj, _ = units.gram(J, r)
    P = J.shape[1]
    jtj_h = jtj.cpu().numpy().reshape(P, P)
    return evidence_update(e_d, e_w, jtj_h, model.alpha, model.beta, len(np.atleast_1d(y)))


@dataclass(frozen=True)
class BrEpochRecord:
    epoch: int
    f_before: float
    f_after: float
    e_d: float
    e_w: float
    alpha: float
    beta: float
    gamma: float
    mu: float
    pinned: bool


def records_from(hist: np.ndarray, count: int) -> list[BrEpochRecord]:
    rows = np.asarray(hist[:count * 10]).reshape(count, 10)
    return [BrEpochRecord(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]),
                          float(r[5]), float(r[6]), float(r[7]), float(r[8]), bool(r[9]))
            for r in rows]


def raise_for_status(st) -> None:
    if int(st["code"]) == _lib.MODEL_SINGULAR:
        raise NumericError(f"damped system singular at mu={float(st['value'])}")
    if int(st["code"]) != _lib.MODEL_OK:
        raise BrbpnnError(f"device status {int(st['code'])}")


def train(X: np.ndarray, y: np.ndarray, hidden: int = DEFAULT_HIDDEN, seed: int = 0,
          config: LmConfig = LmConfig(), estimate_hyperparams: bool = True,
          alpha0: float = HYPER_MIN, beta0: float = 1.0
          ) -> tuple[BrbpnnModel, list[BrEpochRecord]]:
    """Full-batch LM + evidence training on the device (brbpnn.py:286-346)."""
    X = np.atleast_2d(np.asarray(X, dtype=float))
    y = np.asarray(y, dtype=float)
    if len(X) == 0:
        raise ValueError("cannot train on an empty series")
    if len(X) != len(y):
        raise ValueError("X and y lengths differ")
    packed = engine.pack([X], [y])
    data = engine.DeviceData(packed)
    seeds = engine.seeds_table([int(seed)], 0)
    tasks, P = engine.lm_tasks(packed.row_begin, packed.n, packed.d, hidden, config.max_epochs,
                               seeds, True, estimate=int(bool(estimate_hyperparams)),
                               mu0=config.mu0, mu_inc=config.mu_inc, mu_dec=config.mu_dec,
                               mu_max=config.mu_max, alpha0=alpha0, beta0=beta0)
    res = engine.launch_lm(data, tasks, P).fetch()
    st = res.status[0]
    raise_for_status(st)
    w = res.w(0)
    d = X.shape[1]
    hd = hidden * d
    model = BrbpnnModel(w[:hd].reshape(hidden, d).copy(), w[hd:hd + hidden].copy(),
                        w[hd + hidden:hd + 2 * hidden].copy(), float(w[-1]),
                        float(st["alpha"]), float(st["beta"]))
    return model, records_from(res.history, int(st["epochs"]))
