"""ctypes binding of ``libbbml.so`` (the C-ABI declared in ``include/bbml.h``).

This is the only way the package reaches compute: there is no CPU fallback.
If the library is missing, ``lib()`` raises; if CUDA is unavailable the
training / prediction entry points raise ``DeviceUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libbbml.so"

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
MAX_WORDS = 8

# --- struct layouts (must match include/bbml.h; checked at load) ---------
SEED = np.dtype([("words", "<u4", (MAX_WORDS,)), ("n_words", "<i4"), ("mode", "<i4")])
PNN_TASK = np.dtype([
    ("row_begin", "<i8"), ("w_offset", "<i8"), ("hist_offset", "<i8"),
    ("n", "<i4"), ("d", "<i4"), ("h", "<i4"), ("epochs", "<i4"), ("batch", "<i4"),
    ("reserved", "<i4"), ("lr", "<f8"), ("eps", "<f8"), ("seed", SEED)])
LM_TASK = np.dtype([
    ("row_begin", "<i8"), ("w_offset", "<i8"), ("hist_offset", "<i8"),
    ("n", "<i4"), ("d", "<i4"), ("h", "<i4"), ("max_epochs", "<i4"), ("estimate", "<i4"),
    ("reserved", "<i4"), ("mu0", "<f8"), ("mu_inc", "<f8"), ("mu_dec", "<f8"), ("mu_max", "<f8"),
    ("alpha0", "<f8"), ("beta0", "<f8"), ("seed", SEED)])
PRED_TASK = np.dtype([
    ("row_begin", "<i8"), ("w_offset", "<i8"), ("norm_offset", "<i8"), ("out_offset", "<i8"),
    ("n", "<i4"), ("d", "<i4"), ("h", "<i4"), ("kind", "<i4"), ("eps", "<f8")])
STATUS = np.dtype([
    ("code", "<i4"), ("epochs", "<i4"), ("detail", "<i4"), ("trials", "<i4"),
    ("value", "<f8"), ("mu", "<f8"), ("gamma", "<f8"), ("alpha", "<f8"), ("beta", "<f8")])

# device envelope (include/bbml.h)
MAX_INPUTS, PNN_MAX_HIDDEN, LM_MAX_PARAMS = 16, 64, 512

MODEL_OK, MODEL_DIVERGED, MODEL_NONFINITE_GRAD, MODEL_SINGULAR, MODEL_BAD_TASK = range(5)
BLOCK_NAMES = ("W1", "b1", "W2", "b2")

EXPORTS = (
    "bbml_abi_version", "bbml_struct_size", "bbml_version", "bbml_last_error",
    "bbml_seedseq_generate", "bbml_pcg64_state", "bbml_pnn_train", "bbml_lm_train",
    "bbml_predict", "bbml_pnn_loss_grad", "bbml_lm_jacobian", "bbml_lm_solve",
    "bbml_lm_evidence", "bbml_lm_gram", "bbml_adam_step", "bbml_tansig",
    "bbml_fma_peak", "bbml_metrics", "bbml_pooled_metrics", "bbml_heatmaps", "bbml_kde",
)


class BbmlError(RuntimeError):
    """A C-ABI call returned a non-zero bbml_status."""


class DeviceUnavailable(RuntimeError):
    """No CUDA device: this package has no CPU fallback by design."""


_lock = threading.Lock()
_lib = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

_SIGS = {
    "bbml_abi_version": (_i32, []),
    "bbml_struct_size": (_i64, [_i32]),
    "bbml_version": (ctypes.c_char_p, []),
    "bbml_last_error": (ctypes.c_char_p, []),
    "bbml_seedseq_generate": (_i32, [_vp, _i32, _vp, _i32]),
    "bbml_pcg64_state": (_i32, [_vp, _vp]),
    "bbml_pnn_train": (_i32, [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp]),
    "bbml_lm_train": (_i32, [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "bbml_predict": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    "bbml_metrics": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbml_pooled_metrics": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "bbml_heatmaps": (_i32, [_vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "bbml_kde": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    "bbml_pnn_loss_grad": (_i32, [_vp, _i32, _vp, _vp, _i32, _vp, _f64, _vp, _vp, _vp]),
    "bbml_lm_jacobian": (_i32, [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbml_lm_gram": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbml_adam_step": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp, _i32, _f64, _f64, _f64, _f64, _f64,
                              _f64, _vp, _vp]),
    "bbml_tansig": (_i32, [_vp, _vp, _i64, _vp]),
    "bbml_fma_peak": (_i32, [_i32, _i32, _i32, _vp, _vp]),
    "bbml_lm_solve": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbml_lm_evidence": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}


def lib() -> ctypes.CDLL:
    """Load (once) and layout-check the in-tree ``libbbml.so``."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("BBML_LIB", LIB_PATH))
        if not path.exists():
            raise FileNotFoundError(
                f"{path} is missing: build it with `python -m paper_2202_07798_b200.build` "
                "(there is no CPU fallback)")
        so = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        sizes = [so.bbml_struct_size(i) for i in range(5)]
        want = [SEED.itemsize, PNN_TASK.itemsize, LM_TASK.itemsize, PRED_TASK.itemsize,
                STATUS.itemsize]
        if sizes != want:
            raise BbmlError(f"ABI struct layout mismatch: C {sizes} vs Python {want}")
        _lib = so
        return so


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().bbml_last_error().decode(errors="replace")
        raise BbmlError(f"{what} failed (status {status}): {msg}")


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


# --- entropy helpers (numpy SeedSequence int coercion) --------------------

def int_words(value: int) -> list[int]:
    value = int(value)
    if value < 0:
        raise ValueError("seed must be non-negative")
    if value == 0:
        return [0]
    out = []
    while value:
        out.append(value & M32)
        value >>= 32
    return out


def seed_record(entropy, mode: int) -> np.ndarray:
    """One ``bbml_seed``: ``entropy`` is an int (mode 0) or a list of ints."""
    words: list[int] = []
    for item in ([entropy] if isinstance(entropy, (int, np.integer)) else entropy):
        words.extend(int_words(item))
    if len(words) > MAX_WORDS:
        raise ValueError(f"seed entropy needs {len(words)} 32-bit words; at most {MAX_WORDS}")
    rec = np.zeros((), dtype=SEED)
    rec["words"][: len(words)] = words
    rec["n_words"] = len(words)
    rec["mode"] = mode
    return rec


def seedseq_u64(entropy) -> int:
    """SeedSequence(entropy).generate_state(1, uint64)[0] via the C-ABI."""
    flat: list[int] = []
    for item in ([entropy] if isinstance(entropy, (int, np.integer)) else entropy):
        flat.extend(int_words(item))
    words = np.ascontiguousarray(flat, dtype=np.uint32)
    out = np.zeros(2, dtype=np.uint32)
    check(lib().bbml_seedseq_generate(ptr(words), len(words), ptr(out), 2), "bbml_seedseq_generate")
    return int(out[0]) | (int(out[1]) << 32)


def pcg64_state(entropy, mode: int = 0) -> tuple[int, int]:
    rec = seed_record(entropy, mode)
    out = np.zeros(4, dtype=np.uint64)
    check(lib().bbml_pcg64_state(ptr(rec), ptr(out)), "bbml_pcg64_state")
    return (int(out[0]) << 64) | int(out[1]), (int(out[2]) << 64) | int(out[3])
