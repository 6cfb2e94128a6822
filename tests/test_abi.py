"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol ``include/bbml.h`` declares, struct layouts agree with the Python
binding, and the host-side RNG entry points reproduce NumPy's streams."""

import re
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_2202_07798_b200 import _lib, engine
from oracle.rng import Pcg64, generate_u64

HEADER = Path(__file__).resolve().parents[1] / "include" / "bbml.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:bbml_status|int32_t|int64_t|const char\*)\s+(bbml_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    so = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 16
    for name in syms:
        assert hasattr(so, name), name
    assert set(syms) == set(_lib.EXPORTS)


def test_struct_layout_and_version():
    so = _lib.lib()
    assert so.bbml_abi_version() == 1
    assert so.bbml_struct_size(1) == _lib.PNN_TASK.itemsize == 104
    assert so.bbml_struct_size(2) == _lib.LM_TASK.itemsize == 136
    assert so.bbml_struct_size(9) == -1
    assert b"sm_100a" in so.bbml_version()


def test_host_seedseq_matches_numpy():
    rng = np.random.default_rng(5)
    for _ in range(50):
        ent = [int(v) for v in rng.integers(0, 2**63, size=int(rng.integers(1, 6)))]
        assert _lib.seedseq_u64(ent) == generate_u64(ent, 1)[0]
        assert _lib.seedseq_u64(ent) == int(np.random.SeedSequence(ent).generate_state(1, np.uint64)[0])


def test_host_pcg64_state_matches_numpy():
    for seed in (0, 1, 123, 2**63 + 5, 2**64 + 7, 2**127 + 99):
        st = np.random.default_rng(seed).bit_generator.state["state"]
        assert _lib.pcg64_state(seed) == (st["state"], st["inc"])


def test_series_seed_table_matches_scalar_records():
    apps = ["app", "2mm", "gramschmit"]
    kinds = ["pnn", "brbpnn"]
    keys = [(a, k, b) for a in apps for k in (0, 3, 2**33) for b in (0, 1, 77)]
    for base in (0, 7, 2**40, 2**64 - 1):
        for kind in kinds:
            tab = engine.series_seed_table(
                base, np.array([zlib.crc32(k[0].encode()) for k in keys]),
                np.array([k[1] for k in keys]), np.array([k[2] for k in keys]),
                np.full(len(keys), zlib.crc32(kind.encode())))
            for rec, key in zip(tab, keys):
                ent = [base, zlib.crc32(key[0].encode()), key[1], key[2], zlib.crc32(kind.encode())]
                want = _lib.seed_record(ent, 1)
                assert rec.tobytes() == want.tobytes()
                # and the resulting PCG64 state equals numpy's default_rng(series_seed)
            ent = [base, zlib.crc32(keys[0][0].encode()), keys[0][1], keys[0][2],
                   zlib.crc32(kind.encode())]
            s = generate_u64(ent, 1)[0]
            p = Pcg64(s)
            assert _lib.pcg64_state(ent, 1) == (p.state, p.inc)


def test_seed_entropy_limits():
    with pytest.raises(ValueError):
        _lib.seed_record(2**300, 0)
    with pytest.raises(ValueError):
        _lib.seed_record(-1, 0)
