"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of NumPy's PCG64 /
SeedSequence streams as the reference consumes them.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import anything under ``oracle/``; the product path never does.

Third-party dependency restated here: NumPy (the reference pins only
``numpy>=1.24``, ``pkg/pyproject.toml:10``; fixtures were generated with
numpy 2.3.5).  The reference draws from it at:

* ``pnn.py:226`` / ``brbpnn.py:309`` — ``np.random.default_rng(seed)``
  (SeedSequence -> PCG64 seeding),
* ``pnn.py:100-103`` / ``brbpnn.py:326-329`` — ``Generator.uniform`` in the
  order W1 (row-major), b1, W2, b2,
* ``pnn.py:238`` — ``Generator.permutation(n)`` once per epoch,
* ``experiment.py:41-50`` — ``SeedSequence(entropy=[...]).generate_state``,
* ``traces.py:231`` — random split permutation.

Published algorithms restated (NumPy ``bit_generator.pyx`` SeedSequence,
``pcg64.h`` PCG-XSL-RR 128/64, ``distributions.c`` ``random_interval`` with
masked rejection over the buffered 32-bit stream, ``_shuffle_raw``
Fisher-Yates from the top index down).  Checked bit-for-bit against
``numpy.random.default_rng`` in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
M128 = (1 << 128) - 1

# SeedSequence hash constants (NumPy bit_generator.pyx)
_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_L = 0xCA01F9DD
_MIX_R = 0x4973F715
_POOL = 4

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def int_to_words(value: int) -> list[int]:
    """Little-endian 32-bit words of a non-negative int ([0] for zero)."""
    if value < 0:
        raise ValueError("entropy must be non-negative")
    if value == 0:
        return [0]
    words = []
    while value:
        words.append(value & M32)
        value >>= 32
    return words


def entropy_words(entropy) -> list[int]:
    if isinstance(entropy, int):
        return int_to_words(entropy)
    out: list[int] = []
    for item in entropy:
        out.extend(int_to_words(int(item)))
    return out


def seed_pool(entropy) -> list[int]:
    """The 4-word mixed pool of SeedSequence(entropy)."""
    words = entropy_words(entropy)
    hc = _INIT_A

    def hashmix(v: int) -> int:
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * _MULT_A) & M32
        v = (v * hc) & M32
        return v ^ (v >> 16)

    def mix(x: int, y: int) -> int:
        r = (_MIX_L * x - _MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(_POOL)]
    for src in range(_POOL):
        for dst in range(_POOL):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(_POOL, len(words)):
        for dst in range(_POOL):
            pool[dst] = mix(pool[dst], hashmix(words[src]))
    return pool


def generate_words32(pool: list[int], n_words: int) -> list[int]:
    hc = _INIT_B
    out = []
    for i in range(n_words):
        v = pool[i % _POOL]
        v = (v ^ hc) & M32
        hc = (hc * _MULT_B) & M32
        v = (v * hc) & M32
        out.append(v ^ (v >> 16))
    return out


def generate_u64(entropy, n: int) -> list[int]:
    w = generate_words32(seed_pool(entropy), 2 * n)
    return [w[2 * i] | (w[2 * i + 1] << 32) for i in range(n)]


def series_seed_words(base_seed: int, app_crc: int, kernel_id: int, bb_id: int, kind_crc: int) -> int:
    """experiment.py:38-50 restated: one u64 from a 5-item entropy list."""
    return generate_u64([base_seed & M64, app_crc, kernel_id, bb_id, kind_crc], 1)[0]


class Pcg64:
    """PCG-XSL-RR 128/64 with NumPy's buffered 32-bit output."""

    def __init__(self, seed: int | None = None, *, state: int = 0, inc: int = 1):
        if seed is not None:
            s = generate_u64(seed, 4)
            initstate = (s[0] << 64) | s[1]
            initseq = (s[2] << 64) | s[3]
            self.inc = ((initseq << 1) | 1) & M128
            self.state = 0
            self._step()
            self.state = (self.state + initstate) & M128
            self._step()
        else:
            self.state, self.inc = state, inc
        self.has32 = False
        self.buf32 = 0

    def _step(self) -> None:
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self) -> int:
        self._step()
        hi, lo = self.state >> 64, self.state & M64
        x = hi ^ lo
        rot = hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.buf32
        v = self.next64()
        self.has32 = True
        self.buf32 = v >> 32
        return v & M32

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform(self, low: float, high: float) -> float:
        return low + (high - low) * self.next_double()

    def interval(self, mx: int) -> int:
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= M32:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    def permutation(self, n: int) -> list[int]:
        arr = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            arr[i], arr[j] = arr[j], arr[i]
        return arr
