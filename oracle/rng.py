"""ORACLE (test infrastructure): restated numpy Philox4x64-10 + Generator draws.

Restates the third-party algorithm the reference stream wraps
(``simt_forge/rng.py:29-32`` builds ``np.random.Generator(np.random.Philox(key=[seed, sid]))``):

* Philox4x64 with 10 rounds, Random123 constants (numpy ``philox.h``),
* the bit generator's 4-word output buffer and 32-bit half-word cache
  (``philox_next64`` / ``philox_next32``),
* ``Generator.random``  = 53-bit double  (``next_double``),
* ``Generator.integers(lo, hi)`` (int64) = Lemire bounded integers with the
  32-bit path for ranges below 2**32 (``random_bounded_uint64_fill``),
* and the stream's convenience draws (rng.py:40-78).

Pure integer python; checked against numpy itself in tests/test_oracle_pins.py.
"""

from __future__ import annotations

M64 = (1 << 64) - 1
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def philox4x64_10(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + PHILOX_W0) & M64
            k1 = (k1 + PHILOX_W1) & M64
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0, p1 & M64, (p0 >> 64) ^ c3 ^ k1, p0 & M64)
    return (c0, c1, c2, c3)


class OracleStream:
    """Same draws as ``simt_forge.rng.Stream(seed, stream_id)``."""

    def __init__(self, seed: int, stream_id: int = 0):
        self.key = (seed & M64, stream_id & M64)
        self.ctr = [0, 0, 0, 0]
        self.buf = (0, 0, 0, 0)
        self.pos = 4
        self.has32 = False
        self.u32cache = 0
        self.words = 0   # 64-bit words consumed (diagnostics only)

    # bit generator -----------------------------------------------------------
    def next64(self) -> int:
        self.words += 1
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & M64
            if self.ctr[i]:
                break
        self.buf = philox4x64_10(self.ctr, self.key)
        self.pos = 1
        return self.buf[0]

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.u32cache
        v = self.next64()
        self.has32 = True
        self.u32cache = v >> 32
        return v & 0xFFFFFFFF

    # Generator ---------------------------------------------------------------
    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def integers(self, lo: int, hi: int) -> int:
        if hi <= lo:
            raise ValueError("empty range")
        rng = (hi - lo - 1) & M64
        if rng == 0:
            return lo
        if rng <= 0xFFFFFFFF:
            if rng == 0xFFFFFFFF:
                return lo + self.next32()
            ex = rng + 1
            m = self.next32() * ex
            if (m & 0xFFFFFFFF) < ex:
                thr = (0xFFFFFFFF - rng) % ex
                while (m & 0xFFFFFFFF) < thr:
                    m = self.next32() * ex
            return lo + (m >> 32)
        if rng == M64:
            return lo + self.next64()
        ex = rng + 1
        m = self.next64() * ex
        if (m & M64) < ex:
            thr = (M64 - rng) % ex
            while (m & M64) < thr:
                m = self.next64() * ex
        return lo + (m >> 64)

    def u64(self) -> int:
        return self.next64()

    def choice(self, seq):
        if not seq:
            raise ValueError("empty sequence")
        return seq[self.integers(0, len(seq))]

    def weighted_choice(self, seq, weights):
        total = float(sum(weights))
        x = self.random() * total
        acc = 0.0
        for item, w in zip(seq, weights):
            acc += w
            if x < acc:
                return item
        return seq[-1]

    def geometric_small(self, p: float, cap: int) -> int:
        n = 0
        while n < cap and self.random() >= p:
            n += 1
        return n
