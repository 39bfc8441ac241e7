"""O6: Philox4x32-10 counter-based RNG, written from its definition.  TEST INFRASTRUCTURE ONLY.

Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3" (SC'11):
Philox4x32 with R = 10 rounds, multipliers M0 = 0xD2511F53, M1 = 0xCD9E8D57 and Weyl key
increments W0 = 0x9E3779B9, W1 = 0xBB67AE85.  One round maps
(c0, c1, c2, c3) with key (k0, k1) to
    (hi(M1*c2) ^ c1 ^ k0,  lo(M1*c2),  hi(M0*c0) ^ c3 ^ k1,  lo(M0*c0))
and the key is bumped by (W0, W1) between rounds.  Pinned by the published known-answer
vectors (tests/golden/philox_kat.json) and, on the GPU box, by the CUDA toolkit's own
curand_Philox4x32_10.
"""
from __future__ import annotations

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (x & MASK for x in ctr)
    k0, k1 = (x & MASK for x in key)
    for r in range(10):
        if r:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
        p0, p1 = M0 * c0, M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c3 ^ k1) & MASK, p0 & MASK
    return (c0, c1, c2, c3)


class Stream:
    """Sequential u32 draws from counters (c0, c1, c2, block), block = 0, 1, 2, ...

    Word k of the stream is word k % 4 of philox4x32_10((c0, c1, c2, k // 4), key)."""

    def __init__(self, key, c0, c1, c2):
        self.key, self.c = key, (c0, c1, c2)
        self.block, self.buf = 0, []

    def u32(self) -> int:
        if not self.buf:
            self.buf = list(philox4x32_10((*self.c, self.block), self.key))
            self.block += 1
        return self.buf.pop(0)

    def below(self, n: int) -> int:
        """U(n) = (u32 * n) >> 32, an integer in [0, n)."""
        return (self.u32() * n) >> 32
