"""Seeded generator of the drop-in API (reference rng.py:25-67).

Every synthetic input (arrival gaps, output lengths, prompt tokens) is drawn
from xorshift64* seeded through one splitmix64 round, so schedules reproduce
bit for bit from (parameters, seed).  Bit-equality with the reference is
pinned by tests/test_host_api.py against tests/golden/rng.json.
"""

from __future__ import annotations

import math

_M = 0xFFFFFFFFFFFFFFFF
_PHI = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB
_STAR = 0x2545F4914F6CDD1D
_INV53 = 2.0 ** -53


def _finalize(z: int) -> int:
    z = ((z ^ (z >> 30)) * _C1) & _M
    z = ((z ^ (z >> 27)) * _C2) & _M
    return z ^ (z >> 31)


def derive_seed(seed: int, stream: int) -> int:
    """Fold a stream tag into a user seed (two splitmix64 rounds)."""
    tag = _finalize((stream + _PHI) & _M)
    return _finalize((((seed & _M) ^ tag) + _PHI) & _M)


class Xorshift64Star:
    """Vigna's xorshift64* (12/25/27, multiplier 0x2545F4914F6CDD1D)."""

    __slots__ = ("_s",)

    def __init__(self, seed: int, stream: int = 0):
        self._s = derive_seed(seed, stream) or _PHI

    def next_u64(self) -> int:
        s = self._s
        s ^= s >> 12
        s = (s ^ (s << 25)) & _M
        s ^= s >> 27
        self._s = s
        return (s * _STAR) & _M

    def next_float(self) -> float:
        return (self.next_u64() >> 11) * _INV53

    def exponential(self, mean: float) -> float:
        return -mean * math.log1p(-self.next_float())

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + int(self.next_float() * (hi - lo + 1))
