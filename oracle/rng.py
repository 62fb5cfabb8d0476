"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Counter-based randomness and deterministic exp.

derive_seed restates reference core.py:107-118.  The stream / bounded-draw /
exp definitions are DESIGN.md's; the kernels implement
the same integer and IEEE operation sequences.
"""

from __future__ import annotations

import math

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def derive_seed(*parts: int) -> int:
    h = 0x9E3779B97F4A7C15
    for p in parts:
        h = ((h ^ (p & M64)) * 0xBF58476D1CE4E5B9) & M64
        h ^= h >> 31
        h = (h * 0x94D049BB133111EB) & M64
    return h & ((1 << 63) - 1)


def stream_word(h0: int, j: int) -> int:
    """splitmix64 output j of the stream keyed by h0."""
    z = (h0 + (j + 1) * GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Stream:
    """32-bit draws: low half then high half of each 64-bit stream word."""

    def __init__(self, h0: int):
        self.h0 = h0
        self.k = 0
        self.word = 0

    def draw32(self) -> int:
        j, half = divmod(self.k, 2)
        if half == 0:
            self.word = stream_word(self.h0, j)
            out = self.word & 0xFFFFFFFF
        else:
            out = self.word >> 32
        self.k += 1
        return out

    def bounded(self, k: int) -> int:
        return (self.draw32() * k) >> 32


def uniform01(seed63: int) -> float:
    return (seed63 >> 10) * (1.0 / 9007199254740992.0)


_LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
_LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
_INV_LN2 = float.fromhex("0x1.71547652b82fep+0")
_C = [1.0 / math.factorial(k) for k in range(13, 1, -1)]


def exp_clv(x: float) -> float:
    if x < -708.0:
        return 0.0
    k = math.floor(x * _INV_LN2 + 0.5)
    r = (x - k * _LN2_HI) - k * _LN2_LO
    p = _C[0]
    for c in _C[1:]:
        p = p * r + c
    p = p * r + 1.0
    p = p * r + 1.0
    return math.ldexp(p, int(k))
