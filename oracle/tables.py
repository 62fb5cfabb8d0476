"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Independent derivation of the scoring tables.

Restates DESIGN.md "Scoring surrogate" from the raw ProfileTable:
per-edge fixed-point rows thr_q, acc_q, en_q, per-slice idle_q, fp64 lat95 and
the memory mask.  tests/test_oracle_tables.py checks they equal the product's
``ScoringTables`` bit for bit, so the two sides start from identical inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

KINDS = (7, 4, 3, 2, 1)          # SLICE_ORDER compute units (core.py:54-60)


def _p95(row) -> float:
    if row.dist == "deterministic":
        return row.mean_service_ms
    if row.dist == "exponential":
        return row.mean_service_ms * math.log(20.0)
    return row.mean_service_ms * math.exp(1.6448536269514722 * row.sigma - 0.5 * row.sigma * row.sigma)


def _scale(mx: float) -> int:
    return 31 - math.frexp(mx)[1] if mx > 0 else 30


@dataclass
class OracleTables:
    V: int
    thr_q: np.ndarray
    acc_q: np.ndarray
    en_q: np.ndarray
    idle_q: np.ndarray
    lat95: np.ndarray
    mem_ok: np.ndarray
    kt: int
    ke: int
    ki: int
    mean_ms: np.ndarray

    def rate_moment_rows(self):
        """(t2_q, k2, t3_q, k3): fixed-point rows of thr^2 and thr^3, thr = 1000 / mean_ms
        (the second and third moments of the instance service rates)."""
        thr = [1000.0 / float(x) for x in self.mean_ms]
        t2 = [x * x for x in thr]
        t3 = [y * x for x, y in zip(thr, t2)]
        k2, k3 = _scale(max(t2)), _scale(max(t3))
        return (np.array([round(math.ldexp(x, k2)) for x in t2], dtype=np.int64), k2,
                np.array([round(math.ldexp(x, k3)) for x in t3], dtype=np.int64), k3)

    @property
    def E(self) -> int:
        return self.V * 5

    @classmethod
    def from_profile(cls, profile) -> "OracleTables":
        from paper_2304_09781_b200.core import SliceType
        V = profile.variant_count
        thr, lat, at, et, mem, mean = [], [], [], [], [], []
        for v in range(1, V + 1):
            acc = profile.variants[v - 1].accuracy
            for cu in KINDS:
                row = profile.service[(v, SliceType(cu))]
                t = 1000.0 / row.mean_service_ms
                thr.append(t)
                lat.append(_p95(row))
                at.append(t * acc)
                et.append(t * row.energy_wh_per_request)
                mem.append(profile.variants[v - 1].memory_gb <= profile.topology.slice_memory(SliceType(cu)))
                mean.append(row.mean_service_ms)
        idle = [profile.idle_power_w[SliceType(cu)] for cu in KINDS]
        kt, ke, ki = _scale(max(thr)), _scale(max(et)), _scale(max(idle))
        q = lambda xs, k: np.array([round(x * 2.0 ** k) for x in xs], dtype=np.int64)
        return cls(V, q(thr, kt), q(at, kt), q(et, ke), q(idle, ki), np.array(lat),
                   np.array(mem, dtype=bool), kt, ke, ki, np.array(mean))
