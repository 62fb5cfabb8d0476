"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Fleet feasibility (reference mig.py:144-181).

``FeasOracle`` wraps the C sum-set DP in feas.c; ``dfs_partition`` is a direct
restatement of the reference's ordered memoised backtracking for small n
(used to pin the DP and the product's host search).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libclv_oracle_feas.so")
_lib = None


def build() -> str:
    src = os.path.join(_HERE, "feas.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.feas_build.restype = ctypes.c_void_p
        lib.feas_build.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.feas_free.argtypes = [ctypes.c_void_p]
        lib.feas_query.restype = ctypes.c_int
        lib.feas_query.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 6
        lib.feas_query_batch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_void_p]
        lib.feas_count_T.restype = ctypes.c_int64
        lib.feas_count_T.argtypes = [ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


class FeasOracle:
    """Exact 'sum of exactly n table rows' predicate for n <= nmax."""

    def __init__(self, topology, nmax: int):
        lib = _load()
        rows = np.ascontiguousarray(np.array(topology.config_vectors, dtype=np.int32))
        self._rows = rows
        self._h = lib.feas_build(rows.ctypes.data, len(rows), int(nmax))
        if not self._h:
            raise ValueError("feas_build failed")
        self.nmax = int(nmax)
        self._cache: dict = {}

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.feas_free(self._h)
            self._h = None

    def feasible(self, vec, n: int) -> bool:
        key = (tuple(int(x) for x in vec), int(n))
        hit = self._cache.get(key)
        if hit is None:
            r = _lib.feas_query(self._h, int(n), *key[0])
            if r < 0:
                raise ValueError("n=%d beyond the oracle table (nmax=%d)" % (n, self.nmax))
            hit = bool(r)
            self._cache[key] = hit
        return hit

    def feasible_batch(self, vecs: np.ndarray, n: int) -> np.ndarray:
        v = np.ascontiguousarray(vecs, dtype=np.int32).reshape(-1, 5)
        out = np.zeros(len(v), dtype=np.uint8)
        _lib.feas_query_batch(self._h, int(n), v.ctypes.data, len(v), out.ctypes.data)
        return out.astype(bool)

    def count_T(self, N: int) -> int:
        return int(_lib.feas_count_T(self._h, int(N)))

    def count_F(self, n: int) -> int:
        return sum(self.count_T(n - a) for a in range(0, n + 1))


def dfs_partition(topology, vec, n: int):
    """Restatement of the reference's ordered backtracking (mig.py:144-170), small n only."""
    rows = list(zip(topology.config_ids, topology.config_vectors))

    @lru_cache(maxsize=None)
    def search(rem, left, lo):
        if left == 0:
            return () if not any(rem) else None
        tot = sum(rem)
        if tot < left or tot > 7 * left:
            return None
        for i in range(lo, len(rows)):
            cid, row = rows[i]
            if all(r >= c for r, c in zip(rem, row)):
                sub = search(tuple(r - c for r, c in zip(rem, row)), left - 1, i)
                if sub is not None:
                    return (cid,) + sub
        return None

    if n < 1:
        return None
    return search(tuple(int(x) for x in vec), int(n), 0)
