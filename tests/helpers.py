"""Shared seeded generators for the parity tests."""

import numpy as np

from oracle.search import draw_candidate, fleet_graph, Pod
from oracle.tables import OracleTables
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY


def random_fleet_graphs(tables: OracleTables, n: int, count: int, seed: int, V=None):
    """Realizable graphs: uniform config id per GPU, uniform memory-feasible variant per slice."""
    pods = [Pod(tables, None, n, 1.0)]
    out = []
    for i in range(count):
        (parts, assign), = draw_candidate(seed, i, pods, DEFAULT_TOPOLOGY)
        out.append(fleet_graph(parts, assign, DEFAULT_TOPOLOGY, tables))
    return np.array(out, dtype=np.int64)


def perturbed_graphs(base: np.ndarray, count: int, seed: int):
    """Random integer graphs near realizable ones (many infeasible) for mask tests."""
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, len(base), count)
    W = base[idx].copy()
    for k in range(3):
        e1 = rng.integers(0, W.shape[1], count)
        e2 = rng.integers(0, W.shape[1], count)
        take = W[np.arange(count), e1] > 0
        W[np.arange(count)[take], e1[take]] -= 1
        W[np.arange(count)[take], e2[take]] += 1
    return W
