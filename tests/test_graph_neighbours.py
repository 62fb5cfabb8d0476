"""Graph operations and the GED<=4 neighbourhood definition (acceptance 1-2)."""

import numpy as np
import pytest

from oracle.feasibility import FeasOracle
from oracle.neighbours import brute_force_neighbours, enumerate_neighbours
from oracle.tables import OracleTables
from paper_2304_09781_b200.core import SliceType as S
from paper_2304_09781_b200.errors import IncompatibleGraphsError, InfeasibleAssignmentError
from paper_2304_09781_b200.graph import ConfigGraph, build_graph, ged, merge
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY, FleetConfig
from paper_2304_09781_b200.profiles import synthetic_profile
from tests.helpers import random_fleet_graphs


def G(edges, V):
    return ConfigGraph.from_edges(edges, V)


def test_build_graph_examples():
    assert build_graph(FleetConfig([1], [3]), variant_count=3) == G({(3, S.S7G): 1}, 3)
    fc = FleetConfig([10], [3, 2, 1, 1])
    assert build_graph(fc, variant_count=3) == G({(3, S.S3G): 1, (2, S.S2G): 1, (1, S.S1G): 2}, 3)
    assert build_graph(FleetConfig([19, 19], [1] * 14), variant_count=1) == G({(1, S.S1G): 14}, 1)
    bert = synthetic_profile("bert")
    with pytest.raises(InfeasibleAssignmentError):
        build_graph(FleetConfig([19], [6] * 7), bert)


def test_ged_examples_and_merge():
    g = G({(1, S.S1G): 1}, 2)
    assert ged(g, g) == 0
    assert ged(G({(1, S.S1G): 1}, 2), G({(2, S.S1G): 1}, 2)) == 2
    assert ged(G({(1, S.S1G): 1}, 2), G({(1, S.S2G): 1}, 2)) == 2
    assert ged(G({(1, S.S7G): 1}, 2), G({(2, S.S1G): 7}, 2)) == 8
    assert merge(G({(1, S.S1G): 2}, 1), G({(1, S.S1G): 3}, 1)) == G({(1, S.S1G): 5}, 1)
    assert merge(g, ConfigGraph.empty(2)) == g
    a = build_graph(FleetConfig([1], [3]), variant_count=3)
    b = build_graph(FleetConfig([19, 19], [1] * 14), variant_count=3)
    assert merge(a, b) == build_graph(FleetConfig([1, 19, 19], [3] + [1] * 14), variant_count=3)
    with pytest.raises(IncompatibleGraphsError):
        ged(G({(1, S.S1G): 1}, 1), G({(1, S.S1G): 1}, 2))


def test_ged_metric_axioms():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        V = int(rng.integers(1, 6))
        a, b, c = (ConfigGraph(rng.integers(0, 21, V * 5), V) for _ in range(3))
        assert ged(a, b) >= 0 and (ged(a, b) == 0) == (a == b)
        assert ged(a, b) == ged(b, a)
        assert ged(a, c) <= ged(a, b) + ged(b, c)
        assert ged(merge(a, c), merge(b, c)) == ged(a, b)


@pytest.mark.parametrize("family,n", [("efficientnet", 1), ("efficientnet", 2), ("tiny3", 2), ("bert", 1),
                                      ("resnet", 3)])
def test_canonical_neighbours_equal_brute_force(family, n):
    prof = synthetic_profile(family)
    T = OracleTables.from_profile(prof)
    feas = FeasOracle(DEFAULT_TOPOLOGY, n)
    W = random_fleet_graphs(T, n, 12, seed=n + 17)
    for w in W:
        nb = enumerate_neighbours(w, T.mem_ok, T.V, n, feas)
        got = {tuple(x) for x in nb.W.tolist()}
        assert len(got) == len(nb)                     # no duplicates
        exp = brute_force_neighbours(w, T.mem_ok, T.V, n, feas)
        assert got == exp
        assert np.all(np.diff(nb.idx) > 0)             # canonical order
        d = np.abs(nb.W - w[None, :]).sum(axis=1)
        assert set(d.tolist()) <= {2, 4}               # GED in {2, 4}
        assert np.all(nb.W.sum(axis=1) == w.sum())     # instance count preserved


def test_neighbour_spec_examples():
    feas = FeasOracle(DEFAULT_TOPOLOGY, 2)
    # {(v1,7g):1}, V=1: only slice moves; every neighbour realizable
    w = np.zeros(5, dtype=np.int64); w[0] = 1
    nb = enumerate_neighbours(w, np.ones(5, bool), 1, 1, feas)
    assert len(nb) > 0
    for g in nb.W:
        assert feas.feasible(g, 1)
    # {(v1,1g):7}, n=1, V=2: the swap neighbour {(v1,1g):6,(v2,1g):1} is present with GED 2
    w = np.zeros(10, dtype=np.int64); w[4] = 7
    nb = enumerate_neighbours(w, np.ones(10, bool), 2, 1, feas)
    target = w.copy(); target[4] = 6; target[9] = 1
    assert any(np.array_equal(g, target) for g in nb.W)


def test_paper_move_set_adds_unit_moves():
    """moves="paper" = the SPEC neighbourhood plus every realizable, memory-feasible graph at
    L1 distance 1 (one instance added or removed), with the documented indices."""
    import numpy as np
    from oracle.feasibility import FeasOracle
    from oracle.neighbours import enumerate_neighbours
    from oracle.tables import OracleTables
    from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
    from paper_2304_09781_b200.profiles import synthetic_profile
    from tests.helpers import random_fleet_graphs
    prof = synthetic_profile("bert")
    T = OracleTables.from_profile(prof)
    n = 3
    feas = FeasOracle(DEFAULT_TOPOLOGY, n)
    E = T.E
    NP = E * (E + 1) // 2
    for w in random_fleet_graphs(T, n, 6, seed=9):
        spec = enumerate_neighbours(w, T.mem_ok, T.V, n, feas)
        paper = enumerate_neighbours(w, T.mem_ok, T.V, n, feas, moves="paper")
        extra = paper.idx >= E * E + NP * NP
        assert np.array_equal(paper.idx[~extra], spec.idx)
        unit = set()
        for e in range(E):
            for d in (1, -1):
                g = w.copy(); g[e] += d
                if g[e] < 0 or (d > 0 and not T.mem_ok[e]):
                    continue
                svec = g.reshape(T.V, 5).sum(axis=0)
                if feas.feasible(svec, n):
                    unit.add(tuple(g))
        assert {tuple(x) for x in paper.W[extra]} == unit
        assert (np.abs(paper.W[extra] - w).sum(axis=1) == 1).all() and (paper.ged[extra] == 1).all()
