"""Oracle feasibility (C sum-set DP) pinned to the reference's ordered search."""

import json
import os

import numpy as np

from oracle.feasibility import FeasOracle, dfs_partition
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_l0.json")))
SURVEY_COUNTS = [19, 150, 690, 2238, 5771, 12725, 25080, 45443, 77138, 124293, 191927, 286037]


def test_counts_match_reference_and_survey():
    fo = FeasOracle(DEFAULT_TOPOLOGY, 12)
    for n_str, c in GOLDEN["feasible_counts"].items():
        assert fo.count_F(int(n_str)) == c
    assert [fo.count_F(n) for n in range(1, 13)] == SURVEY_COUNTS


def test_dfs_restatement_matches_golden_partitions():
    for n_str, block in GOLDEN["partition_fleet"].items():
        for key, exp in block["feasible"].items():
            v = tuple(int(x) for x in key.split(","))
            assert list(dfs_partition(DEFAULT_TOPOLOGY, v, int(n_str))) == exp


def test_dp_equals_dfs_exhaustive_small():
    fo = FeasOracle(DEFAULT_TOPOLOGY, 5)
    for n in range(1, 6):
        vecs = [(a, b, c, d, e) for a in range(n + 1) for b in range(7 * n // 4 + 1)
                for c in range(7 * n // 3 + 1) for d in range(7 * n // 2 + 1)
                for e in range(max(0, 7 * n - 7 * a - 4 * b - 3 * c - 2 * d) + 1)
                if 7 * a + 4 * b + 3 * c + 2 * d <= 7 * n]
        got = fo.feasible_batch(np.array(vecs), n)
        exp = np.array([DEFAULT_TOPOLOGY.is_feasible_vector(v, n) for v in vecs])
        assert np.array_equal(got, exp), n


def test_host_partition_greedy_matches_dfs_random():
    rng = np.random.default_rng(11)
    for n in (6, 8, 10):
        for _ in range(40):
            v = (int(rng.integers(0, 2)), int(rng.integers(0, n)), int(rng.integers(0, n)),
                 int(rng.integers(0, 2 * n)), int(rng.integers(0, 3 * n)))
            assert DEFAULT_TOPOLOGY.partition_vector(v, n) == dfs_partition(DEFAULT_TOPOLOGY, v, n)
