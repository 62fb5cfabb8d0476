"""Fleet feasibility at n = 16, 32, 64 against the REFERENCE (mig.py:144-181,
MigTopology.partition_fleet), SURVEY 4.4 / VERDICT r01 item 5: golden cases from
tests/golden/make_feas_large.py (random slice vectors, half of them drawn at the capacity
boundary, each answered by the reference under a per-query time limit).

CPU: the oracle's sum-set DP (oracle/feas.c) gives the reference's answer on every case, and
the host data model's canonical partition (paper_2304_09781_b200/mig.py) equals the reference's
smallest ascending id tuple.  GPU: the device tables (clv_feasible, K6) give the same answers,
and clv_realize returns the reference's canonical partition."""
import json
import os

import numpy as np
import pytest

from oracle.feasibility import FeasOracle
from paper_2304_09781_b200.core import SLICE_ORDER
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY

PATH = os.path.join(os.path.dirname(__file__), "golden", "feas_large.json")


def _cases():
    with open(PATH) as fh:
        d = json.load(fh)
    assert d["slice_order"] == [s.label for s in SLICE_ORDER]
    return d


@pytest.fixture(scope="module")
def golden():
    return _cases()


@pytest.fixture(scope="module")
def feas64():
    return FeasOracle(DEFAULT_TOPOLOGY, 64)


def _by_n(golden, n):
    rows = [c for c in golden["cases"] if c[0] == n]
    vec = np.array([c[1:6] for c in rows], dtype=np.int32)
    part = [c[6] for c in rows]
    return vec, part


def test_fixture_shape(golden):
    for n in (16, 32, 64):
        vec, part = _by_n(golden, n)
        assert len(vec) >= 4000
        assert sum(p is None for p in part) > 0 or n > 16   # infeasible cases present


@pytest.mark.parametrize("n", [16, 32, 64])
def test_oracle_dp_matches_reference(golden, feas64, n):
    vec, part = _by_n(golden, n)
    got = feas64.feasible_batch(vec, n)
    want = np.array([p is not None for p in part])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [16, 32, 64])
def test_host_canonical_partition_matches_reference(golden, n):
    vec, part = _by_n(golden, n)
    for v, p in list(zip(vec, part))[:1500]:
        slices = [s for s, c in zip(SLICE_ORDER, v) for _ in range(int(c))]
        got = DEFAULT_TOPOLOGY.partition_fleet(slices, n)
        assert (None if got is None else list(got)) == p


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 32, 64])
def test_device_feasibility_and_realize_match_reference(golden, engine, n):
    vec, part = _by_n(golden, n)
    engine.build_feasibility(64)
    got = engine.feasible(vec, n).cpu().numpy().astype(bool)
    assert np.array_equal(got, np.array([p is not None for p in part]))
    feas = [(v, p) for v, p in zip(vec, part) if p is not None]
    for v, p in feas[:300]:
        assert list(engine.partition(v, n)) == p
