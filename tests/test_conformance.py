"""Data-model conformance with the reference (core.py, mig.py, errors.py).

Against the committed golden vectors (tests/golden/reference_l0.json, made by
tests/golden/make_golden.py from the reference) and, when /root/reference is
present, against the live reference package.
"""

import itertools
import json
import math
import os
import sys

import pytest

from paper_2304_09781_b200 import core, errors, mig
from paper_2304_09781_b200.core import SLICE_ORDER, ObjectiveParams, SliceType, derive_seed
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY, FleetConfig, from_slice_vector

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_l0.json")))


def test_derive_seed_golden():
    for parts, val in GOLDEN["derive_seed"]:
        assert derive_seed(*parts) == val


def test_slice_types():
    assert [int(s) for s in SLICE_ORDER] == GOLDEN["slice_order"]
    assert {s.label: int(s) for s in SliceType} == GOLDEN["labels"]
    assert SliceType.from_label("3g") is SliceType.S3G
    with pytest.raises(errors.CarbonSchedError):
        SliceType.from_label("5g")


def test_topology_table_and_anchors():
    assert DEFAULT_TOPOLOGY.to_json_dict() == GOLDEN["topology"]
    assert list(DEFAULT_TOPOLOGY.config_ids) == GOLDEN["config_ids"]
    # SPEC:106-120 anchors
    S = SliceType
    assert DEFAULT_TOPOLOGY.config_slices(19) == (S.S1G,) * 7
    assert sorted(DEFAULT_TOPOLOGY.config_slices(10)) == sorted((S.S3G, S.S2G, S.S1G, S.S1G))
    assert DEFAULT_TOPOLOGY.config_slices(3) == (S.S4G, S.S2G, S.S1G)
    assert DEFAULT_TOPOLOGY.config_slices(1) == (S.S7G,)
    assert [DEFAULT_TOPOLOGY.slice_memory(s) for s in (S.S1G, S.S2G, S.S7G)] == [5.0, 10.0, 40.0]
    with pytest.raises(errors.InvalidConfigError):
        DEFAULT_TOPOLOGY.config_slices(20)
    for cid in DEFAULT_TOPOLOGY.config_ids:
        sl = DEFAULT_TOPOLOGY.config_slices(cid)
        assert sum(int(s) for s in sl) <= 7 and len(sl) <= 7


def test_partition_fleet_golden_exhaustive():
    for n_str, block in GOLDEN["partition_fleet"].items():
        n = int(n_str)
        feas = block["feasible"]
        checked = 0
        for a in range(n + 1):
            for b in range(7 * n // 4 + 1):
                for c in range(7 * n // 3 + 1):
                    for d in range(7 * n // 2 + 1):
                        rem = 7 * n - 7 * a - 4 * b - 3 * c - 2 * d
                        for e in range(rem + 1) if rem >= 0 else []:
                            checked += 1
                            key = "%d,%d,%d,%d,%d" % (a, b, c, d, e)
                            got = DEFAULT_TOPOLOGY.partition_fleet(from_slice_vector((a, b, c, d, e)), n)
                            exp = feas.get(key)
                            assert (list(got) if got is not None else None) == exp, (key, n)
        assert checked == block["checked"]


def test_feasibility_kats_and_closure():
    S = SliceType
    for labels, n, exp in GOLDEN["feasible_kats"]:
        assert mig.is_feasible_fleet([S.from_label(x) for x in labels], n) == exp
    # closure under union of any two rows
    for a, b in itertools.product(DEFAULT_TOPOLOGY.config_ids, repeat=2):
        sl = DEFAULT_TOPOLOGY.config_slices(a) + DEFAULT_TOPOLOGY.config_slices(b)
        assert DEFAULT_TOPOLOGY.is_feasible_fleet(sl, 2)


def test_objective_params_golden():
    for kw, outcome, lam in GOLDEN["objective_params"]:
        kw = {k: (float(v) if isinstance(v, str) else v) for k, v in kw.items()}
        if outcome == "ok":
            assert ObjectiveParams(**kw).carbon_weight == lam
        else:
            with pytest.raises(getattr(errors, outcome)):
                ObjectiveParams(**kw)


def test_fleet_config_golden():
    for fx in GOLDEN["fleets"]:
        fc = FleetConfig(fx["partitions"], fx["assignments"])
        assert [[g, int(s)] for g, s in fc.slices()] == fx["slices"]
        assert [[g, int(s), v] for g, s, v in fc.instances()] == fx["instances"]
        assert {str(int(k)): v for k, v in fc.slice_counts().items()} == fx["slice_counts"]
        assert fc.n_gpus == len(fx["partitions"]) and fc.n_instances == len(fx["assignments"])
    for p, a, outcome in GOLDEN["fleet_errors"]:
        with pytest.raises(getattr(errors, outcome)):
            FleetConfig(p, a)


CTOR_OUTCOME = {"invalid_config": "InvalidConfigError", "length": "CarbonSchedError",
                "variant_lt1": "CarbonSchedError", "infeasible": "ok", None: "ok"}


def test_fleet_error_precedence_golden():
    """Rows with several defects: FleetConfig here and the oracle's fleet_row_error (the
    checker of clv_score_x's error reporting) both follow the reference's order."""
    from oracle.search import fleet_row_error
    from oracle.tables import OracleTables
    from paper_2304_09781_b200.profiles import synthetic_profile
    T = OracleTables.from_profile(synthetic_profile("bert"))
    for p, a, outcome in GOLDEN["fleet_error_precedence"]:
        assert CTOR_OUTCOME[fleet_row_error(p, a, DEFAULT_TOPOLOGY, T)] == outcome, (p, a)
        if outcome == "ok":
            FleetConfig(p, a)
        else:
            with pytest.raises(errors.CarbonSchedError) as ei:
                FleetConfig(p, a)
            assert type(ei.value).__name__ == outcome


def test_load_topology_roundtrip(tmp_path):
    path = tmp_path / "topo.json"
    path.write_text(json.dumps(DEFAULT_TOPOLOGY.to_json_dict()))
    t = mig.load_topology(str(path))
    assert t.to_json_dict() == DEFAULT_TOPOLOGY.to_json_dict()
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"configs": {"1": ["7g"]}, "memory_gb": {"7g": 40}}))
    with pytest.raises(errors.InvalidConfigError):
        mig.load_topology(str(bad))


@pytest.mark.reference
def test_live_reference_equivalence():
    sys.path.insert(0, "/root/reference/pkg/src")
    from carbon_sched import core as rcore, mig as rmig
    import random
    rnd = random.Random(5)
    for _ in range(500):
        parts = [rnd.getrandbits(64) for _ in range(rnd.randint(0, 6))]
        assert derive_seed(*parts) == rcore.derive_seed(*parts)
    for n in (5, 6):
        for _ in range(300):
            v = (rnd.randint(0, 1), rnd.randint(0, n), rnd.randint(0, n), rnd.randint(0, 2 * n), rnd.randint(0, 4 * n))
            got = DEFAULT_TOPOLOGY.partition_vector(v, n)
            exp = rmig.DEFAULT_TOPOLOGY.partition_fleet(rmig.from_slice_vector(v), n)
            assert got == exp
