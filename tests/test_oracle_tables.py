"""The oracle's independently derived scoring tables equal the product's bit for bit."""

import numpy as np
import pytest

from oracle.tables import OracleTables
from paper_2304_09781_b200.errors import ProfileError
from paper_2304_09781_b200.profiles import (FAMILIES, ServiceRow, VariantSpec, ProfileTable, intensity_at,
                                            CarbonTrace, load_trace, synthetic_profile, synthetic_trace)
from paper_2304_09781_b200.core import SliceType, SLICE_ORDER


@pytest.mark.parametrize("family", sorted(FAMILIES))
def test_tables_identical(family):
    p = synthetic_profile(family)
    a, b = p.scoring_tables(), OracleTables.from_profile(p)
    for f in ("thr_q", "acc_q", "en_q", "idle_q", "mem_ok"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.lat95.view(np.uint64), b.lat95.view(np.uint64))
    assert (a.kt, a.ke, a.ki) == (b.kt, b.ke, b.ki)
    assert a.thr_q.max() < 2 ** 31 and a.en_q.max() < 2 ** 31


def test_profile_invariants():
    p = synthetic_profile("efficientnet")
    # accuracy strictly increasing; latency non-increasing with slice size
    acc = [v.accuracy for v in p.variants]
    assert all(x < y for x, y in zip(acc, acc[1:]))
    for v in range(1, 8):
        means = [p.mean_service_ms(v, s) for s in sorted(SLICE_ORDER, key=int)]
        assert all(x >= y for x, y in zip(means, means[1:]))
    bert = synthetic_profile("bert")
    # memory 12 GB variant: infeasible on 1g and 2g
    assert not bert.memory_feasible(6, SliceType.S1G) and not bert.memory_feasible(6, SliceType.S2G)
    assert bert.memory_feasible(6, SliceType.S3G)
    bad = [VariantSpec(1, 0.8, 1.0), VariantSpec(2, 0.7, 1.0)]
    rows = {(v, s): ServiceRow(10.0) for v in (1, 2) for s in SLICE_ORDER}
    with pytest.raises(ProfileError):
        ProfileTable("bad", bad, rows, {s: 1.0 for s in SLICE_ORDER})


def test_trace_ops(tmp_path):
    t = CarbonTrace([(0, 500), (3600, 100)])
    assert intensity_at(t, 1800) == 500 and intensity_at(t, 3600) == 100 and intensity_at(t, 7200) == 100
    assert intensity_at(t, -5) == 500
    f = tmp_path / "t.csv"
    f.write_text("timestamp_s,gco2_per_kwh\n0,500\n3600,100\n")
    assert len(load_trace(str(f))) == 2
    tr = synthetic_trace()
    assert len(tr) == 288 and all(50 <= c <= 600 for _, c in tr.samples)
