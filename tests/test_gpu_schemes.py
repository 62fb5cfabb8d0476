"""run_trace for every scheme (reference SPEC.md:506-560, 592-631) and the comparison
report: BASE never re-optimises and keeps a_base; CO2OPT's total carbon is at
most BASE's; timelines are deterministic and cumulative carbon is monotone."""

import pytest

from paper_2304_09781_b200.controller import ControllerParams, run_trace
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile, synthetic_trace
from paper_2304_09781_b200 import reports as R

pytestmark = pytest.mark.gpu


def test_all_schemes_and_comparison(engine, tmp_path):
    prof = synthetic_profile("efficientnet")
    tr = synthetic_trace(hours=3.0)
    ap = AnnealParams(proposal="uniform", max_steps=16)
    reps = {s: run_trace(engine, tr, s, 8, prof, 0.5, ap, ControllerParams(), seed=11, chains=16)
            for s in ("base", "co2opt", "blover", "clover", "oracle")}
    base = reps["base"]
    assert base.summary["replans"] == 0
    assert all(r["accuracy"] == base.summary["base_accuracy"] for r in base.rows)
    assert reps["co2opt"].summary["total_gco2"] <= base.summary["total_gco2"]
    for rep in reps.values():
        cum = [r["cumulative_gco2"] for r in rep.rows]
        assert all(b >= a for a, b in zip(cum, cum[1:]))
        assert rep.summary["total_gco2"] == cum[-1]
    again = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=11, chains=16)
    R.write_timeline_csv(str(tmp_path / "a.csv"), reps["clover"])
    R.write_timeline_csv(str(tmp_path / "b.csv"), again)
    assert open(tmp_path / "a.csv").read() == open(tmp_path / "b.csv").read()
    rows = R.comparison_rows(list(reps.values()))
    assert [r["scheme"] for r in rows] == list(reps)
    assert rows[0]["carbon_saved_pct"] == 0.0 and rows[0]["p95_norm_to_base"] == 1.0
    assert max(r["carbon_saved_pct"] for r in rows) > 0.0
