"""Profile ingestion and the report writers on CPU."""

import csv
import json
import os

import numpy as np
import pytest

from paper_2304_09781_b200.controller import TimelineReport
from paper_2304_09781_b200.core import SliceType
from paper_2304_09781_b200.engine import LOG_DTYPE
from paper_2304_09781_b200.errors import ProfileError
from paper_2304_09781_b200.profiles import load_profiles, profile_from_dict, save_profile, synthetic_profile
from paper_2304_09781_b200 import reports as R


def doc3(acc=(0.7, 0.75, 0.8), mem=(1.0, 4.0, 12.0)):
    labels = [s.label for s in SliceType]
    return {
        "name": "three",
        "variants": [{"id": v + 1, "accuracy": acc[v], "memory_gb": mem[v]} for v in range(3)],
        "latency": [{"variant": v, "slice": s, "mean_service_ms": 10.0 * v * (8 - SliceType.from_label(s).compute_units),
                     "dist": "deterministic"} for v in (1, 2, 3) for s in labels],
        "energy": [{"variant": v, "slice": s, "wh_per_request": 0.001 * v} for v in (1, 2, 3) for s in labels],
        "idle": [{"slice": s, "watts": 5.0 * SliceType.from_label(s).compute_units} for s in labels],
    }


def test_well_formed_file_and_memory_mask(tmp_path):
    p = tmp_path / "p.json"
    p.write_text(json.dumps(doc3()))
    t = load_profiles(str(p))
    assert len(t.service) == 15                                   # 3 variants x 5 slices
    # memory_gb = 12 -> S1g (5 GB) and S2g (10 GB) infeasible, S3g (20 GB) feasible
    assert not t.memory_feasible(3, SliceType.from_label("1g")) and not t.memory_feasible(3, SliceType.from_label("2g"))
    assert t.memory_feasible(3, SliceType.from_label("3g"))
    assert t.memory_feasible(2, SliceType.from_label("1g"))


def test_yaml_document(tmp_path):
    yaml = pytest.importorskip("yaml")
    p = tmp_path / "p.yaml"
    p.write_text(yaml.safe_dump(doc3()))
    assert load_profiles(str(p)).to_json_dict() == profile_from_dict(doc3()).to_json_dict()


def test_round_trip(tmp_path):
    for fam in ("efficientnet", "resnet", "bert"):
        prof = synthetic_profile(fam)
        f = tmp_path / (fam + ".json")
        save_profile(prof, str(f))
        again = load_profiles(str(f))
        assert again.to_json_dict() == prof.to_json_dict()
        assert again.scoring_tables().thr_q.tolist() == prof.scoring_tables().thr_q.tolist()


@pytest.mark.parametrize("mutate", [
    lambda d: d["variants"].__setitem__(1, dict(d["variants"][1], accuracy=0.6)),     # non-monotone accuracy
    lambda d: d["latency"].append(dict(d["latency"][0])),                              # duplicate row
    lambda d: d["energy"].pop(),                                                      # latency/energy mismatch
    lambda d: d.pop("idle"),                                                          # missing section
    lambda d: d["latency"][0].pop("mean_service_ms"),                                 # missing field
    lambda d: d["latency"][0].__setitem__("slice", "9g"),                             # unknown slice
    lambda d: d["latency"][0].__setitem__("dist", "gamma"),                           # unknown distribution
])
def test_schema_errors(mutate):
    d = doc3()
    mutate(d)
    with pytest.raises(ProfileError):
        profile_from_dict(d)


def test_evals_csv(tmp_path):
    log = np.zeros((2, 4), dtype=LOG_DTYPE)
    log["iter"] = np.arange(4)
    log["temp"] = [1.0, 0.95, 0.9, 0.85]
    log["h"] = -1.5
    log["accepted"] = 1
    f = tmp_path / "evals.csv"
    assert R.write_evals_csv(str(f), log[:1], steps=[3]) == 3
    rows = list(csv.reader(open(f)))
    assert rows[0] == list(R.EVAL_FIELDS)                      # SPEC:487 header
    assert rows[1][:2] == ["0", "1.0"] and rows[3][1] == "0.9" and rows[1][7] == "1"
    assert R.write_evals_csv(str(f), log) == 8
    assert list(csv.reader(open(f)))[0][0] == "chain"


def _report(scheme, carbon, acc_delta, p95):
    r = TimelineReport()
    r.rows = [dict(t=float(i), ci=100.0, scheme=scheme, p95_ms=p95, sla_met=True, accuracy=0.8,
                   gco2_per_request=0.1, cumulative_gco2=0.1 * (i + 1), optimizing=False) for i in range(3)]
    r.summary = dict(scheme=scheme, carbon_saved_vs_base_pct=carbon, accuracy_delta_vs_base_pct=acc_delta,
                     total_gco2=0.3, mean_accuracy=0.8, replans=0, candidates_scored=0, sla_violation_ticks=0)
    return r


def test_timeline_summary_comparison(tmp_path):
    reps = [_report("base", 0.0, 0.0, 50.0), _report("clover", 42.0, -1.0, 40.0)]
    rows = R.comparison_rows(reps)
    assert rows[0]["p95_norm_to_base"] == 1.0 and rows[1]["p95_norm_to_base"] == 0.8
    R.write_comparison_csv(str(tmp_path / "comparison.csv"), rows)
    got = list(csv.reader(open(tmp_path / "comparison.csv")))
    assert got[0] == list(R.COMPARISON_FIELDS) and got[2][0] == "clover" and got[2][1] == "42.0"
    R.write_trace_run(str(tmp_path / "out"), reps[1])
    for name in ("timeline.csv", "summary.json", "evals.csv"):
        assert os.path.exists(tmp_path / "out" / name)
    a = open(tmp_path / "out" / "timeline.csv").read()
    R.write_trace_run(str(tmp_path / "out2"), reps[1])
    assert a == open(tmp_path / "out2" / "timeline.csv").read()          # byte-identical
    assert json.load(open(tmp_path / "out" / "summary.json"))["scheme"] == "clover"
