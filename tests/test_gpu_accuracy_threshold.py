"""accuracy_threshold_mode (reference SPEC.md:612-627) on the device: candidates whose
dA < -max_loss_pct count as SLA-violating in best tracking (h unchanged), bit-exact
against the oracle, plus the SPEC examples at the ORACLE / controller level."""

from dataclasses import replace

import numpy as np
import pytest

from oracle.evaluator import calibrate, evaluate
from oracle.search import select_best
from oracle.tables import OracleTables
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile, synthetic_trace
from tests.helpers import random_fleet_graphs

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64), np.asarray(b, np.float64).view(np.uint64))


@pytest.mark.parametrize("loss", [0.0, 0.5, 3.0])
def test_score_graphs_with_threshold_bit_exact(engine, loss):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    sc = replace(calibrate(prof, T, 8, 350.0, 0.5), max_accuracy_loss_pct=loss)
    W = random_fleet_graphs(T, 8, 3000, seed=41)
    best, outs = engine.score_graphs(W, prof, sc)
    ev = evaluate(W, T, sc)
    feas = outs["feasible"].cpu().numpy().astype(bool)
    assert np.array_equal(outs["sla"].cpu().numpy()[feas].astype(bool), ev.sla[feas])
    assert bits_equal(outs["h"].cpu().numpy()[feas], ev.h[feas])
    assert best["index"] == select_best(np.where(feas, ev.h, np.inf), ev.sla & feas)
    dA = (ev.A - sc.obj.base_accuracy) * (100.0 / sc.obj.base_accuracy)
    assert not np.any(ev.sla & (dA < -loss))


def test_oracle_examples(engine):
    prof = synthetic_profile("efficientnet")
    sc = engine.calibrate(prof, 1, 400.0, 0.5)
    plain = engine.oracle_search(prof, sc)
    # max_loss_pct = 100 never binds: identical output
    same = engine.oracle_search(prof, replace(sc, max_accuracy_loss_pct=100.0))
    assert (same["index"], same["f"], same["h"]) == (plain["index"], plain["f"], plain["h"])
    # max_loss_pct = 0 leaves only configurations of the largest variant
    zero = engine.oracle_search(prof, replace(sc, max_accuracy_loss_pct=0.0))
    assert zero["found"] and zero["sla_met"]
    _cid, assign = engine.oracle_decode(prof, zero["index"])
    assert set(assign) == {prof.variant_count}


def test_controller_never_deploys_beyond_the_threshold(engine):
    from paper_2304_09781_b200.controller import ControllerParams, run_trace
    prof = synthetic_profile("efficientnet")
    tr = synthetic_trace(hours=2.0)
    ap = AnnealParams(proposal="uniform", max_steps=16)
    for loss in (0.2, 0.8):
        rep = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=3, chains=16,
                        max_acc_loss_pct=loss)
        a_base = rep.summary["base_accuracy"]
        assert all((r["accuracy"] - a_base) * (100.0 / a_base) >= -loss - 1e-12 for r in rep.rows)
    free = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=3, chains=16)
    capped = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=3, chains=16,
                       max_acc_loss_pct=100.0)
    assert [r["accuracy"] for r in free.rows] == [r["accuracy"] for r in capped.rows]
