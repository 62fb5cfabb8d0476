"""The SPEC-signature entry points (reference SPEC.md:196, 206, 461, 526, 536) through
search.py, against the oracle: anneal, oracle_search, blover_search, realize."""

import numpy as np
import pytest

from oracle.anneal import anneal_chain
from oracle.tables import OracleTables
from paper_2304_09781_b200 import search as SP
from paper_2304_09781_b200.core import ObjectiveParams
from paper_2304_09781_b200.graph import ConfigGraph, build_graph
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile
from tests.helpers import random_fleet_graphs

pytestmark = pytest.mark.gpu


def _setup(engine, n):
    prof = synthetic_profile("efficientnet")
    sc = engine.calibrate(prof, n, 350.0, 0.5)
    wl = SP.Workload(sc.arrival_rps)
    return prof, sc, wl, sc.obj


def test_anneal_spec_signature_matches_oracle(engine, feas64):
    n = 8
    prof, sc, wl, obj = _setup(engine, n)
    T = OracleTables.from_profile(prof)
    start = ConfigGraph(random_fleet_graphs(T, n, 1, seed=12)[0], T.V, prof.name)
    for ap in (None, AnnealParams(max_steps=20)):                   # SPEC-literal default, full neighbourhood
        best, log, sim_time = SP.anneal(start, n, prof, wl, 350.0, obj, ap, rng=99, engine=engine)
        ap_eff = ap or AnnealParams(proposal="uniform", evaluate="proposal")
        sc_eff = SP.scenario_for(n, wl, 350.0, obj)
        ref = anneal_chain(np.array(start.weights), n, T, sc_eff, ap_eff, 99, 0, feas64)
        assert np.array_equal(np.array(best.graph.weights), ref.best_w)
        assert len(log) == ref.steps
        n_evals = ref.evals if ap_eff.evaluate == "proposal" else 1 + ref.steps
        assert sim_time == n_evals * ap_eff.eval_cost_s
        if ap is None:
            assert sim_time <= ap_eff.time_budget_s + ap_eff.eval_cost_s   # <= 7 evaluations


def test_oracle_search_and_realize(engine):
    n = 4
    prof, sc, wl, obj = _setup(engine, n)
    res = SP.oracle_search(n, prof, wl, 350.0, obj, engine=engine)
    ref = engine.oracle_search(prof, SP.scenario_for(n, wl, 350.0, obj))
    assert res.f_value == ref["f"] and res.h_value == ref["h"] and res.sla_met == bool(ref["sla_met"])
    fc = SP.realize(res.graph, n, engine=engine)
    assert build_graph(fc, prof) == res.graph and fc.n_gpus == n
    assert fc.partitions == tuple(DEFAULT_TOPOLOGY.partition_vector(res.graph.slice_vector(), n))


def test_blover_search_log_and_best(engine):
    n = 8
    prof, sc, wl, obj = _setup(engine, n)
    best, log = SP.blover_search(n, prof, wl, 350.0, obj, rng=5, engine=engine)
    assert 1 <= len(log) <= 7                                        # 300 s / 45 s budget
    nb = [r for r in log if r["new_best"]]
    assert nb and best.h_value == nb[-1]["h"] and best.sla_met == nb[-1]["sla_met"]
    assert log[0]["new_best"]
