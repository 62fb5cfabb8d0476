"""SURVEY D2's optional paper move set (one-instance add / remove on top of the SPEC's
GED <= 4 swaps and slice moves) and SPEC:492's multiplicative cooling option,
device chain kernel vs oracle/anneal.py bit for bit (status, steps, evaluations, best and final
graphs, f / h / p95 bits, per-step acceptance, h and temperature logs) in every proposal mode."""
import numpy as np
import pytest

from oracle.evaluator import calibrate, base_graph
from oracle.tables import OracleTables
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile
from tests.helpers import random_fleet_graphs
from tests.test_gpu_parity import _chain_compare

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("proposal,evaluate_mode", [("best", "all"), ("uniform", "all"), ("uniform", "proposal")])
@pytest.mark.parametrize("cooling", ["subtractive", "multiplicative"])
def test_paper_moves_n16(engine, feas64, proposal, evaluate_mode, cooling):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 16
    sc = calibrate(prof, T, n, 380.0, 0.5)
    starts = np.concatenate([random_fleet_graphs(T, n, 5, seed=1601), base_graph(7, n)[None, :]])
    ap = AnnealParams(proposal=proposal, evaluate=evaluate_mode, max_steps=24, move_set="paper", cooling=cooling)
    _chain_compare(engine, prof, T, starts, [sc], ap, 31, n, feas64, cluster=2)


def test_paper_moves_n64(engine, feas64):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 64
    sc = calibrate(prof, T, n, 350.0, 0.5)
    starts = np.concatenate([random_fleet_graphs(T, n, 3, seed=6401), base_graph(7, n)[None, :]])
    ap = AnnealParams(max_steps=16, move_set="paper")
    _chain_compare(engine, prof, T, starts, [sc], ap, 5, n, feas64)


def test_paper_moves_change_instance_count(engine, feas64):
    """Uniform proposals reach the unit moves: accepted GED-1 steps change m (the SPEC move
    set keeps m forever), still bit-exact with the oracle."""
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 8
    sc = calibrate(prof, T, n, 400.0, 0.5)
    starts = random_fleet_graphs(T, n, 8, seed=801)
    ap = AnnealParams(proposal="uniform", evaluate="proposal", max_steps=60, stall_limit=60, move_set="paper",
                      time_budget_s=float("inf"))
    _chain_compare(engine, prof, T, starts, [sc], ap, 17, n, feas64)
    host = engine.anneal(starts, prof, [sc], ap, 17, n=n, log=True).host()
    steps = host["results"]["steps"]
    unit = [bool(((host["log"][c]["ged_from_center"][: steps[c]] == 1) & (host["log"][c]["accepted"][: steps[c]] != 0)).any())
            for c in range(len(starts))]
    assert any(unit)
    assert (starts.sum(axis=1) != host["final_w"].astype(np.int64).sum(axis=1)).any()


def test_multiplicative_temperatures(engine, feas64):
    """T_k = max(t_floor, t_init (1 - cooling)^k) iterated, logged bit-equal to the oracle."""
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 8
    sc = calibrate(prof, T, n, 400.0, 0.5)
    ap = AnnealParams(proposal="uniform", evaluate="proposal", max_steps=60, stall_limit=60, cooling="multiplicative",
                      time_budget_s=float("inf"))
    starts = base_graph(7, n)[None, :]
    host = engine.anneal(starts, prof, [sc], ap, 3, n=n, log=True).host()
    temps = host["log"][0]["temp"][: int(host["results"][0]["steps"])]
    t, want = ap.t_init, []
    for _ in range(len(temps)):
        want.append(max(ap.t_floor, t))
        t = t * (1.0 - ap.cooling_step)
    assert np.array_equal(np.asarray(temps, dtype=np.float64).view(np.uint64), np.array(want).view(np.uint64))
    assert temps[-1] == ap.t_floor
