"""ORACLE / anneal properties on the CPU oracle (acceptance 3, 8)."""

import numpy as np
import pytest

from oracle.anneal import anneal_chain
from oracle.evaluator import base_graph, calibrate, evaluate
from oracle.feasibility import FeasOracle
from oracle.search import oracle_search, oracle_space, select_oracle
from oracle.tables import OracleTables
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
from paper_2304_09781_b200.objective import AnnealParams, delta_accuracy, delta_carbon
from paper_2304_09781_b200.profiles import synthetic_profile


def test_oracle_space_sizes():
    T1 = OracleTables.from_profile(synthetic_profile("efficientnet", variants=1))
    assert oracle_space(DEFAULT_TOPOLOGY, T1)[1] == 19
    T2 = OracleTables.from_profile(synthetic_profile("efficientnet", variants=2))
    space, _ = oracle_space(DEFAULT_TOPOLOGY, T2)
    assert [c for cid, _k, _r, c, _o in space if cid == 19] == [128]
    T7 = OracleTables.from_profile(synthetic_profile("efficientnet"))
    assert oracle_space(DEFAULT_TOPOLOGY, T7)[1] == 983_899


def test_lambda_sweep_monotone():
    prof = synthetic_profile("tiny3")
    T = OracleTables.from_profile(prof)
    dcs, das = [], []
    for lam in (0.1, 0.3, 0.5, 0.7, 0.9):
        sc = calibrate(prof, T, 2, 400.0, lam)
        i, ev, _W = oracle_search(DEFAULT_TOPOLOGY, T, sc, 2)
        dcs.append(delta_carbon(float(ev.E[i]), sc.ci, sc.obj))
        das.append(delta_accuracy(float(ev.A[i]), sc.obj))
    assert all(x <= y + 1e-9 for x, y in zip(dcs, dcs[1:]))
    assert all(x >= y - 1e-9 for x, y in zip(das, das[1:]))


def test_anneal_best_h_non_increasing_and_stall_from_optimum():
    prof = synthetic_profile("efficientnet", variants=1)
    T = OracleTables.from_profile(prof)
    feas = FeasOracle(DEFAULT_TOPOLOGY, 1)
    sc = calibrate(prof, T, 1, 400.0, 0.5)
    # global optimum over every realizable n=1 graph (one variant: the 19 rows)
    W = np.array([[c * 1 for c in row] for row in DEFAULT_TOPOLOGY.config_vectors], dtype=np.int64)
    ev = evaluate(W, T, sc)
    best = np.lexsort((np.arange(len(W)), ev.h, ~ev.sla))[0]
    ap = AnnealParams(proposal="uniform", evaluate="proposal", max_steps=100, time_budget_s=1e9)
    out = anneal_chain(W[best], 1, T, sc, ap, 7, 0, feas, log=True)
    assert out.evals <= 6
    out = anneal_chain(base_graph(1, 1), 1, T, sc, ap, 3, 0, feas, log=True)
    bests = [r["h"] for r in out.log if r["new_best"]]
    assert all(x >= y for x, y in zip(bests, bests[1:]))


def test_anneal_near_oracle_small_instance():
    """Acceptance 3 analogue: full-neighbourhood anneal from BASE reaches within 5% of ORACLE's f."""
    prof = synthetic_profile("tiny3")
    T = OracleTables.from_profile(prof)
    feas = FeasOracle(DEFAULT_TOPOLOGY, 2)
    sc = calibrate(prof, T, 2, 400.0, 0.5)
    i, ev, _W = oracle_search(DEFAULT_TOPOLOGY, T, sc, 2)
    f_star = float(ev.f[i])
    hits = 0
    for seed in range(10):
        out = anneal_chain(base_graph(3, 2), 2, T, sc, AnnealParams(proposal="uniform", max_steps=40), seed, 0, feas)
        hits += out.best["sla"] and out.best["f"] >= f_star - 0.05 * abs(f_star)
    assert hits >= 9
