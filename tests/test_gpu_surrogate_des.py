"""The surrogate's p95 / SLA against the SPEC's serving simulator
(the device DES that tests/test_gpu_des.py pins bit for bit to oracle/des.py).

Population: what the search visits on the c2 shape (n = 64, EfficientNet, 0.7 x BASE) --
centres of 64 chains from perturbed starts after 2..64 steps plus their winners.  Both SLA
classes must be populated.  Bars (deterministic service): SLA agreement >= 95 %, at least
20 % SLA-meeting fleets, Spearman rank correlation of p95 >= 0.8."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 64


def test_surrogate_sla_agrees_with_des(engine):
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from validate_surrogate import spearman, trajectory_fleets
    from paper_2304_09781_b200 import sim as S
    from paper_2304_09781_b200.graph import build_graph
    from paper_2304_09781_b200.profiles import synthetic_profile
    from paper_2304_09781_b200.search import base_config
    engine.ensure_feasibility(N)
    prof = synthetic_profile("efficientnet")
    sc = engine.calibrate(prof, N, 350.0, 0.5)
    base = base_config(N, prof)
    w = S.Workload(sc.arrival_rps, 600.0, 230409781)
    l_tail_des = S.simulate(base, prof, w, engine=engine).p95_ms
    fleets = trajectory_fleets(engine, prof, sc, base, N, chains=64)
    W = np.array([build_graph(f, prof).weights for f in fleets], dtype=np.uint16)
    _best, outs = engine.score_graphs(W, prof, sc)
    L = outs["p95"].cpu().numpy()
    sla_s = L <= sc.obj.latency_slo_ms
    dP = np.array([r.p95_ms for r in S.simulate_fleets(fleets, prof, w, l_tail_des, engine=engine)])
    sla_d = dP <= l_tail_des
    agree = float(np.mean(sla_s == sla_d))
    assert sla_d.mean() >= 0.2 and (~sla_d).mean() >= 0.2, sla_d.mean()
    assert agree >= 0.95, agree
    assert spearman(L, dP) >= 0.8
