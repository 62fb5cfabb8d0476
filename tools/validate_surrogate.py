"""Validate the table surrogate against the SPEC's own evaluator, the
serving DES, on the c2 fleet shape: random realizable n=64 fleets and
the re-plan winners of 128 annealing chains, 10 simulated minutes at 0.7 x BASE.

Reports, per population: accuracy and energy-per-request agreement, rank correlation of
the p95 estimates, and the SLA confusion matrix (surrogate L <= L_tail(BASE) vs simulated
p95 <= simulated p95 of BASE).  Run on the GPU box:  python tools/validate_surrogate.py
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_09781_b200 import sim as S  # noqa: E402
from paper_2304_09781_b200.engine import CloverEngine  # noqa: E402
from paper_2304_09781_b200.graph import ConfigGraph, build_graph  # noqa: E402
from paper_2304_09781_b200.objective import AnnealParams  # noqa: E402
from paper_2304_09781_b200.profiles import synthetic_profile  # noqa: E402
from paper_2304_09781_b200.search import anneal_chains, base_config, random_fleets  # noqa: E402


def surrogate_AE(W, tables, sc):
    """Surrogate A and E of each graph, evaluated on the host for this report."""
    W = W.astype(np.float64)
    thr = W @ np.asarray(tables.thr_q, dtype=np.float64)
    acc = W @ np.asarray(tables.acc_q, dtype=np.float64)
    en = W @ np.asarray(tables.en_q, dtype=np.float64)
    cnt = np.stack([W[:, s::5].sum(axis=1) for s in range(5)], axis=1)
    idle = cnt @ np.asarray(tables.idle_q, dtype=np.float64)
    R = sc.arrival_rps
    A = acc / thr
    rho = np.minimum(np.ldexp(R, tables.kt) / thr, 1.0)
    E = (en / thr) * 2.0 ** (tables.kt - tables.ke) + ((1.0 - rho) * idle * 2.0 ** (-tables.ki)) / (3600.0 * R)
    return A, E


def many_server_L(W, tables, sc, mode):
    """Candidate p95 models on the host: Lmax * (1 + rho^k / (m (1 - rho))) with k = 8 or sqrt(2(m+1))."""
    W = W.astype(np.float64)
    thr = W @ np.asarray(tables.thr_q, dtype=np.float64)
    lat = np.asarray(tables.lat95, dtype=np.float64)
    lmax = np.where(W > 0, lat[None, :], 0.0).max(axis=1)
    rho = np.minimum(np.ldexp(sc.arrival_rps, tables.kt) / thr, sc.rho_sat)
    m = W.sum(axis=1)
    k = 8.0 if mode == "k8" else np.sqrt(2.0 * (m + 1.0))
    return lmax * (1.0 + rho ** k / (m * (1.0 - rho)))


def spearman(a, b):
    ra = np.argsort(np.argsort(a)).astype(np.float64)
    rb = np.argsort(np.argsort(b)).astype(np.float64)
    return float(np.corrcoef(ra, rb)[0, 1])


def compare(name, fleets, eng, prof, sc, w, l_tail_des):
    W = np.array([build_graph(f, prof).weights for f in fleets], dtype=np.uint16)
    _best, outs = eng.score_graphs(W, prof, sc)
    L = outs["p95"].cpu().numpy()
    sla_s = outs["sla"].cpu().numpy().astype(bool)
    A, E = surrogate_AE(W, prof.scoring_tables(), sc)
    reps = S.simulate_fleets(fleets, prof, w, l_tail_des, engine=eng)
    dA = np.array([r.accuracy for r in reps])
    dE = np.array([r.energy_wh_total / r.completed for r in reps])
    dP = np.array([r.p95_ms for r in reps])
    sla_d = dP <= l_tail_des
    base_W = np.array([build_graph(base_config(64, prof), prof).weights], dtype=np.uint16)
    alt = {}
    for mode in ("k8", "sakasegawa"):
        Lm = many_server_L(W, prof.scoring_tables(), sc, mode)
        lt = many_server_L(base_W, prof.scoring_tables(), sc, mode)[0]
        s_m = Lm <= lt
        alt[mode] = {"p95_spearman": spearman(Lm, dP), "l_tail_ms": float(lt), "p95_median_ms": float(np.median(Lm)),
                     "sla_agreement": float(np.mean(s_m == sla_d)), "sla_meet": int(s_m.sum()),
                     "median_rel_err": float(np.median(np.abs(Lm - dP) / dP))}
    return {
        "many_server_models": alt,
        "population": name, "fleets": len(fleets),
        "accuracy_mean_abs_diff": float(np.mean(np.abs(A - dA))),
        "accuracy_max_abs_diff": float(np.max(np.abs(A - dA))),
        "energy_per_request_mean_rel_diff": float(np.mean(np.abs(E - dE) / dE)),
        "p95_spearman": spearman(L, dP),
        "p95_surrogate_ms_median": float(np.median(L)), "p95_des_ms_median": float(np.median(dP)),
        "sla_confusion": {"both_meet": int(np.sum(sla_s & sla_d)), "surrogate_only": int(np.sum(sla_s & ~sla_d)),
                          "des_only": int(np.sum(~sla_s & sla_d)), "neither": int(np.sum(~sla_s & ~sla_d))},
        "sla_agreement": float(np.mean(sla_s == sla_d)),
    }


def main():
    n = 64
    eng = CloverEngine(n_max=n)
    prof = synthetic_profile("efficientnet")
    sc = eng.calibrate(prof, n, 350.0, 0.5)
    w = S.Workload(sc.arrival_rps, 600.0, 230409781)
    l_tail_des = S.simulate(base_config(n, prof), prof, w, engine=eng).p95_ms
    out = {"n_gpus": n, "rate_rps": sc.arrival_rps, "des_window_s": 600.0,
           "l_tail_surrogate_ms": sc.obj.latency_slo_ms, "l_tail_des_ms": l_tail_des}
    rnd = random_fleets(eng, prof, n, 7, 512, 0)
    out["random"] = compare("random realizable fleets", rnd, eng, prof, sc, w, l_tail_des)
    starts = np.array([build_graph(f, prof).weights for f in random_fleets(eng, prof, n, 11, 128, 0)],
                      dtype=np.uint16)
    res = anneal_chains(eng, starts, prof, sc, AnnealParams(max_steps=64), 5, exchange=False)
    winners = [eng.realize(ConfigGraph(g.astype(np.int64), prof.variant_count, prof.name), n) for g in res.best_w]
    out["winners"] = compare("re-plan winners of 128 chains (best-h proposal)", winners, eng, prof, sc, w,
                             l_tail_des)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
