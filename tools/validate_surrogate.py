"""Validate the table surrogate's p95 / SLA against the SPEC's own evaluator,
the serving DES, on fleets that straddle L_tail.

Per family (efficientnet = deterministic service, the headline catalog; resnet =
exponential; bert = lognormal) at n GPUs, 10 simulated minutes at 0.7 x BASE capacity:
  * perturbed : re-plan starts around BASE (search.perturbed_fleets, keep in 0.5..0.95),
  * random    : BLOVER draws (search.random_fleets),
  * trajectory: what the search visits -- the centres of 128 chains from perturbed starts
                after 2, 4, 8, 16, 32 and 64 steps, plus their winners (efficientnet only).
Reports accuracy / energy agreement, Spearman rank correlation (tie-aware) of surrogate
L vs simulated p95, and the SLA confusion matrix (surrogate L <= L_tail(BASE) vs
simulated p95 <= simulated p95 of BASE).  Run on a GPU box:
    python tools/validate_surrogate.py [--n 64] [--out profiles/r02_surrogate_vs_des.json]
"""

import argparse
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
from paper_2304_09781_b200.search import (anneal_chains, base_config, perturbed_fleets,  # noqa: E402
                                          random_fleets)


def spearman(a, b):
    """Spearman's rho with average ranks for ties."""
    def ranks(x):
        x = np.asarray(x, dtype=np.float64)
        order = np.argsort(x, kind="stable")
        r = np.empty(len(x))
        xs = x[order]
        i = 0
        while i < len(x):
            j = i
            while j + 1 < len(x) and xs[j + 1] == xs[i]:
                j += 1
            r[order[i:j + 1]] = 0.5 * (i + j)
            i = j + 1
        return r
    ra, rb = ranks(a), ranks(b)
    if ra.std() == 0 or rb.std() == 0:
        return float("nan")
    return float(np.corrcoef(ra, rb)[0, 1])


DUMP = {}


def compare(name, fleets, eng, prof, sc, w, l_tail_des):
    W = np.array([build_graph(f, prof).weights for f in fleets], dtype=np.uint16)
    _best, outs = eng.score_graphs(W, prof, sc)
    L = outs["p95"].cpu().numpy()
    sla_s = L <= sc.obj.latency_slo_ms
    reps = S.simulate_fleets(fleets, prof, w, l_tail_des, engine=eng)
    dP = np.array([r.p95_ms for r in reps])
    sla_d = dP <= l_tail_des
    key = "%s_%s" % (prof.name, name.split()[0])
    DUMP[key + "_W"], DUMP[key + "_L"], DUMP[key + "_dP"] = W, L, dP
    DUMP[key + "_mean"] = np.array([r.mean_latency_ms for r in reps])
    DUMP[key + "_lt"] = np.array([sc.obj.latency_slo_ms, l_tail_des, sc.arrival_rps])
    return {
        "population": name, "fleets": len(fleets),
        "p95_spearman": spearman(L, dP),
        "p95_median_abs_rel_err": float(np.median(np.abs(L - dP) / dP)),
        "sla_agreement": float(np.mean(sla_s == sla_d)),
        "des_sla_meet_fraction": float(np.mean(sla_d)),
        "sla_confusion": {"both_meet": int(np.sum(sla_s & sla_d)), "surrogate_only": int(np.sum(sla_s & ~sla_d)),
                          "des_only": int(np.sum(~sla_s & sla_d)), "neither": int(np.sum(~sla_s & ~sla_d))},
    }


def run_family(eng, fam, n, count, seed=230409781):
    prof = synthetic_profile(fam)
    sc = eng.calibrate(prof, n, 350.0, 0.5)
    w = S.Workload(sc.arrival_rps, 600.0, seed)
    base = base_config(n, prof)
    l_tail_des = S.simulate(base, prof, w, engine=eng).p95_ms
    out = {"family": fam, "n_gpus": n, "rate_rps": sc.arrival_rps, "des_window_s": 600.0,
           "l_tail_surrogate_ms": sc.obj.latency_slo_ms, "l_tail_des_ms": l_tail_des}
    pert = []
    for k, keep in enumerate((0.5, 0.65, 0.8, 0.9, 0.95)):
        pert += perturbed_fleets(base, prof, 17 + k, count // 5, keep=keep)
    out["perturbed"] = compare("perturbations of BASE (keep 0.5..0.95)", pert, eng, prof, sc, w, l_tail_des)
    out["random"] = compare("BLOVER random realizable fleets", random_fleets(eng, prof, n, 7, count, 0),
                            eng, prof, sc, w, l_tail_des)
    if fam == "efficientnet":
        out["trajectory"] = compare("chain centres after 2..64 steps and the winners, 128 chains from perturbed "
                                    "starts", trajectory_fleets(eng, prof, sc, base, n), eng, prof, sc, w, l_tail_des)
    return out


def trajectory_fleets(eng, prof, sc, base, n, chains=128):
    """Graphs the search visits: chain centres after k steps (k = 2..64) and the winners."""
    starts = np.array([build_graph(f, prof).weights for f in perturbed_fleets(base, prof, 11, chains)],
                      dtype=np.uint16)
    graphs = []
    for k in (2, 4, 8, 16, 32, 64):
        res = anneal_chains(eng, starts, prof, sc, AnnealParams(max_steps=k), 5, exchange=False)
        graphs += list(res.final_w)
    res = anneal_chains(eng, starts, prof, sc, AnnealParams(max_steps=256), 5, exchange=False)
    graphs += list(res.best_w)
    return [eng.realize(ConfigGraph(g.astype(np.int64), prof.variant_count, prof.name), n) for g in graphs]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--count", type=int, default=500)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    eng = CloverEngine(n_max=args.n)
    res = {"model": "DESIGN.md §3: p95 = nearest-rank over instance-pull request shares x many-server factor",
           "families": [run_family(eng, fam, args.n, args.count) for fam in ("efficientnet", "resnet", "bert")]}
    text = json.dumps(res, indent=1)
    print(text)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text + "\n")
        np.savez_compressed(os.path.splitext(args.out)[0] + "_dump.npz", **DUMP)


if __name__ == "__main__":
    main()
