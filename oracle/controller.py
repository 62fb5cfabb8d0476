"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The trace-driven control loop.

Restates run_trace for the 'clover' scheme on top of the oracle's anneal chains
and evaluator: re-plan when |dci|/ci > threshold (prev = 0 always), chains
start from the incumbent and are seeded by derive_seed(seed, tick), the winner
(SLA desc, h asc, chain asc) replaces the incumbent only if it is better and
meets the SLA, carbon accrues R * step * E/1000 * ci * PUE per tick.
"""

from __future__ import annotations

import numpy as np

from .anneal import anneal_chain
from .evaluator import base_graph, calibrate, evaluate_one
from .rng import derive_seed


def _chain_job(args):
    return anneal_chain(*args)


def _serial_map(fn, jobs):
    return [fn(j) for j in jobs]


def intensity_at(samples, t):
    val = samples[0][1]
    for ts, c in samples:
        if ts <= t:
            val = c
        else:
            break
    return val


def run_trace_clover(samples, n, profile, tables, lam, ap, seed, chains, feas, step_s=300.0, threshold=0.05,
                     utilization=0.7, pue=1.5, map_fn=None, chain_base=0, ticks=None):
    """map_fn(fn, args) runs a re-plan's independent chains, e.g. a process pool's map;
    ticks stops after that many ticks (a prefix of the same run)."""
    ci_mean = sum(c for _, c in samples) / len(samples)
    base_sc = calibrate(profile, tables, n, ci_mean, lam, utilization, ci_base=ci_mean, pue=pue)
    V = tables.V
    bw = base_graph(V, n)
    w = bw.copy()
    prev = 0.0
    cum = 0.0
    out = []
    steps = int(round((samples[-1][0] - samples[0][0]) / step_s)) + 1
    if ticks is not None:
        steps = min(steps, int(ticks))
    for tick in range(steps):
        t = samples[0][0] + tick * step_s
        ci = intensity_at(samples, t)
        sc = base_sc.with_ci(ci)
        replanned = accepted = False
        if prev <= 0 or abs(ci - prev) / prev > threshold:
            replanned = True
            s = derive_seed(seed, tick)
            jobs = [(w, n, tables, sc, ap, s, chain_base + c, feas) for c in range(chains)]
            res = (map_fn or _serial_map)(_chain_job, jobs)
            keys = [(0 if r.best["sla"] else 1, r.best["h"], c) for c, r in enumerate(res) if r.status >= 0]
            _, _, c = min(keys)
            cand = res[c]
            cur = evaluate_one(w, tables, sc)
            better = (cand.best["sla"] and not cur["sla"]) or (cand.best["sla"] == cur["sla"] and cand.best["h"] < cur["h"])
            if better and cand.best["sla"]:
                w = cand.best_w.copy()
                accepted = True
            prev = ci
        act = evaluate_one(w, tables, sc)
        cum += sc.arrival_rps * step_s * (act["E"] / 1000.0 * ci * pue)
        out.append(dict(tick=tick, ci=ci, replanned=replanned, accepted=accepted, w=w.copy(), cum=cum,
                        sla=act["sla"], accuracy=act["A"]))
    return out
