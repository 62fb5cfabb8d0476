"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The annealing chain.

One chain, sequential by definition.  Step semantics follow
DESIGN.md "Chain step": temperature T_k = max(t_floor,
t_init - k*cooling) (or t_init (1 - cooling)^k, SPEC:492's multiplicative
option); move set SPEC (default) or paper (+ unit add/remove); best tracking SLA-first then lowest h,
ties keep the incumbent; stall after ``stall_limit``
steps without a new best; Eq. 7 acceptance with
u = uniform01(derive_seed(seed, chain, k, 0)).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .evaluator import evaluate, evaluate_one
from .neighbours import enumerate_neighbours
from .rng import derive_seed, exp_clv, uniform01

MAX_STEPS, STALLED, NO_NEIGHBOR = 0, 1, 2


@dataclass
class ChainOut:
    best_w: np.ndarray
    best: dict
    best_step: int
    best_idx: int
    final_w: np.ndarray
    status: int
    steps: int
    evals: int
    log: list = field(default_factory=list)


def _better(sla_a, h_a, sla_b, h_b) -> bool:
    return (sla_a and not sla_b) or (sla_a == sla_b and h_a < h_b)


def anneal_chain(w0, n, tables, scenario, ap, seed, chain, feas, log=False) -> ChainOut:
    V = tables.V
    w = np.asarray(w0, dtype=np.int64).copy()
    cur = evaluate_one(w, tables, scenario)
    best, best_w, best_step, best_idx = dict(cur), w.copy(), -1, -1
    evals, stall, status, steps = 1, 0, MAX_STEPS, 0
    rows = []
    moves = getattr(ap, "move_set", "spec")
    mult = getattr(ap, "cooling", "subtractive") == "multiplicative"
    t_raw, factor = ap.t_init, 1.0 - ap.cooling_step
    for k in range(ap.step_limit()):
        if mult:                                 # T_k = max(t_floor, t_init (1 - cooling)^k), iterated
            T = max(ap.t_floor, t_raw)
            t_raw = t_raw * factor
        else:
            T = max(ap.t_floor, ap.t_init - k * ap.cooling_step)
        nb = enumerate_neighbours(w, tables.mem_ok, V, n, feas, moves)
        if len(nb) == 0:
            status = NO_NEIGHBOR
            break
        if ap.evaluate == "all":
            ev = evaluate(nb.W, tables, scenario)
            evals += len(nb)
            c = int(np.lexsort((nb.idx, ev.h, ~ev.sla))[0])
            cand = {k2: (bool(getattr(ev, k2)[c]) if k2 == "sla" else float(getattr(ev, k2)[c]))
                    for k2 in ("A", "E", "L", "f", "h", "sla")}
            if ap.proposal == "best":
                p = int(np.lexsort((nb.idx, ev.h))[0])
        if ap.proposal == "uniform":
            keys = [(derive_seed(seed, chain, k, int(i) + 1), int(i)) for i in nb.idx]
            p = min(range(len(keys)), key=keys.__getitem__)
        if ap.evaluate == "all":
            prop = {k2: (bool(getattr(ev, k2)[p]) if k2 == "sla" else float(getattr(ev, k2)[p]))
                    for k2 in ("A", "E", "L", "f", "h", "sla")}
        else:
            prop = evaluate_one(nb.W[p], tables, scenario)
            evals += 1
            c, cand = p, prop
        new_best = _better(cand["sla"], cand["h"], best["sla"], best["h"])
        if new_best:
            best, best_w, best_step, best_idx = dict(cand), nb.W[c].copy(), k, int(nb.idx[c])
            stall = 0
        else:
            stall += 1
        u = uniform01(derive_seed(seed, chain, k, 0))
        hp, hc = prop["h"], cur["h"]
        accept = hp <= hc or u < exp_clv(-(hp - hc) / T)
        if log:
            rows.append(dict(iter=k, temp=T, ged_from_center=int(nb.ged[p]), n_neighbours=len(nb), f=prop["f"],
                             h=prop["h"], p95_ms=prop["L"], sla_met=prop["sla"],
                             accepted=bool(accept), new_best=bool(new_best)))
        if accept:
            w = nb.W[p].copy()
            cur = prop
        steps = k + 1
        if stall >= ap.stall_limit:
            status = STALLED
            break
    return ChainOut(best_w, best, best_step, best_idx, w, status, steps, evals, rows)
