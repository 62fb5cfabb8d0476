"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The table-surrogate evaluator.

Restates DESIGN.md "Scoring surrogate" (the replacement for SPEC:334-372's DES,
SURVEY 7.2 D1) and Eqs. 1, 2, 3, 6 in numpy.  The p95 term is the
nearest-rank p95 over requests of the fleet's service-time mixture:
request shares follow the instance-pull dispatch of SPEC:335 at utilisation
rho < 1 (every instance waits W0 = (1000 m / R)(1 - rho) ms in the idle queue
between services, so instance j serves 1000 / (s_j + W0) requests/s; W0 -> 0
gives SPEC:390's throughput shares under saturation), walked from the slowest
edge down until the tail holds more than 5 % of the arrival rate R.  Eq. 1 / Eq. 2 use
the algebraically identical forms (A - A_base) * (100 / A_base) and
100 - E * (ci / (10 C_base)); tests pin them to the SPEC-literal quotients.
Aggregates are recomputed from scratch per candidate (W @ rows, int64), so this
is independent of the device's incremental neighbour scoring.  Every fp64
operation is one IEEE-rounded numpy ufunc in the documented order; the kernels
compile with -fmad=false and reproduce the same bits.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .tables import OracleTables


@dataclass
class Evaluated:
    A: np.ndarray
    E: np.ndarray
    L: np.ndarray
    f: np.ndarray
    h: np.ndarray
    sla: np.ndarray


def constants(tables: OracleTables, scenario):
    R = float(scenario.arrival_rps)
    return dict(R_q=math.ldexp(R, tables.kt), inv_3600R=1.0 / (3600.0 * R),
                en_scale=math.ldexp(1.0, tables.kt - tables.ke),
                idle_scale=math.ldexp(1.0, -tables.ki),
                kW=1000.0 / R, c20=20000.0 / R)


def rank_order(tables: OracleTables) -> list:
    """Edges by ascending p95 service latency, ties by edge index (the device's rank)."""
    return sorted(range(tables.E), key=lambda e: (float(tables.lat95[e]), e))


def p95_walk(W: np.ndarray, tables: OracleTables, W0: np.ndarray, c20: float) -> np.ndarray:
    """Service p95 of each fleet (rows of W) given its idle-queue time W0 (ms).

    Present edges are visited from the highest latency rank down; the tail's request
    rate sum_j 1000 w_j / (s_j + W0) is kept as the fraction P / Q (no division):
    d = s + W0, P <- P d + w Q, Q <- Q d; the walk stops at the first edge where
    P * (20000 / R) > Q (the tail now holds > 5 % of R), else at the lowest present
    edge.  The p95 is that edge's lat95."""
    W = np.asarray(W, dtype=np.int64).reshape(-1, tables.E)
    n = len(W)
    P = np.zeros(n)
    Q = np.ones(n)
    done = np.zeros(n, dtype=bool)
    lq = np.zeros(n)
    with np.errstate(over="ignore", invalid="ignore"):
        for e in reversed(rank_order(tables)):
            act = ~done & (W[:, e] > 0)
            if not act.any():
                continue
            d = float(tables.mean_ms[e]) + W0
            Pn = P * d + W[:, e].astype(np.float64) * Q
            Qn = Q * d
            P = np.where(act, Pn, P)
            Q = np.where(act, Qn, Q)
            lq = np.where(act, float(tables.lat95[e]), lq)
            done = done | (act & (P * c20 > Q))
    return lq


def aggregates(W: np.ndarray, tables: OracleTables):
    W = np.asarray(W, dtype=np.int64).reshape(-1, tables.E)
    s_thr = W @ tables.thr_q
    s_acc = W @ tables.acc_q
    s_en = W @ tables.en_q
    cnt = W.reshape(len(W), tables.V, 5).sum(axis=1)
    s_idle = cnt @ tables.idle_q
    m = W.sum(axis=1)
    return s_thr, s_acc, s_en, s_idle, W, m


def epilogue(s_thr, s_acc, s_en, s_idle, W, m, tables, scenario) -> Evaluated:
    c = constants(tables, scenario)
    obj = scenario.obj
    a_base, c_base, slo = obj.base_accuracy, obj.base_carbon_g, obj.latency_slo_ms
    lam, ci = obj.carbon_weight, float(scenario.ci)
    kA = 100.0 / a_base                       # Eq. 1 as (A - A_base) * kA
    kC = ci / (10.0 * c_base)                 # Eq. 2 as 100 - E * kC
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / s_thr.astype(np.float64)
        A = s_acc.astype(np.float64) * inv
        rho = c["R_q"] * inv
        e_act = (s_en.astype(np.float64) * inv) * c["en_scale"]
        rho_c = np.minimum(rho, 1.0)
        p_idle = s_idle.astype(np.float64) * c["idle_scale"]
        E = e_act + ((1.0 - rho_c) * p_idle) * c["inv_3600R"]
        md = np.asarray(m, dtype=np.float64)
        W0 = (md * c["kW"]) * (1.0 - rho_c)           # idle-queue time between services (ms)
        lq = p95_walk(W, tables, W0, c["c20"])
        rho_q = np.minimum(rho, scenario.rho_sat)
        # queueing factor of m servers: L = lq * (1 + rho^8 / (m (1 - rho)))
        q1 = 1.0 - rho_q
        r2 = rho_q * rho_q
        r4 = r2 * r2
        r8 = r4 * r4
        wq = r8 / (md * q1)
        L = lq * (1.0 + wq)
        dA = (A - a_base) * kA
        dC = 100.0 - E * kC
        f = lam * dC + (1.0 - lam) * dA
        lat_ok = L <= slo
        # accuracy_threshold_mode: SLA class also needs dA >= -max_loss; h unchanged
        sla = lat_ok & (dA >= -float(getattr(scenario, "max_accuracy_loss_pct", math.inf)))
        soft = np.where((f >= 0) | bool(scenario.strict_eq6), -f * (slo / L), -f * (L / slo))
        h = np.where(lat_ok, -f, soft)
    return Evaluated(A, E, L, f, h, sla)


def evaluate(W, tables: OracleTables, scenario) -> Evaluated:
    return epilogue(*aggregates(W, tables), tables, scenario)


def evaluate_one(w, tables, scenario) -> dict:
    ev = evaluate(np.asarray(w)[None, :], tables, scenario)
    return {k: (bool(getattr(ev, k)[0]) if k == "sla" else float(getattr(ev, k)[0]))
            for k in ("A", "E", "L", "f", "h", "sla")}


def base_graph(V: int, n: int) -> np.ndarray:
    """BASE: largest variant on every unpartitioned GPU."""
    w = np.zeros(V * 5, dtype=np.int64)
    w[(V - 1) * 5 + 0] = n
    return w


def calibrate(profile, tables: OracleTables, n: int, ci: float, lam: float = 0.5,
              utilization: float = 0.7, ci_base=None, strict: bool = False, pue: float = 1.5):
    """R = utilization x BASE capacity; A_base, C_base, L_tail from BASE
    (C_base without PUE per SURVEY D7)."""
    from paper_2304_09781_b200.core import ObjectiveParams, SliceType
    from paper_2304_09781_b200.objective import Scenario
    V = profile.variant_count
    R = utilization * n * (1000.0 / profile.mean_service_ms(V, SliceType.S7G))
    probe = Scenario(n, R, float(ci), ObjectiveParams(1.0, 1.0, 1.0, lam, pue), strict)
    ev = evaluate_one(base_graph(V, n), tables, probe)
    cb = float(ci if ci_base is None else ci_base)
    obj = ObjectiveParams(ev["A"], ev["E"] / 1000.0 * cb, ev["L"], lam, pue)
    return Scenario(n, R, float(ci), obj, strict)
