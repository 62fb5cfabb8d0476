"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The table-surrogate evaluator.

Restates DESIGN.md "Scoring surrogate" (the replacement for SPEC:334-372's DES,
SURVEY 7.2 D1) and Eqs. 1, 2, 3, 6 in numpy.  The p95 term is the
nearest-rank p95 over requests of the fleet's service-time mixture:
request shares follow the instance-pull dispatch of SPEC:335 at utilisation
rho < 1 (every instance waits W ms in the idle queue between services, so instance j
serves 1 / (s_j + W) requests/s, W the root of "the instances' rates sum to R" over a
2-point Gauss quadrature of the fleet's service rates; W = 0 gives SPEC:390's
throughput shares under saturation), walked from the slowest edge down until the
tail carries more than 5 % of R.  Eq. 1 / Eq. 2 use
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
                R=R, c20=20000.0 / R)


def rank_order(tables: OracleTables) -> list:
    """Edges by ascending p95 service latency, ties by edge index (the device's rank)."""
    return sorted(range(tables.E), key=lambda e: (float(tables.lat95[e]), e))


def idle_wait_ms(m, s1, s2, s3, R, R_q, inv, rho_c, tables):
    """Idle-queue wait W (ms) of every fleet: the root of sum_j w_j x_j / (1 + W x_j) = R
    (instance j serves 1 / (s_j + W) requests per second, x_j = 1 / s_j, the rates summing
    to the arrival rate R) with the rate distribution replaced by its 2-point Gauss
    quadrature (matching sum w x, sum w x^2, sum w x^3).  By Vieta the nodes drop out:
    with a_k = sum w x^k, D = a2 m - a1^2, N0 = a1 a3 - a2^2, N1 = a1 a2 - a3 m the root
    solves R N0 W^2 - (R N1 + m N0) W + (R - a1) D = 0 (the cancellation-free branch of the
    quadratic formula).  Homogeneous fleets (D <= 1e-9 a2 m) and degenerate roots take
    the homogeneous solution W = (m / R)(1 - rho); saturated fleets (rho >= 1) W = 0.  W is clamped
    to m / R (a bound of the exact root, so the kernels' screen may use 1000 m / R as W0's bound)."""
    t2, k2, t3, k3 = tables.rate_moment_rows()
    a1 = s1 * math.ldexp(1.0, -tables.kt)
    a2 = s2 * math.ldexp(1.0, -k2)
    a3 = s3 * math.ldexp(1.0, -k3)
    D = a2 * m - a1 * a1
    N0 = a1 * a3 - a2 * a2
    N1 = a1 * a2 - a3 * m
    A = R * N0
    B = -(R * N1) - m * N0
    C = (R - a1) * D
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        x = B * B - (4.0 * A) * C
        sq = np.sqrt(np.where(x > 0.0, x, 0.0))
        num = np.where(B >= 0.0, -2.0 * C, sq - B)
        den = np.where(B >= 0.0, B + sq, 2.0 * A)
        root = num / np.where(den > 0.0, den, 1.0)
        homo = (m * (1.0 / R)) * (1.0 - rho_c)
        ok = (den > 0.0) & (root >= 0.0) & (root < np.inf) & ~(D <= (1e-9 * a2) * m)
        W = np.where(ok, root, homo)
        W = np.where(rho_c >= 1.0, 0.0, W)
        mR = m * (1.0 / R)                    # W < m / R for the exact root; clamp the rounded one
        W = np.where(W < mR, W, mR)
    return 1000.0 * W


def p95_walk(W: np.ndarray, tables: OracleTables, W0: np.ndarray, c20: float) -> np.ndarray:
    """Service p95 of each fleet (rows of W) given its idle-queue wait W0 (ms).

    Present edges are visited from the highest latency rank down; the tail's request rate,
    scaled by c20 = 20000 / R, (20000 / R) sum_j w_j / (s_j + W0), is kept as the fraction
    P / Q (no division): d = s + W0, P <- P d + (w c20) Q, Q <- Q d; the walk stops at the
    first edge where P > Q (the tail now carries more than 5 % of the arrival rate R),
    else at the lowest present edge.  The p95 is that edge's lat95."""
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
            Pn = P * d + (W[:, e].astype(np.float64) * c20) * Q
            Qn = Q * d
            P = np.where(act, Pn, P)
            Q = np.where(act, Qn, Q)
            lq = np.where(act, float(tables.lat95[e]), lq)
            done = done | (act & (P > Q))
    return lq


def walk_lengths(W: np.ndarray, tables: OracleTables, scenario) -> np.ndarray:
    """Ranks visited by each fleet's p95 walk (the K of the per-candidate work model in
    DESIGN.md; measurement only, not part of the evaluator)."""
    s_thr, s_acc, s_en, s_idle, (Wm, s2, s3), m = aggregates(W, tables)
    c = constants(tables, scenario)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / s_thr.astype(np.float64)
        rho_c = np.minimum(c["R_q"] * inv, 1.0)
        W0 = idle_wait_ms(np.asarray(m, dtype=np.float64), s_thr.astype(np.float64), np.asarray(s2, dtype=np.float64),
                          np.asarray(s3, dtype=np.float64), c["R"], c["R_q"], inv, rho_c, tables)
    n = len(Wm)
    P, Q = np.zeros(n), np.ones(n)
    done = np.zeros(n, dtype=bool)
    K = np.zeros(n, dtype=np.int64)
    with np.errstate(over="ignore", invalid="ignore"):
        for e in reversed(rank_order(tables)):
            act = ~done & (Wm[:, e] > 0)
            d = float(tables.mean_ms[e]) + W0
            Pn = P * d + (Wm[:, e].astype(np.float64) * c["c20"]) * Q
            P = np.where(act, Pn, P)
            Q = np.where(act, Q * d, Q)
            K += act
            done = done | (act & (P > Q))
    return K


def aggregates(W: np.ndarray, tables: OracleTables):
    W = np.asarray(W, dtype=np.int64).reshape(-1, tables.E)
    s_thr = W @ tables.thr_q
    s_acc = W @ tables.acc_q
    s_en = W @ tables.en_q
    cnt = W.reshape(len(W), tables.V, 5).sum(axis=1)
    s_idle = cnt @ tables.idle_q
    m = W.sum(axis=1)
    t2, _k2, t3, _k3 = tables.rate_moment_rows()
    return s_thr, s_acc, s_en, s_idle, (W, W @ t2, W @ t3), m


def epilogue(s_thr, s_acc, s_en, s_idle, walk_in, m, tables, scenario) -> Evaluated:
    W, s2, s3 = walk_in
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
        W0 = idle_wait_ms(md, s_thr.astype(np.float64), np.asarray(s2, dtype=np.float64),
                          np.asarray(s3, dtype=np.float64), c["R"], c["R_q"], inv, rho_c, tables)
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
