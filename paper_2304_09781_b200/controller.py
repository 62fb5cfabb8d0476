"""Trace-driven re-planning controller (BASELINE configs[3]).

``run_trace`` ticks through a carbon-intensity trace every ``trace_step_s``; when
``reopt_needed`` fires (|Δci|/ci > 5 %) it re-plans with
the chosen scheme starting from the incumbent, seeded by
``derive_seed(seed, tick)``, keeps the incumbent unless the result
meets the p95 SLA (strict SLA), diffs the realized FleetConfigs for the
reconfiguration downtime and accrues carbon between ticks
(× PUE).  Every re-plan's time-to-solution is recorded (device time
of the search launch + winner exchange, and host wall time including realize).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from .core import derive_seed
from .engine import CloverEngine
from .errors import CarbonSchedError
from .graph import ConfigGraph, build_graph
from .objective import AnnealParams, Scenario
from .profiles import CarbonTrace, ProfileTable, intensity_at

SCHEMES = ("base", "co2opt", "blover", "clover", "oracle")


@dataclass(frozen=True)
class ControllerParams:
    """SPEC:569-572."""

    reopt_threshold: float = 0.05
    reconfig_downtime_s: float = 30.0
    trace_step_s: float = 300.0

    def __post_init__(self):
        if not self.reopt_threshold > 0 or self.reconfig_downtime_s < 0 or not self.trace_step_s > 0:
            raise CarbonSchedError("invalid controller parameters")


def reopt_needed(prev_ci: float, ci: float, p: ControllerParams = ControllerParams()) -> bool:
    """|ci - prev| / prev > threshold; prev = 0 always re-optimises."""
    if prev_ci <= 0:
        return True
    return abs(ci - prev_ci) / prev_ci > p.reopt_threshold


@dataclass
class Replan:
    tick: int
    t: float
    ci: float
    prev_ci: float
    device_ms: float
    wall_ms: float
    evals: int
    accepted: bool
    f: float
    h: float
    p95_ms: float
    sla_met: bool
    changed_gpus: int


@dataclass
class TimelineReport:
    rows: list = field(default_factory=list)
    replans: list = field(default_factory=list)
    summary: dict = field(default_factory=dict)
    evals_log: Optional[np.ndarray] = None     # LOG_DTYPE [1, max_steps] of the last Clover re-plan
    evals_steps: Optional[list] = None


def _score(engine, profile, w, scenario):
    best, _ = engine.score_graphs(np.asarray(w, dtype=np.uint16)[None, :], profile, scenario, outputs=False)
    if not best["found"]:
        raise CarbonSchedError("active configuration is not realizable")
    return best


def _changed_gpus(a, b) -> int:
    """GPUs whose partition or any assignment differs between two realized fleets."""
    if a is None:
        return len(b.partitions)
    ga, gb = a.instances(), b.instances()
    per_a = {}
    for g, s, v in ga:
        per_a.setdefault(g, []).append((int(s), v))
    per_b = {}
    for g, s, v in gb:
        per_b.setdefault(g, []).append((int(s), v))
    return sum(1 for g in range(len(b.partitions)) if per_a.get(g) != per_b.get(g))


def run_trace(engine: CloverEngine, trace: CarbonTrace, scheme: str, n: int, profile: ProfileTable,
              lam: float = 0.5, ap: Optional[AnnealParams] = None, cp: ControllerParams = ControllerParams(),
              seed: int = 0, chains: int = 128, utilization: float = 0.7, strict_sla: bool = True,
              pue: float = 1.5, chain_base: int = 0, group=None, des_window_s: float = 0.0,
              des_top: int = 16, log_evals: bool = False,
              max_acc_loss_pct: Optional[float] = None) -> TimelineReport:
    """Trace-driven control loop for ``scheme`` in SCHEMES.

    ``des_window_s`` > 0 turns on DES confirmation: L_tail_DES is the
    simulated p95 of BASE (sla_from_base); at every Clover re-plan the
    ``des_top`` best distinct chain winners (surrogate order: SLA first, then h) are
    realized and simulated in one batch, and the first whose simulated p95 meets
    L_tail_DES is the candidate; every timeline row carries the simulated p95 of the
    active fleet.  ``log_evals`` keeps the winning chain's per-step log of the last
    Clover re-plan (evals.csv).  ``max_acc_loss_pct`` is accuracy_threshold_mode
    (SPEC:612-627): candidates losing more accuracy than that count as SLA-violating
    in best tracking, so the controller never deploys them."""
    import torch
    from .search import anneal_chains, base_config, co2opt_config
    if scheme not in SCHEMES:
        raise CarbonSchedError("unknown scheme %r" % scheme)
    ap = ap or AnnealParams(proposal="uniform", evaluate="all", max_steps=64)
    ci_mean = trace.mean()
    # L_tail and C_base from BASE at the trace's mean intensity (D7)
    base_sc = engine.calibrate(profile, n, ci_mean, lam, utilization, ci_base=ci_mean, pue=pue)
    if max_acc_loss_pct is not None:
        base_sc = replace(base_sc, max_accuracy_loss_pct=float(max_acc_loss_pct))
    base_w = np.array(build_graph(base_config(n, profile), profile).weights, dtype=np.int64)
    if scheme == "co2opt":
        w = np.array(build_graph(co2opt_config(n, profile), profile).weights, dtype=np.int64)
    else:
        w = base_w.copy()
    fleet = engine.realize(ConfigGraph(w, profile.variant_count, profile.name), n)
    rep = TimelineReport()
    des_cache: dict = {}
    l_tail_des = None
    if des_window_s > 0:
        from .sim import Workload, simulate_fleets
        from .search import base_config as _bc
        des_w = Workload(base_sc.arrival_rps, float(des_window_s), derive_seed(seed, 0x5EED))
        l_tail_des = simulate_fleets([_bc(n, profile)], profile, des_w, engine=engine)[0].p95_ms

        def des_p95(fleets):
            todo = [f for f in fleets if f not in des_cache]
            if todo:
                for f, r in zip(todo, simulate_fleets(todo, profile, des_w, l_tail_des, engine=engine)):
                    des_cache[f] = r.p95_ms
            return [des_cache[f] for f in fleets]
    prev_ci = 0.0
    cum, cum_base, acc_sum = 0.0, 0.0, 0.0
    steps = int(round((trace.samples[-1][0] - trace.samples[0][0]) / cp.trace_step_s)) + 1
    t0 = trace.samples[0][0]
    for tick in range(steps):
        t = t0 + tick * cp.trace_step_s
        ci = intensity_at(trace, t)
        sc = base_sc.with_ci(ci)
        optimizing = False
        if scheme in ("clover", "oracle", "blover") and reopt_needed(prev_ci, ci, cp):
            optimizing = True
            tick_seed = derive_seed(seed, tick)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if scheme == "clover":
                starts = np.repeat(w[None, :].astype(np.uint16), chains, axis=0)
                res = anneal_chains(engine, starts, profile, sc, ap, tick_seed, chain_base=chain_base,
                                    group=group, log=log_evals)
                cand_w = np.asarray(res.best.graph.weights, dtype=np.int64)
                cand = dict(f=res.best.f_value, h=res.best.h_value, p95_ms=res.best.p95_ms,
                            sla_met=res.best.sla_met)
                evals = res.evals
                if log_evals and res.log is not None:
                    loc = res.best_chain - chain_base
                    rep.evals_log = res.log[loc:loc + 1]
                    rep.evals_steps = [int(res.results[loc]["steps"])]
                if des_window_s > 0:
                    cand_w, cand, des_evals = _des_confirm(engine, profile, n, res, des_p95, l_tail_des, des_top,
                                                           cand_w, cand)
                    evals += des_evals
            elif scheme == "oracle":
                o = engine.oracle_search(profile, sc)
                cid, assign = engine.oracle_decode(profile, o["index"])
                from .mig import FleetConfig
                fc = FleetConfig([cid] * n, list(assign) * n, profile.topology)
                cand_w = np.array(build_graph(fc, profile).weights, dtype=np.int64)
                cand = dict(f=o["f"], h=o["h"], p95_ms=o["p95_ms"], sla_met=bool(o["sla_met"]))
                evals = o["valid_count"]
            else:
                # the same termination rules as the anneal re-plan (SPEC acceptance 7): draws
                # bounded by max_steps + 1 and the time budget, stall_limit without a new best
                from .search import blover_run
                fc, best, blog = blover_run(engine, profile, sc, n, ap, tick_seed)
                cand_w = np.array(build_graph(fc, profile).weights, dtype=np.int64)
                cand = dict(f=best["f"], h=best["h"], p95_ms=best["p95_ms"], sla_met=bool(best["sla_met"]))
                evals = len(blog)
            e1.record()
            torch.cuda.synchronize()
            dev_ms = e0.elapsed_time(e1)
            cur = _score(engine, profile, w, sc)
            better = (cand["sla_met"] and not cur["sla_met"]) or \
                     (cand["sla_met"] == bool(cur["sla_met"]) and cand["h"] < cur["h"])
            accepted = bool(better and (cand["sla_met"] or not strict_sla))
            changed = 0
            if accepted:
                new_fleet = engine.realize(ConfigGraph(cand_w, profile.variant_count, profile.name), n)
                changed = _changed_gpus(fleet, new_fleet)
                fleet, w = new_fleet, cand_w
            wall_ms = 1000.0 * (time.perf_counter() - w0)
            rep.replans.append(Replan(tick, t, ci, prev_ci, dev_ms, wall_ms, int(evals), accepted, cand["f"],
                                      cand["h"], cand["p95_ms"], bool(cand["sla_met"]), changed))
            prev_ci = ci
        elif prev_ci <= 0:
            prev_ci = ci
        act = _score(engine, profile, w, sc)
        base = _score(engine, profile, base_w, sc)
        reqs = sc.arrival_rps * cp.trace_step_s
        g_req = act["energy_wh"] / 1000.0 * ci * pue
        cum += reqs * g_req
        cum_base += reqs * (base["energy_wh"] / 1000.0 * ci * pue)   # same op order as the active fleet
        acc_sum += act["accuracy"]
        row = dict(t=t, ci=ci, scheme=scheme, p95_ms=act["p95_ms"], sla_met=bool(act["sla_met"]),
                   accuracy=act["accuracy"], gco2_per_request=g_req, cumulative_gco2=cum, optimizing=optimizing)
        if des_window_s > 0:
            dp = des_p95([fleet])[0]
            row.update(des_p95_ms=dp, des_sla_met=bool(dp <= l_tail_des))
        rep.rows.append(row)
    tts = [r.device_ms for r in rep.replans]
    rep.summary = dict(
        scheme=scheme, n_gpus=n, ticks=steps, replans=len(rep.replans), total_gco2=cum,
        carbon_saved_vs_base_pct=100.0 * (cum_base - cum) / cum_base if cum_base > 0 else 0.0,
        mean_accuracy=acc_sum / steps, base_accuracy=base_sc.obj.base_accuracy,
        accuracy_delta_vs_base_pct=100.0 * (acc_sum / steps - base_sc.obj.base_accuracy) / base_sc.obj.base_accuracy,
        sla_violation_ticks=sum(1 for r in rep.rows if not r["sla_met"]),
        replan_device_ms_mean=float(np.mean(tts)) if tts else 0.0,
        replan_device_ms_max=float(np.max(tts)) if tts else 0.0,
        replan_wall_ms_mean=float(np.mean([r.wall_ms for r in rep.replans])) if tts else 0.0,
        candidates_scored=int(sum(r.evals for r in rep.replans)),
        # share of the trace span spent optimising (here: measured re-plan wall time)
        optimization_time_fraction_pct=100.0 * sum(r.wall_ms for r in rep.replans) / 1000.0
        / max(steps * cp.trace_step_s, 1e-9),
        reconfigured_gpus=int(sum(r.changed_gpus for r in rep.replans)),
        downtime_gpu_s=float(sum(r.changed_gpus for r in rep.replans) * cp.reconfig_downtime_s))
    if des_window_s > 0:
        rep.summary.update(des_window_s=float(des_window_s), des_l_tail_ms=l_tail_des,
                           des_sla_violation_ticks=sum(1 for r in rep.rows if not r["des_sla_met"]),
                           des_simulations=len(des_cache))
    return rep


def _des_confirm(engine, profile, n, res, des_p95, l_tail_des, top, cand_w, cand):
    """Simulate the best distinct chain winners; keep the first (surrogate order) whose
    simulated p95 meets L_tail_DES.  Returns (graph, candidate dict, simulations run)."""
    order = np.lexsort((np.arange(len(res.results)), res.results["h"], res.results["sla_met"] == 0))
    graphs, rows, seen = [], [], set()
    for c in order:
        key = res.best_w[c].tobytes()
        if key in seen or res.results[c]["status"] < 0:
            continue
        seen.add(key)
        graphs.append(res.best_w[c].astype(np.int64))
        rows.append(res.results[c])
        if len(graphs) >= top:
            break
    fleets = [engine.realize(ConfigGraph(g, profile.variant_count, profile.name), n) for g in graphs]
    p95s = des_p95(fleets)
    for g, r, p in zip(graphs, rows, p95s):
        if p <= l_tail_des:
            return g, dict(f=float(r["f"]), h=float(r["h"]), p95_ms=float(r["p95_ms"]), sla_met=bool(r["sla_met"]),
                           des_p95_ms=p), len(fleets)
    cand = dict(cand)
    cand["sla_met"] = False                  # no simulated winner meets the SLA: keep the incumbent
    return cand_w, cand, len(fleets)
