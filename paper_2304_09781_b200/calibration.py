"""Profile calibration to the SPEC's anchors (reference SPEC.md:300-303, acceptance 5).

The SPEC ships its default profile *calibrated*: (a) CO2OPT's per-request carbon is
about 30 % below an unpartitioned fleet running the same (smallest) variant -- the
partitioning opportunity of PAPER §3 -- and (b) a mixed standardized configuration
exists with >= 60 % carbon saving at <= 5 % accuracy loss.  Calibration "adjusts energy
rows" (the profile's `energy` and `idle` rows): at the calibrated arrival rate the
fleets run far below capacity, so idle power dominates the per-request carbon and
hides the partitioning gain.  The idle rows are scaled by gamma in [0, 1] (bisection)
and, only if gamma = 0 still misses the gap, the active energy of slice s by
(cu / 7)^beta.  Every candidate is evaluated on the device (``clv_score_graphs``);
anchor (b) is checked with the device ORACLE under the accuracy threshold
(``clv_oracle_search``).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .graph import build_graph
from .mig import FleetConfig
from .profiles import ProfileTable


@dataclass
class CalibrationReport:
    gamma: float                # idle-power scale
    beta: float
    co2opt_gap: float           # 1 - E(CO2OPT) / E(unpartitioned, same variant)
    best_saving_pct: float      # max Delta-Carbon of a standardized config within the accuracy loss
    best_accuracy_loss_pct: float
    anchor_a: bool
    anchor_b: bool


def scale_energy(profile: ProfileTable, beta: float, gamma: float = 1.0,
                 name: Optional[str] = None) -> ProfileTable:
    """Active energy per request of slice s times (cu(s) / 7)^beta; idle power times gamma."""
    service = {}
    for (v, s), row in profile.service.items():
        k = (s.compute_units / 7.0) ** beta
        service[(v, s)] = replace(row, energy_wh_per_request=row.energy_wh_per_request * k)
    idle = {s: w * gamma for s, w in profile.idle_power_w.items()}
    return ProfileTable(name or "%s_b%.4f_g%.4f" % (profile.name, beta, gamma), profile.variants, service,
                        idle, profile.topology)


def _bisect(f, lo, hi, target, iters):
    """x in [lo, hi] with f(x) ~ target for a monotone f (either direction)."""
    f_lo, f_hi = f(lo), f(hi)
    if (f_lo - target) * (f_hi - target) > 0:
        return lo if abs(f_lo - target) <= abs(f_hi - target) else hi
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        f_mid = f(mid)
        if (f_lo - target) * (f_mid - target) <= 0:
            hi = mid
        else:
            lo, f_lo = mid, f_mid
    return 0.5 * (lo + hi)


def _co2opt_gap(engine, profile: ProfileTable, n: int, ci: float) -> float:
    from .search import co2opt_config
    co = co2opt_config(n, profile)
    same = FleetConfig([1] * n, [1] * n, profile.topology)
    sc = engine.calibrate(profile, n, ci, 0.5)
    W = np.array([build_graph(co, profile).weights, build_graph(same, profile).weights], dtype=np.uint16)
    energies = []
    for w in W:
        best, _ = engine.score_graphs(w[None, :], profile, sc, outputs=False)
        energies.append(best["energy_wh"])
    return 1.0 - energies[0] / energies[1]


def calibrate_profile(profile: ProfileTable, engine=None, gap: float = 0.30, n: int = 8, ci: float = 400.0,
                      max_loss_pct: float = 5.0, min_saving_pct: float = 60.0,
                      iters: int = 40) -> tuple[ProfileTable, CalibrationReport]:
    """Scale the energy rows so that CO2OPT saves ``gap`` of the same-variant unpartitioned
    fleet's per-request carbon, then report anchor (b) from the device ORACLE (n = 1)."""
    if engine is None:
        from .search import default_engine
        engine = default_engine(profile.topology)
    gap_of = lambda beta, gamma: _co2opt_gap(engine, scale_energy(profile, beta, gamma), n, ci)
    gamma = _bisect(lambda g: gap_of(0.0, g), 0.0, 1.0, gap, iters)
    beta = 0.0
    if gap_of(0.0, gamma) < gap - 0.05:                   # idle alone cannot open the gap
        gamma = 0.0
        beta = _bisect(lambda b: gap_of(b, 0.0), 0.0, 4.0, gap, iters)
    out = scale_energy(profile, beta, gamma, name=profile.name + "_calibrated")
    achieved = _co2opt_gap(engine, out, n, ci)
    # anchor (b): best Delta-Carbon of a standardized configuration within the accuracy loss
    sc = engine.calibrate(out, 1, ci, 1.0)
    sc = replace(sc, max_accuracy_loss_pct=float(max_loss_pct))
    best = engine.oracle_search(out, sc)
    acc_loss = 100.0 * (sc.obj.base_accuracy - best["accuracy"]) / sc.obj.base_accuracy if best["found"] else 100.0
    saving = best["f"] if best["found"] and best["sla_met"] else float("-inf")   # lambda = 1: f = Delta-Carbon
    rep = CalibrationReport(gamma, beta, achieved, saving, acc_loss, abs(achieved - gap) <= 0.05,
                            bool(best["found"] and best["sla_met"] and saving >= min_saving_pct))
    return out, rep
