"""Serving simulator API (SPEC serving-sim module, reference SPEC.md:316-393).

The SPEC's evaluator is a deterministic discrete-event simulation of the
producer / global-FIFO-queue / instance-pull serving system.  Here
every simulation runs on the GPU (``clv_simulate``, csrc/clv_sim.cu: one warp
per fleet, many fleets per launch); this module keeps the SPEC's operation
names and argument meaning:

* ``simulate(fc, profile, w)``            -> SimReport
* ``simulate_fleets(fcs, profile, w)``    -> [SimReport]      (batched, one launch)
* ``p95(latencies)``                      nearest rank
* ``overall_accuracy(report, profile)``
* ``calibrate_arrival_rate(fc, profile, u)``
* ``sla_from_base(n, profile, workload)``

Model details that the SPEC leaves open are fixed in DESIGN.md §11 (integer-ns
time, counter-RNG arrivals and service draws, idle-longest dispatch among idle
instances, warm-up by completion order); ``oracle/des.py`` restates them on the
CPU for the parity tests.  There is no CPU simulation path: without the
library or a GPU these functions raise ``DeviceError``.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .core import SliceType
from .errors import InfeasibleAssignmentError, SimulationError
from .mig import FleetConfig
from .profiles import ProfileTable


@dataclass(frozen=True)
class Workload:
    """Poisson request stream.

    ``periodic`` selects the SPEC's degenerate test mode (arrivals every
    1/arrival_rate_rps seconds); ``warmup`` is the number of first
    completions excluded from latency statistics (None = max(100, 5 % of the
    requests)).  The table surrogate uses the rate only.
    """

    arrival_rate_rps: float
    duration_s: float = 600.0
    seed: int = 0
    periodic: bool = False
    warmup: Optional[int] = None

    def __post_init__(self):
        if not (self.arrival_rate_rps > 0 and math.isfinite(self.arrival_rate_rps)):
            raise SimulationError("arrival_rate_rps must be positive and finite")
        if not (self.duration_s > 0 and math.isfinite(self.duration_s)):
            raise SimulationError("duration_s must be positive and finite")
        if self.warmup is not None and int(self.warmup) < 0:
            raise SimulationError("warmup must be >= 0")


@dataclass(frozen=True)
class SimReport:
    """SPEC:326-330 (+ ``counted``: requests inside the latency statistics, and the
    overall accuracy of SPEC:358 precomputed on the device)."""

    p95_ms: float
    mean_latency_ms: float
    completed: int
    throughput_rps: float
    energy_wh_total: float
    energy_wh_per_request: float
    per_instance_counts: dict = field(default_factory=dict)
    per_variant_counts: dict = field(default_factory=dict)
    sla_met: bool = True
    counted: int = 0
    accuracy: float = float("nan")

    KEYS = ("p95_ms", "mean_latency_ms", "completed", "throughput_rps", "energy_wh_total",
            "energy_wh_per_request", "per_instance_counts", "per_variant_counts", "sla_met", "counted",
            "accuracy")

    def to_json(self) -> str:
        """Fixed key order -- byte-identical for identical reports."""
        d = {}
        for k in self.KEYS:
            v = getattr(self, k)
            if isinstance(v, dict):
                v = {str(kk): int(vv) for kk, vv in sorted(v.items())}
            d[k] = v
        return json.dumps(d, separators=(",", ":"))


def fleet_instances(fc: FleetConfig, profile: ProfileTable) -> np.ndarray:
    """Edge id (v-1)*5 + slice index of every instance, FleetConfig.instances() order."""
    V = profile.variant_count
    out = []
    for _g, s, v in fc.instances():
        if not 1 <= v <= V:
            raise InfeasibleAssignmentError("variant %d not in the %d-variant catalog" % (v, V))
        if not profile.memory_feasible(v, s):
            raise InfeasibleAssignmentError("variant %d does not fit a %s slice" % (v, SliceType(s).label))
        out.append((v - 1) * 5 + SliceType(s).index)
    return np.array(out, dtype=np.uint8)


def _engine(engine):
    if engine is not None:
        return engine
    from .search import default_engine
    return default_engine()


def simulate_fleets(fleets: Sequence[FleetConfig], profile: ProfileTable, w: Workload,
                    l_tail_ms: Optional[float] = None, engine=None, raise_errors: bool = True) -> list:
    """Simulate every fleet under the same workload (common random numbers), one launch."""
    eng = _engine(engine)
    edges, offs = [], [0]
    for fc in fleets:
        e = fleet_instances(fc, profile)
        if len(e) == 0:
            raise SimulationError("fleet has zero instances")
        edges.append(e)
        offs.append(offs[-1] + len(e))
    inst = np.concatenate(edges) if edges else np.zeros(0, dtype=np.uint8)
    reps, vc, ic, _n = eng.simulate(inst, np.array(offs, dtype=np.int64), profile, w,
                                    math.inf if l_tail_ms is None else float(l_tail_ms))
    out = []
    for c, r in enumerate(reps):
        if r["status"] != 0:
            if raise_errors:
                from ._native import STATUS_TO_ERROR
                raise STATUS_TO_ERROR.get(int(r["status"]), SimulationError)(
                    "simulation of fleet %d failed (status %d)" % (c, int(r["status"])))
            out.append(None)
            continue
        per_inst = {j: int(x) for j, x in enumerate(ic[offs[c]:offs[c + 1]])}
        per_var = {v + 1: int(vc[c][v]) for v in range(profile.variant_count)}
        out.append(SimReport(float(r["p95_ms"]), float(r["mean_latency_ms"]), int(r["completed"]),
                             float(r["throughput_rps"]), float(r["energy_wh_total"]),
                             float(r["energy_wh_per_request"]), per_inst, per_var, bool(r["sla_met"]),
                             int(r["counted"]), float(r["accuracy"])))
    return out


def simulate(fc: FleetConfig, profile: ProfileTable, w: Workload, l_tail_ms: Optional[float] = None,
             engine=None) -> SimReport:
    """SPEC:333-343.  Raises InfeasibleAssignmentError / SimulationError as the SPEC lists."""
    return simulate_fleets([fc], profile, w, l_tail_ms, engine)[0]


def p95(latencies: Sequence[float]) -> float:
    """Nearest-rank p95: sorted ascending, element ceil(0.95 N) (1-based)."""
    if len(latencies) == 0:
        raise SimulationError("p95 of an empty sequence")
    v = sorted(latencies)
    n = len(v)
    return v[(95 * n + 99) // 100 - 1]


def overall_accuracy(report: SimReport, profile: ProfileTable) -> float:
    """sum_v count(v) * accuracy(v) / completed."""
    if report.completed <= 0:
        raise SimulationError("no completed requests")
    acc = 0.0
    for v in sorted(report.per_variant_counts):
        acc = acc + float(report.per_variant_counts[v]) * profile.accuracy(v)
    return acc / float(report.completed)


def calibrate_arrival_rate(fc_base: FleetConfig, profile: ProfileTable, utilization_target: float) -> float:
    """utilization_target x sum over instances of 1 / mean_service."""
    if not 0.0 < utilization_target < 1.0:
        raise SimulationError("utilization_target must be in (0, 1)")
    rate = 0.0
    for _g, s, v in fc_base.instances():
        rate = rate + 1000.0 / profile.mean_service_ms(v, s)
    return utilization_target * rate


def sla_from_base(n: int, profile: ProfileTable, workload: Workload, engine=None) -> float:
    """p95 of the BASE configuration under ``workload``."""
    from .search import base_config
    return simulate(base_config(n, profile), profile, workload, engine=engine).p95_ms
