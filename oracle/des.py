"""ORACLE -- TEST INFRASTRUCTURE ONLY.  The serving simulator (SPEC serving-sim module).

A pure-Python restatement of the SPEC's discrete-event simulator
(reference SPEC.md:316-393: simulate, p95, overall_accuracy,
calibrate_arrival_rate) in the exact form DESIGN.md §11 fixes for the device:

* time is integer nanoseconds; arrivals are Poisson (counter RNG, gaps rounded
  to ns) or periodic (the SPEC's degenerate test mode);
* one global FIFO queue, instance-pull dispatch: request i, in
  arrival order, is served by the instance that became idle first
  (argmin (free_j, j)), start = max(a_i, free_j);
* service time of request i on edge e: deterministic mean, or the mean times a
  unit-mean exponential / lognormal multiplier drawn from request i's counter
  stream (common random numbers across candidates);
* warm-up: the first W completions (ordered by (completion, request)) are
  excluded from latency statistics, W = max(100, N // 20) by default
  (SPEC:361); p95 is nearest-rank;
* energy = sum of per-request active energy + per-instance idle power x idle
  time over [0, max(duration, last completion)].

Everything that feeds a comparison is an exact integer or a fixed sequence of
IEEE operations (log_clv, ndtri_clv, exp_clv use only + - * / sqrt, frexp and
ldexp), so the CUDA kernel reproduces every report field bit for bit.  This
module uses heapq and runs at ~1 us per request: keep N <= ~2e5 in tests.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

from .rng import derive_seed, exp_clv

# fdlibm e_log.c constants (public domain algorithm, restated)
_LN2_HI = 6.93147180369123816490e-01
_LN2_LO = 1.90821492927058770002e-10
_LG = (6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,
       2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,
       1.479819860511658591e-01)
_SQRT_HALF = 0.70710678118654752440

# Acklam's rational approximation of the standard-normal quantile
_A = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
      1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_B = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
      6.680131188771972e+01, -1.328068155288572e+01)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
      -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
      3.754408661907416e+00)
_P_LOW = 0.02425

TWO_M53 = 1.0 / 9007199254740992.0
TWO_M52 = 1.0 / 4503599627370496.0


def log_clv(x: float) -> float:
    """Natural log of a positive finite double (fdlibm kernel over frexp)."""
    m, e = math.frexp(x)
    if m < _SQRT_HALF:
        m = m * 2.0
        e -= 1
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    w = z * z
    t1 = w * (_LG[1] + w * (_LG[3] + w * _LG[5]))
    t2 = z * (_LG[0] + w * (_LG[2] + w * (_LG[4] + w * _LG[6])))
    r = t2 + t1
    hfsq = 0.5 * f * f
    dk = float(e)
    return dk * _LN2_HI - ((hfsq - (s * (hfsq + r) + dk * _LN2_LO)) - f)


def ndtri_clv(p: float) -> float:
    """Standard-normal quantile for p in (0, 1) (Acklam, |rel err| < 1.2e-9)."""
    if p < _P_LOW:
        q = math.sqrt(-2.0 * log_clv(p))
        num = ((((_C[0] * q + _C[1]) * q + _C[2]) * q + _C[3]) * q + _C[4]) * q + _C[5]
        den = (((_D[0] * q + _D[1]) * q + _D[2]) * q + _D[3]) * q + 1.0
        return num / den
    if p > 1.0 - _P_LOW:
        q = math.sqrt(-2.0 * log_clv(1.0 - p))
        num = ((((_C[0] * q + _C[1]) * q + _C[2]) * q + _C[3]) * q + _C[4]) * q + _C[5]
        den = (((_D[0] * q + _D[1]) * q + _D[2]) * q + _D[3]) * q + 1.0
        return -(num / den)
    q = p - 0.5
    r = q * q
    num = (((((_A[0] * r + _A[1]) * r + _A[2]) * r + _A[3]) * r + _A[4]) * r + _A[5]) * q
    den = ((((_B[0] * r + _B[1]) * r + _B[2]) * r + _B[3]) * r + _B[4]) * r + 1.0
    return num / den


def round_ns(x: float) -> int:
    return int(math.floor(x + 0.5))


# ----------------------------------------------------------------- inputs ---
@dataclass(frozen=True)
class SimEdge:
    """Per-(variant, slice) service row of the simulator."""

    mean_ms: float
    dist: int            # 0 deterministic, 1 exponential, 2 lognormal
    sigma: float
    energy_wh: float


@dataclass(frozen=True)
class SimInput:
    edges: Sequence[SimEdge]          # E = 5 V, index (v-1)*5 + slice index
    idle_w: Sequence[float]           # per slice kind (SLICE_ORDER index)
    accuracy: Sequence[float]         # per variant (0-based)


def sim_input(profile) -> SimInput:
    """Simulator rows of a ProfileTable-like object."""
    dists = {"deterministic": 0, "exponential": 1, "lognormal": 2}
    V = profile.variant_count
    slices = sorted(profile.idle_power_w, key=lambda s: s.index)
    edges = []
    for v in range(1, V + 1):
        for s in slices:
            row = profile.service[(v, s)]
            edges.append(SimEdge(row.mean_service_ms, dists[row.dist], row.sigma if row.dist == "lognormal" else 0.0,
                                 row.energy_wh_per_request))
    return SimInput(edges, [profile.idle_power_w[s] for s in slices], [profile.accuracy(v) for v in range(1, V + 1)])


def fleet_edges(fc) -> list[int]:
    """Edge (v-1)*5 + slice index of every instance, in FleetConfig.instances() order."""
    return [(v - 1) * 5 + s.index for _g, s, v in fc.instances()]


def default_warmup(n_requests: int) -> int:
    return max(100, n_requests // 20)


def arrivals(rate_rps: float, duration_s: float, seed: int, periodic: bool) -> list[int]:
    d_ns = round_ns(duration_s * 1e9)
    out = []
    if periodic:
        period = round_ns(1e9 / rate_rps)
        if period < 1:
            period = 1
        i = 0
        while i * period < d_ns:
            out.append(i * period)
            i += 1
        return out
    scale = 1e9 / rate_rps
    t = 0
    i = 0
    while True:
        u = ((derive_seed(seed, 1, i) >> 10) + 1) * TWO_M53
        g = -log_clv(u)
        t += round_ns(g * scale)
        if t >= d_ns:
            return out
        out.append(t)
        i += 1


def multipliers(seed: int, i: int) -> tuple[float, float]:
    """(unit exponential, standard normal) draws of request i."""
    v = ((derive_seed(seed, 2, i) >> 10) + 1) * TWO_M53
    w = ((derive_seed(seed, 3, i) >> 11) + 0.5) * TWO_M52
    return -log_clv(v), ndtri_clv(w)


def service_ns(edge: SimEdge, ex: float, z: float) -> int:
    mean_ns = edge.mean_ms * 1e6
    if edge.dist == 0:
        return round_ns(mean_ns)
    if edge.dist == 1:
        return round_ns(mean_ns * ex)
    hs = (0.5 * edge.sigma) * edge.sigma
    return round_ns(mean_ns * exp_clv(edge.sigma * z - hs))


@dataclass
class OracleReport:
    p95_ms: float
    mean_latency_ms: float
    completed: int
    counted: int
    throughput_rps: float
    energy_wh_total: float
    energy_wh_per_request: float
    accuracy: float
    sla_met: bool
    per_instance_counts: list = field(default_factory=list)
    per_variant_counts: list = field(default_factory=list)
    latencies_ns: Optional[list] = None
    trace: Optional[list] = None         # (arrival, start, completion, instance) per request


def nearest_rank(m: int) -> int:
    """1-based nearest rank of the 95th percentile: ceil(0.95 m)."""
    return (95 * m + 99) // 100


def simulate(instances: Sequence[int], sim: SimInput, rate_rps: float, duration_s: float, seed: int,
             periodic: bool = False, warmup: Optional[int] = None, l_tail_ms: float = math.inf,
             keep_latencies: bool = False, trace: bool = False) -> OracleReport:
    """instances: edge index per instance, in FleetConfig.instances() order."""
    K = len(instances)
    if K == 0:
        raise ValueError("zero instances")
    arr = arrivals(rate_rps, duration_s, seed, periodic)
    N = len(arr)
    W = default_warmup(N) if warmup is None else int(warmup)
    if N - W < 1:
        raise ValueError("no request left after warm-up")
    heap = [(0, j) for j in range(K)]          # (free time, instance): argmin (free, j)
    cnt = [0] * K
    busy = [0] * K
    comp = [0] * N
    lat = [0] * N
    need_rand = any(sim.edges[e].dist != 0 for e in instances)
    tr = [] if trace else None
    for i, a in enumerate(arr):
        free, j = heapq.heappop(heap)
        start = a if a > free else free
        ex, z = multipliers(seed, i) if need_rand else (0.0, 0.0)
        s = service_ns(sim.edges[instances[j]], ex, z)
        c = start + s
        heapq.heappush(heap, (c, j))
        cnt[j] += 1
        busy[j] += s
        comp[i] = c
        lat[i] = c - a
        if tr is not None:
            tr.append((a, start, c, j))
    t_end = max(round_ns(duration_s * 1e9), max(comp))
    order = sorted(range(N), key=lambda i: (comp[i], i))
    counted = sorted(lat[i] for i in order[W:])
    M = len(counted)
    p95_ns = counted[nearest_rank(M) - 1]
    mean_ms = (float(sum(counted)) / float(M)) / 1e6
    E = len(sim.edges)
    cnt_e = [0] * E
    idle_s = [0] * 5
    for j, e in enumerate(instances):
        cnt_e[e] += cnt[j]
        idle_s[e % 5] += t_end - busy[j]
    active = 0.0
    for e in range(E):
        active = active + float(cnt_e[e]) * sim.edges[e].energy_wh
    total = active
    for s_ in range(5):
        total = total + sim.idle_w[s_] * float(idle_s[s_]) / 3.6e12
    V = len(sim.accuracy)
    cnt_v = [sum(cnt_e[(v * 5):(v * 5 + 5)]) for v in range(V)]
    acc = 0.0
    for v in range(V):
        acc = acc + float(cnt_v[v]) * sim.accuracy[v]
    acc = acc / float(N)
    p95_ms = float(p95_ns) / 1e6
    return OracleReport(p95_ms=p95_ms, mean_latency_ms=mean_ms, completed=N, counted=M,
                        throughput_rps=float(N) / duration_s, energy_wh_total=total,
                        energy_wh_per_request=active / float(N), accuracy=acc,
                        sla_met=p95_ms <= l_tail_ms, per_instance_counts=cnt, per_variant_counts=cnt_v,
                        latencies_ns=lat if keep_latencies else None, trace=tr)


def p95(values: Sequence[float]) -> float:
    """Nearest-rank p95 of a non-empty sequence."""
    if not values:
        raise ValueError("empty input")
    v = sorted(values)
    return v[nearest_rank(len(v)) - 1]


def aggregate_service_rate(instances: Sequence[int], sim: SimInput) -> float:
    """sum over instances of 1 / mean_service (requests per second)."""
    tot = 0.0
    for e in instances:
        tot = tot + 1000.0 / sim.edges[e].mean_ms
    return tot
