"""Performance profiles, carbon traces and the fixed-point scoring tables.

* ``ProfileTable`` -- per-variant accuracy/memory, per-(variant, slice) service
  time + distribution + energy, per-slice idle power.
* ``CarbonTrace`` / ``intensity_at`` / ``load_trace``.
* ``synthetic_profile`` -- seeded generators for the benchmark families
  (EfficientNet B1-B7, ResNet, BERT, a 3-variant test catalog), seeded by
  ``derive_seed(230409781, family, v, cu)``.
* ``ScoringTables`` -- the per-edge fixed-point rows the device stages in
  shared memory.  Aggregates over a graph are exact int64 sums of these rows,
  so a candidate's score does not depend on summation order; this is what
  makes incremental (delta) neighbour scoring bit-identical to a full
  recompute and to the CPU oracle.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Optional, Sequence

import numpy as np

from .core import SLICE_ORDER, SliceType, derive_seed
from .errors import ProfileError, TraceError
from .mig import DEFAULT_TOPOLOGY, MigTopology

N_KINDS = len(SLICE_ORDER)
DISTS = ("deterministic", "exponential", "lognormal")
Z95 = 1.6448536269514722          # standard-normal 95th percentile
MAX_VARIANTS_DEVICE = 8           # device edge masks are 64-bit; E = 5 V <= 40
PROFILE_SEED = 230409781


@dataclass(frozen=True)
class VariantSpec:
    variant: int
    accuracy: float
    memory_gb: float
    name: str = ""


@dataclass(frozen=True)
class ServiceRow:
    mean_service_ms: float
    dist: str = "deterministic"
    sigma: float = 0.0
    energy_wh_per_request: float = 0.0


def service_p95_ms(row: ServiceRow) -> float:
    """95th percentile of the service-time distribution (host-only transcendental)."""
    if row.dist == "deterministic":
        return row.mean_service_ms
    if row.dist == "exponential":
        return row.mean_service_ms * math.log(20.0)
    # lognormal with the given mean: mu = ln(mean) - sigma^2 / 2
    return row.mean_service_ms * math.exp(Z95 * row.sigma - 0.5 * row.sigma * row.sigma)


class ProfileTable:
    """Immutable profile table with the SPEC:244-247 invariants enforced at construction."""

    def __init__(self, name: str, variants: Sequence[VariantSpec],
                 service: Mapping[tuple[int, SliceType], ServiceRow],
                 idle_power_w: Mapping[SliceType, float],
                 topology: MigTopology = DEFAULT_TOPOLOGY):
        self.name = str(name)
        vs = tuple(sorted(variants, key=lambda x: x.variant))
        if not vs:
            raise ProfileError("profile needs at least one variant")
        if [v.variant for v in vs] != list(range(1, len(vs) + 1)):
            raise ProfileError("variant ids must be contiguous 1..V")
        for a, b in zip(vs, vs[1:]):
            if not b.accuracy > a.accuracy:
                raise ProfileError("accuracy must be strictly increasing in the variant ordinal "
                                   "(v%d=%r, v%d=%r)" % (a.variant, a.accuracy, b.variant, b.accuracy))
        for v in vs:
            if not (0.0 < v.accuracy <= 1.0) or not math.isfinite(v.accuracy):
                raise ProfileError("accuracy of v%d must be in (0,1]" % v.variant)
            if not (v.memory_gb >= 0 and math.isfinite(v.memory_gb)):
                raise ProfileError("memory of v%d must be finite and >= 0" % v.variant)
        rows: dict[tuple[int, SliceType], ServiceRow] = {}
        for (v, s), row in service.items():
            key = (int(v), SliceType(s))
            if key in rows:
                raise ProfileError("duplicate (variant, slice) row %r" % (key,))
            if not 1 <= key[0] <= len(vs):
                raise ProfileError("service row for unknown variant %d" % key[0])
            if row.dist not in DISTS:
                raise ProfileError("unknown service distribution %r" % row.dist)
            if row.dist == "lognormal" and not row.sigma > 0:
                raise ProfileError("lognormal rows need sigma > 0")
            if not (row.mean_service_ms > 0 and math.isfinite(row.mean_service_ms)):
                raise ProfileError("mean_service_ms must be positive")
            if not (row.energy_wh_per_request >= 0 and math.isfinite(row.energy_wh_per_request)):
                raise ProfileError("energy must be >= 0")
            rows[key] = row
        for v in vs:
            for s in SLICE_ORDER:
                if (v.variant, s) not in rows:
                    raise ProfileError("missing service row for (v%d, %s)" % (v.variant, s.label))
            # mean service time non-increasing as compute units grow
            by_cu = sorted(SLICE_ORDER, key=lambda s: s.compute_units)
            for small, big in zip(by_cu, by_cu[1:]):
                if rows[(v.variant, big)].mean_service_ms > rows[(v.variant, small)].mean_service_ms:
                    raise ProfileError("mean_service_ms of v%d grows from %s to %s"
                                       % (v.variant, small.label, big.label))
        idle = {}
        for s in SLICE_ORDER:
            w = float(idle_power_w.get(s, idle_power_w.get(s.label, 0.0)) if isinstance(idle_power_w, dict)
                      else idle_power_w[s])
            if not (w >= 0 and math.isfinite(w)):
                raise ProfileError("idle power must be >= 0")
            idle[s] = w
        self.variants = vs
        self.service = rows
        self.idle_power_w = idle
        self.topology = topology

    # -- lookups ---------------------------------------------------------
    @property
    def variant_count(self) -> int:
        return len(self.variants)

    def accuracy(self, v: int) -> float:
        return self.variants[int(v) - 1].accuracy

    def memory_gb(self, v: int) -> float:
        return self.variants[int(v) - 1].memory_gb

    def memory_feasible(self, v: int, s: SliceType) -> bool:
        """memory_gb(v) <= slice_memory(s)."""
        if not 1 <= int(v) <= len(self.variants):
            raise ProfileError("unknown variant %r" % (v,))
        return self.memory_gb(v) <= self.topology.slice_memory(SliceType(s))

    def mean_service_ms(self, v: int, s: SliceType) -> float:
        return self.service[(int(v), SliceType(s))].mean_service_ms

    def p95_service_ms(self, v: int, s: SliceType) -> float:
        return service_p95_ms(self.service[(int(v), SliceType(s))])

    def energy_wh(self, v: int, s: SliceType) -> float:
        return self.service[(int(v), SliceType(s))].energy_wh_per_request

    def feasible_variants(self, s: SliceType) -> tuple[int, ...]:
        return tuple(v.variant for v in self.variants if self.memory_feasible(v.variant, s))

    def scoring_tables(self) -> "ScoringTables":
        return ScoringTables.from_profile(self)

    def to_json_dict(self) -> dict:
        return {
            "name": self.name,
            "variants": [{"id": v.variant, "name": v.name, "accuracy": v.accuracy,
                          "memory_gb": v.memory_gb} for v in self.variants],
            "latency": [{"variant": v, "slice": s.label, "mean_service_ms": r.mean_service_ms,
                         "dist": r.dist, "sigma": r.sigma}
                        for (v, s), r in sorted(self.service.items(), key=lambda kv: (kv[0][0], kv[0][1].index))],
            "energy": [{"variant": v, "slice": s.label, "wh_per_request": r.energy_wh_per_request}
                       for (v, s), r in sorted(self.service.items(), key=lambda kv: (kv[0][0], kv[0][1].index))],
            "idle": [{"slice": s.label, "watts": self.idle_power_w[s]} for s in SLICE_ORDER],
        }


PROFILE_SECTIONS = ("variants", "latency", "energy", "idle")


def profile_from_dict(doc: Mapping, topology: MigTopology = DEFAULT_TOPOLOGY) -> ProfileTable:
    """Key/value profile document -> ProfileTable.

    Sections ``variants`` (id, accuracy, memory_gb[, name]), ``latency`` (variant,
    slice, mean_service_ms, dist[, sigma]), ``energy`` (variant, slice,
    wh_per_request), ``idle`` (slice, watts).  Schema violations, duplicate
    (variant, slice) rows and non-monotone accuracy raise ProfileError.
    """
    if not isinstance(doc, Mapping):
        raise ProfileError("profile document must be a key/value mapping")
    for sec in PROFILE_SECTIONS:
        if sec not in doc or not isinstance(doc[sec], (list, tuple)):
            raise ProfileError("profile section %r missing or not a list" % sec)

    def field_of(row, key, kind, sec):
        if not isinstance(row, Mapping) or key not in row:
            raise ProfileError("%s row lacks field %r" % (sec, key))
        try:
            return kind(row[key])
        except (TypeError, ValueError) as exc:
            raise ProfileError("%s.%s: %s" % (sec, key, exc)) from exc

    def slice_of(row, sec):
        label = field_of(row, "slice", str, sec)
        try:
            return SliceType.from_label(label)
        except Exception as exc:
            raise ProfileError("%s: unknown slice %r" % (sec, label)) from exc

    variants = []
    seen_v = set()
    for row in doc["variants"]:
        vid = field_of(row, "id", int, "variants")
        if vid in seen_v:
            raise ProfileError("duplicate variant id %d" % vid)
        seen_v.add(vid)
        variants.append(VariantSpec(vid, field_of(row, "accuracy", float, "variants"),
                                    field_of(row, "memory_gb", float, "variants"),
                                    str(row.get("name", "")) if isinstance(row, Mapping) else ""))
    lat: dict = {}
    for row in doc["latency"]:
        key = (field_of(row, "variant", int, "latency"), slice_of(row, "latency"))
        if key in lat:
            raise ProfileError("duplicate latency row (v%d, %s)" % (key[0], key[1].label))
        dist = field_of(row, "dist", str, "latency")
        sigma = float(row.get("sigma", 0.0) or 0.0)
        lat[key] = (field_of(row, "mean_service_ms", float, "latency"), dist, sigma)
    energy: dict = {}
    for row in doc["energy"]:
        key = (field_of(row, "variant", int, "energy"), slice_of(row, "energy"))
        if key in energy:
            raise ProfileError("duplicate energy row (v%d, %s)" % (key[0], key[1].label))
        energy[key] = field_of(row, "wh_per_request", float, "energy")
    idle: dict = {}
    for row in doc["idle"]:
        s = slice_of(row, "idle")
        if s in idle:
            raise ProfileError("duplicate idle row %s" % s.label)
        idle[s] = field_of(row, "watts", float, "idle")
    if set(lat) != set(energy):
        raise ProfileError("latency and energy rows cover different (variant, slice) pairs")
    missing = [s.label for s in SLICE_ORDER if s not in idle]
    if missing:
        raise ProfileError("idle rows missing for %s" % ",".join(missing))
    service = {k: ServiceRow(m, d, sg, energy[k]) for k, (m, d, sg) in lat.items()}
    return ProfileTable(str(doc.get("name", "profile")), variants, service, idle, topology)


def load_profiles(path: str, topology: MigTopology = DEFAULT_TOPOLOGY) -> ProfileTable:
    """load_profiles(path) -> ProfileTable: a JSON (or YAML) key/value document."""
    import json
    try:
        with open(path, "r", encoding="utf-8") as fh:
            text = fh.read()
    except OSError as exc:
        raise ProfileError("cannot read profile %s: %s" % (path, exc)) from exc
    try:
        doc = json.loads(text)
    except ValueError:
        try:
            import yaml
            doc = yaml.safe_load(text)
        except Exception as exc:
            raise ProfileError("profile %s is neither JSON nor YAML: %s" % (path, exc)) from exc
    return profile_from_dict(doc, topology)


def save_profile(profile: ProfileTable, path: str) -> None:
    """Serialise a ProfileTable (round-trips through load_profiles)."""
    import json
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        json.dump(profile.to_json_dict(), fh, indent=1, sort_keys=False)
        fh.write("\n")


def _pow2_scale(max_value: float, bits: int = 31) -> int:
    """Largest k such that max_value * 2**k < 2**bits (k may be negative)."""
    if max_value <= 0:
        return bits - 1
    _m, ex = math.frexp(max_value)      # max_value < 2**ex
    return bits - ex


@dataclass(frozen=True)
class ScoringTables:
    """Per-edge rows of the scoring surrogate, in device edge order e = (v-1)*5 + s.index.

    thr_q[e]  = round(thr(e) * 2^kt)            thr = 1000 / mean_service_ms  (req/s)
    acc_q[e]  = round(thr(e) * acc(v) * 2^kt)   (same scale: A = sum acc_q / sum thr_q)
    en_q[e]   = round(thr(e) * energy(e) * 2^ke)  (Wh/s)
    idle_q[s] = round(idle_w(s) * 2^ki)          (W)
    lat95[e]  = p95 service time (ms), fp64
    svc_ms[e] = mean service time (ms): request shares of the p95 walk
    mem_ok[e] = memory feasibility of the edge
    Each row is < 2^31, so sums over up to 2^21 instances are exact in int64
    and convert exactly to fp64.
    """

    name: str
    variant_count: int
    thr_q: np.ndarray
    acc_q: np.ndarray
    en_q: np.ndarray
    idle_q: np.ndarray
    lat95: np.ndarray
    mem_ok: np.ndarray
    kt: int
    ke: int
    ki: int
    thr: np.ndarray = field(repr=False)
    svc_ms: np.ndarray = field(repr=False, default=None)

    @property
    def n_edges(self) -> int:
        return self.variant_count * N_KINDS

    @classmethod
    def from_profile(cls, p: ProfileTable) -> "ScoringTables":
        V = p.variant_count
        E = V * N_KINDS
        thr = [0.0] * E
        lat = [0.0] * E
        acc_thr = [0.0] * E
        en_thr = [0.0] * E
        mem = [False] * E
        for v in range(1, V + 1):
            for s in SLICE_ORDER:
                e = (v - 1) * N_KINDS + s.index
                row = p.service[(v, s)]
                thr[e] = 1000.0 / row.mean_service_ms
                lat[e] = service_p95_ms(row)
                acc_thr[e] = thr[e] * p.accuracy(v)
                en_thr[e] = thr[e] * row.energy_wh_per_request
                mem[e] = p.memory_feasible(v, s)
        kt = _pow2_scale(max(thr))
        ke = _pow2_scale(max(en_thr))
        ki = _pow2_scale(max(p.idle_power_w.values()))
        thr_q = np.array([round(math.ldexp(x, kt)) for x in thr], dtype=np.int64)
        acc_q = np.array([round(math.ldexp(x, kt)) for x in acc_thr], dtype=np.int64)
        en_q = np.array([round(math.ldexp(x, ke)) for x in en_thr], dtype=np.int64)
        idle_q = np.array([round(math.ldexp(p.idle_power_w[s], ki)) for s in SLICE_ORDER],
                          dtype=np.int64)
        if np.any(thr_q <= 0):
            raise ProfileError("throughput underflows the fixed-point scale")
        svc = [p.service[(v, s)].mean_service_ms for v in range(1, V + 1) for s in SLICE_ORDER]
        return cls(p.name, V, thr_q, acc_q, en_q, idle_q, np.array(lat, dtype=np.float64),
                   np.array(mem, dtype=bool), kt, ke, ki, np.array(thr, dtype=np.float64),
                   np.array(svc, dtype=np.float64))


# ---------------------------------------------------------------------------
# Synthetic families; accuracies are public top-1 / GLUE-style
# numbers used as table inputs, everything else is a seeded model.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class FamilySpec:
    family_id: int
    name: str
    variant_names: tuple
    accuracy: tuple
    memory_gb: tuple
    lat_lo_ms: float
    lat_hi_ms: float
    dist: str = "deterministic"
    sigma: float = 0.0
    power_lo_w: float = 150.0
    power_hi_w: float = 300.0
    idle_full_w: float = 60.0
    alpha: float = 0.8


FAMILIES: dict[str, FamilySpec] = {
    "efficientnet": FamilySpec(0, "efficientnet", ("B1", "B2", "B3", "B4", "B5", "B6", "B7"),
                               (0.791, 0.801, 0.816, 0.829, 0.836, 0.840, 0.843),
                               (0.35, 0.45, 0.6, 0.9, 1.4, 2.0, 2.8), 5.0, 60.0),
    "resnet": FamilySpec(1, "resnet", ("R18", "R34", "R50", "R101", "R152"),
                         (0.698, 0.733, 0.761, 0.774, 0.783),
                         (0.5, 0.8, 1.0, 1.7, 2.3), 4.0, 40.0, "exponential"),
    "bert": FamilySpec(2, "bert", ("tiny", "mini", "small", "medium", "base", "large"),
                       (0.70, 0.75, 0.78, 0.80, 0.84, 0.865),
                       (0.3, 0.6, 1.5, 3.0, 6.0, 11.0), 3.0, 80.0, "lognormal", 0.35,
                       120.0, 320.0),
    "tiny3": FamilySpec(3, "tiny3", ("small", "medium", "large"), (0.70, 0.76, 0.80),
                        (2.0, 6.0, 12.0), 8.0, 40.0),
}


def _unit(*parts: int) -> float:
    return (derive_seed(PROFILE_SEED, *parts) >> 10) * (1.0 / 9007199254740992.0)


def synthetic_profile(name: str = "efficientnet", variants: Optional[int] = None,
                      topology: MigTopology = DEFAULT_TOPOLOGY) -> ProfileTable:
    """Seeded synthetic profile of a named family (optionally its first ``variants`` members).

    mean_service_ms(v, s) = base(v) * (7 / cu(s))^alpha * (1 +- 2%), base geometric
    lat_lo -> lat_hi; active power (cu/7) * P(v); energy = power * service time;
    idle power per slice proportional to cu.
    """
    spec = FAMILIES[name]
    V = len(spec.accuracy) if variants is None else int(variants)
    if not 1 <= V <= len(spec.accuracy):
        raise ProfileError("family %s has %d variants" % (name, len(spec.accuracy)))
    vs = [VariantSpec(v + 1, spec.accuracy[v], spec.memory_gb[v], spec.variant_names[v])
          for v in range(V)]
    full = len(spec.accuracy)
    service: dict[tuple[int, SliceType], ServiceRow] = {}
    for v in range(1, V + 1):
        frac = (v - 1) / (full - 1) if full > 1 else 0.0
        base = spec.lat_lo_ms * (spec.lat_hi_ms / spec.lat_lo_ms) ** frac
        power_full = spec.power_lo_w + (spec.power_hi_w - spec.power_lo_w) * frac
        prev = None
        for s in SLICE_ORDER:                      # 7g first: enforce monotone growth
            cu = s.compute_units
            jitter = 1.0 + 0.04 * (_unit(spec.family_id, v, cu) - 0.5)
            mean = base * (7.0 / cu) ** spec.alpha * jitter
            if prev is not None and mean < prev:
                mean = prev
            prev = mean
            pj = 1.0 + 0.04 * (_unit(spec.family_id, v, cu, 1) - 0.5)
            power = power_full * cu / 7.0 * pj
            energy = power * mean / 1000.0 / 3600.0
            service[(v, s)] = ServiceRow(mean, spec.dist, spec.sigma, energy)
    idle = {s: spec.idle_full_w * s.compute_units / 7.0 for s in SLICE_ORDER}
    return ProfileTable(name if variants is None else "%s%d" % (name, V), vs, service, idle,
                        topology)


# ---------------------------------------------------------------------------
# Carbon-intensity traces
# ---------------------------------------------------------------------------

class CarbonTrace:
    def __init__(self, samples: Iterable[tuple[float, float]]):
        pts = tuple((float(t), float(c)) for t, c in samples)
        if not pts:
            raise TraceError("trace needs at least one sample")
        for (t0, _), (t1, _) in zip(pts, pts[1:]):
            if not t1 > t0:
                raise TraceError("timestamps must be strictly increasing")
        for _, c in pts:
            if not (c >= 0 and math.isfinite(c)):
                raise TraceError("carbon intensity must be finite and >= 0")
        self.samples = pts

    def __len__(self) -> int:
        return len(self.samples)

    def mean(self) -> float:
        return sum(c for _, c in self.samples) / len(self.samples)


def intensity_at(trace: CarbonTrace, t: float) -> float:
    """Step interpolation: latest sample with timestamp <= t, else the first."""
    pts = trace.samples
    lo, hi = 0, len(pts)
    while lo < hi:
        mid = (lo + hi) // 2
        if pts[mid][0] <= t:
            lo = mid + 1
        else:
            hi = mid
    return pts[max(lo - 1, 0)][1]


def load_trace(path: str) -> CarbonTrace:
    """CSV ``timestamp_s,gco2_per_kwh``."""
    try:
        with open(path, "r", encoding="utf-8", newline="") as fh:
            reader = csv.reader(fh)
            header = next(reader, None)
            if header is None or [h.strip() for h in header] != ["timestamp_s", "gco2_per_kwh"]:
                raise TraceError("trace header must be timestamp_s,gco2_per_kwh")
            rows = [(float(r[0]), float(r[1])) for r in reader if r]
    except (OSError, ValueError, IndexError) as exc:
        raise TraceError("malformed trace %s: %s" % (path, exc)) from exc
    return CarbonTrace(rows)


def synthetic_trace(seed: int = 230409781, hours: float = 24.0, step_s: float = 300.0,
                    mean: float = 250.0, amplitude: float = 150.0, noise: float = 20.0) -> CarbonTrace:
    """Diurnal ci = mean + amp*sin(2 pi t / 1 day) + N(0, noise), clipped to [50, 600]."""
    n = int(round(hours * 3600.0 / step_s))
    out = []
    for i in range(n):
        t = i * step_s
        u1 = ((derive_seed(seed, i, 1) >> 10) + 1) * (1.0 / 9007199254740993.0)
        u2 = (derive_seed(seed, i, 2) >> 10) * (1.0 / 9007199254740992.0)
        z = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
        ci = mean + amplitude * math.sin(2.0 * math.pi * t / 86400.0) + noise * z
        out.append((t, min(600.0, max(50.0, ci))))
    return CarbonTrace(out)
