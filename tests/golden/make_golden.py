"""Generate golden fixtures from the REFERENCE implementation (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference package (carbon_sched: core.py, mig.py,
errors.py) and records its outputs; the GPU box has no /root/reference, so the
tests compare against these committed vectors there.
"""

import itertools
import json
import math
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from carbon_sched import core, mig, errors  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_l0.json")


def vectors(n):
    for a in range(n + 1):
        for b in range(7 * n // 4 + 1):
            for c in range(7 * n // 3 + 1):
                for d in range(7 * n // 2 + 1):
                    rem = 7 * n - 7 * a - 4 * b - 3 * c - 2 * d
                    if rem < 0:
                        continue
                    for e in range(rem + 1):
                        yield (a, b, c, d, e)


def main():
    topo = mig.DEFAULT_TOPOLOGY
    g = {"source": "reference pkg/src/carbon_sched (core.py, mig.py, errors.py)"}
    rnd = random.Random(230409781)
    seeds = []
    for k in range(60):
        parts = [rnd.getrandbits(rnd.choice([8, 32, 63, 64])) for _ in range(rnd.randint(0, 5))]
        if k % 7 == 0:
            parts.append(-rnd.getrandbits(20))
        seeds.append([parts, core.derive_seed(*parts)])
    g["derive_seed"] = seeds
    g["slice_order"] = [int(s) for s in core.SLICE_ORDER]
    g["labels"] = {s.label: int(s) for s in core.SliceType}
    g["topology"] = topo.to_json_dict()
    g["config_ids"] = list(topo.config_ids)
    # canonical partitions (ordered search) for every vector with CU <= 7n, n <= 4
    parts = {}
    for n in (1, 2, 3, 4):
        feas = {}
        total = 0
        for v in vectors(n):
            total += 1
            r = topo.partition_fleet(mig.from_slice_vector(v), n)
            if r is not None:
                feas[",".join(map(str, v))] = list(r)
        parts[str(n)] = {"checked": total, "feasible": feas}
    g["partition_fleet"] = parts
    # |F_n| by the reference search for n <= 6 (survey: 19, 150, 690, 2238, 5771, 12725)
    counts = {}
    for n in (1, 2, 3, 4, 5, 6):
        counts[str(n)] = sum(1 for v in vectors(n) if topo.is_feasible_fleet(mig.from_slice_vector(v), n))
    g["feasible_counts"] = counts
    # SPEC KAT anchors through the reference code
    g["feasible_kats"] = [
        [["7g"], 1, topo.is_feasible_fleet([core.SliceType.S7G], 1)],
        [["1g"] * 7, 1, topo.is_feasible_fleet([core.SliceType.S1G] * 7, 1)],
        [["7g", "1g"], 1, topo.is_feasible_fleet([core.SliceType.S7G, core.SliceType.S1G], 1)],
    ]
    # ObjectiveParams validation / clamping
    cases = [dict(base_accuracy=0.8, base_carbon_g=10.0, latency_slo_ms=100.0, carbon_weight=w)
             for w in (1.7, -0.2, 0.0, 0.5, 1.0)]
    cases += [dict(base_accuracy=0.0, base_carbon_g=1.0, latency_slo_ms=1.0),
              dict(base_accuracy=1.2, base_carbon_g=1.0, latency_slo_ms=1.0),
              dict(base_accuracy=0.8, base_carbon_g=0.0, latency_slo_ms=1.0),
              dict(base_accuracy=0.8, base_carbon_g=1.0, latency_slo_ms=0.0),
              dict(base_accuracy=0.8, base_carbon_g=1.0, latency_slo_ms=1.0, pue=0.9),
              dict(base_accuracy=float("nan"), base_carbon_g=1.0, latency_slo_ms=1.0),
              dict(base_accuracy=0.8, base_carbon_g=1.0, latency_slo_ms=float("inf"))]
    obj = []
    for kw in cases:
        try:
            o = core.ObjectiveParams(**kw)
            obj.append([{k: (None if isinstance(v, float) and not math.isfinite(v) else v) for k, v in kw.items()},
                        "ok", o.carbon_weight])
        except errors.CarbonSchedError as exc:
            obj.append([{k: (repr(v) if isinstance(v, float) and not math.isfinite(v) else v) for k, v in kw.items()},
                        type(exc).__name__, None])
    g["objective_params"] = obj
    # FleetConfig decode
    fleets = []
    for p in ([1], [10], [19, 19], [3, 12, 1], [2, 17, 18]):
        m = sum(len(topo.config_slices(c)) for c in p)
        a = [rnd.randint(1, 7) for _ in range(m)]
        fc = mig.FleetConfig(p, a)
        fleets.append({"partitions": p, "assignments": a,
                       "slices": [[gi, int(s)] for gi, s in fc.slices()],
                       "instances": [[gi, int(s), v] for gi, s, v in fc.instances()],
                       "slice_counts": {str(int(k)): v for k, v in fc.slice_counts().items()}})
    g["fleets"] = fleets
    bad = []
    for p, a in (([1], []), ([1], [1, 2]), ([], []), ([1], [0]), ([99], [1])):
        try:
            mig.FleetConfig(p, a)
            bad.append([p, a, "ok"])
        except errors.CarbonSchedError as exc:
            bad.append([p, a, type(exc).__name__])
    g["fleet_errors"] = bad
    # error precedence of FleetConfig.__init__ on rows with several defects at once
    # (own RNG so the fixtures above are unchanged)
    r2 = random.Random(2304097810)
    ids = list(topo.config_ids)
    prec = []
    for k in range(200):
        n = r2.randint(1, 6)
        p = [r2.choice(ids) for _ in range(n)]
        m = sum(len(topo.config_slices(c)) for c in p)
        a = [r2.randint(1, 7) for _ in range(m)]
        if r2.random() < 0.3:
            p[r2.randrange(n)] = r2.choice([0, 20, 42, 200])
        if r2.random() < 0.3:
            if a and r2.random() < 0.5:
                a.pop(r2.randrange(len(a)))
            else:
                a.insert(r2.randrange(len(a) + 1), r2.randint(1, 7))
        if a and r2.random() < 0.3:
            a[r2.randrange(len(a))] = 0
        try:
            mig.FleetConfig(p, a)
            prec.append([p, a, "ok"])
        except errors.CarbonSchedError as exc:
            prec.append([p, a, type(exc).__name__])
    g["fleet_error_precedence"] = prec
    with open(OUT, "w") as fh:
        json.dump(g, fh, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
