"""CPU tests of the serving-simulator restatement (oracle/des.py) and the host-side
simulator API (paper_2304_09781_b200/sim.py): the SPEC serving-sim examples
(reference SPEC.md:340-375), its invariants and the deterministic
transcendental helpers the kernel shares."""

import math
import statistics

import numpy as np
import pytest

from oracle import des
from paper_2304_09781_b200 import sim as S
from paper_2304_09781_b200.core import SliceType
from paper_2304_09781_b200.mig import FleetConfig
from paper_2304_09781_b200.profiles import ProfileTable, ServiceRow, VariantSpec, synthetic_profile


def one_edge(mean_ms=10.0, energy=0.001, idle=0.0, dist=0, sigma=0.0):
    return des.SimInput([des.SimEdge(mean_ms, dist, sigma, energy)] * 5, [idle] * 5, [0.8])


def test_log_clv_matches_libm():
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.random(20000), 10.0 ** rng.uniform(-300, 300, 20000), [1.0, 2.0, 0.5, 1e-308]])
    worst = 0.0
    for x in xs:
        x = float(x)
        if x <= 0:
            continue
        b = math.log(x)
        a = des.log_clv(x)
        if b != 0:
            worst = max(worst, abs(a - b) / abs(b))
        else:
            assert a == 0.0
    assert worst < 5e-16


def test_ndtri_clv_matches_normal_quantile():
    nd = statistics.NormalDist()
    for p in (1e-300, 1e-12, 1e-6, 0.001, 0.02, 0.02425, 0.1, 0.3, 0.5, 0.7, 0.9, 0.975, 0.99, 1 - 1e-9):
        assert abs(des.ndtri_clv(p) - nd.inv_cdf(p)) <= 1.2e-9 * max(1.0, abs(nd.inv_cdf(p)))


def test_spec_p95_examples():
    # SPEC:353-356
    assert des.p95(list(range(1, 101))) == 95
    assert des.p95([7]) == 7
    assert des.p95([5] * 20) == 5
    assert S.p95(list(range(1, 101))) == 95 and S.p95([7]) == 7 and S.p95([5] * 20) == 5
    with pytest.raises(Exception):
        S.p95([])


def test_spec_unloaded_periodic_queue():
    # 1 instance, 10 ms deterministic, arrivals every 20 ms, 100 requests
    r = des.simulate([0], one_edge(), 50.0, 2.0, 1, periodic=True, warmup=0)
    assert r.completed == 100 and r.p95_ms == 10.0 and r.throughput_rps == 50.0
    assert r.mean_latency_ms == 10.0


def test_spec_saturated_periodic_queue():
    # arrivals every 5 ms -> request i waits (i-1)*5 ms; p95 = 10 + 94*5 = 480 ms
    r = des.simulate([0], one_edge(), 200.0, 0.5, 1, periodic=True, warmup=0, keep_latencies=True)
    assert r.completed == 100
    assert r.latencies_ns == [(10 + 5 * i) * 1_000_000 for i in range(100)]
    assert r.p95_ms == 480.0


def test_spec_energy_without_idle_power():
    # idle_power = 0, N completed, e per request -> total = N e
    r = des.simulate([0], one_edge(energy=0.25), 50.0, 2.0, 1, periodic=True, warmup=0)
    assert r.energy_wh_total == 100 * 0.25 == r.energy_wh_per_request * r.completed


def test_idle_energy_makes_total_larger():
    r = des.simulate([0, 1], one_edge(energy=0.001, idle=30.0), 20.0, 5.0, 9, warmup=0)
    assert r.energy_wh_per_request * r.completed < r.energy_wh_total


def test_determinism_and_counts_invariant():
    sim = des.sim_input(synthetic_profile("resnet"))
    a = des.simulate([0, 7, 13, 24], sim, 150.0, 30.0, 5)
    b = des.simulate([0, 7, 13, 24], sim, 150.0, 30.0, 5)
    assert a == b
    assert a.completed == sum(a.per_instance_counts) == sum(a.per_variant_counts)
    assert a.counted == a.completed - des.default_warmup(a.completed)


def test_fifo_on_single_deterministic_instance():
    r = des.simulate([0], one_edge(mean_ms=7.0), 180.0, 3.0, 4, trace=True)
    comps = [c for (_a, _s, c, _j) in r.trace]
    assert comps == sorted(comps)


def test_work_conservation():
    sim = des.sim_input(synthetic_profile("bert"))
    inst = [0, 6, 12, 18, 24]
    r = des.simulate(inst, sim, 400.0, 10.0, 11, trace=True)
    busy_until = []
    free = [0] * len(inst)
    for (a, s, c, j) in r.trace:
        if s > a:                    # the request queued: every instance was busy at its arrival
            assert all(f > a for f in free)
        assert s == max(a, free[j]) and free[j] == min(free)
        free[j] = c
        busy_until.append(c)


def test_throughput_share_under_saturation():
    # two instances with rates mu1 > mu2 under saturation share requests ~ mu1/mu2
    sim = des.SimInput([des.SimEdge(10.0, 0, 0.0, 0.0), des.SimEdge(25.0, 0, 0.0, 0.0)] + [des.SimEdge(1.0, 0, 0.0, 0.0)] * 3,
                       [0.0] * 5, [0.8])
    r = des.simulate([0, 1], sim, 200.0, 60.0, 2)      # capacity 140 rps < 200 rps
    assert r.completed >= 10_000
    ratio = r.per_instance_counts[0] / r.per_instance_counts[1]
    assert abs(ratio / 2.5 - 1.0) < 0.05


def test_exponential_and_lognormal_service_means():
    n = 20000
    for dist, sigma in ((1, 0.0), (2, 0.5)):
        e = des.SimEdge(10.0, dist, sigma, 0.0)
        xs = [des.service_ns(e, *des.multipliers(17, i)) for i in range(n)]
        m = sum(xs) / n / 1e6
        assert abs(m / 10.0 - 1.0) < 0.03


def test_overall_accuracy_examples():
    # SPEC:362-366
    p = synthetic_profile("tiny3")
    rep = lambda counts: S.SimReport(1.0, 1.0, sum(counts.values()), 1.0, 1.0, 1.0, {}, counts)
    a = {v: p.accuracy(v) for v in (1, 2, 3)}
    assert S.overall_accuracy(rep({1: 0, 2: 0, 3: 10}), p) == a[3]
    assert abs(S.overall_accuracy(rep({1: 50, 2: 0, 3: 50}), p) - (a[1] + a[3]) / 2) < 1e-15
    assert abs(S.overall_accuracy(rep({1: 25, 2: 0, 3: 75}), p) - (0.25 * a[1] + 0.75 * a[3])) < 1e-15


def _flat_profile(mean_ms):
    vs = [VariantSpec(1, 0.8, 1.0)]
    service = {(1, s): ServiceRow(mean_ms, "deterministic", 0.0, 0.001) for s in SliceType}
    return ProfileTable("flat", vs, service, {s: 0.0 for s in SliceType})


def test_calibrate_arrival_rate_examples():
    # SPEC:372-375
    p100 = _flat_profile(100.0)
    fc10 = FleetConfig([1] * 10, [1] * 10, p100.topology)
    assert abs(S.calibrate_arrival_rate(fc10, p100, 0.7) - 70.0) < 1e-12
    p10 = _flat_profile(10.0)
    assert abs(S.calibrate_arrival_rate(FleetConfig([1], [1], p10.topology), p10, 0.5) - 50.0) < 1e-12


def test_report_json_is_byte_stable():
    r = S.SimReport(1.5, 1.0, 10, 2.0, 3.0, 0.3, {1: 4, 0: 6}, {2: 10, 1: 0}, True, 8, 0.8)
    assert r.to_json() == S.SimReport(1.5, 1.0, 10, 2.0, 3.0, 0.3, {0: 6, 1: 4}, {1: 0, 2: 10}, True, 8, 0.8).to_json()
    assert r.to_json().index('"p95_ms"') < r.to_json().index('"per_variant_counts"')


def test_fleet_instances_order_and_memory_errors():
    p = synthetic_profile("efficientnet")
    fc = FleetConfig([19, 1], [1] * 7 + [7], p.topology)
    e = S.fleet_instances(fc, p)
    assert list(e) == des.fleet_edges(fc)
    bad = FleetConfig([19], [7] * 7, p.topology)       # B7 (2.8 GB) still fits 1g (5 GB)
    S.fleet_instances(bad, p)
    big = synthetic_profile("bert")                     # large (11 GB) does not fit 1g / 2g
    with pytest.raises(S.InfeasibleAssignmentError):
        S.fleet_instances(FleetConfig([19], [6] * 7, big.topology), big)


def test_workload_validation():
    with pytest.raises(S.SimulationError):
        S.Workload(0.0)
    with pytest.raises(S.SimulationError):
        S.Workload(1.0, duration_s=-1)
    with pytest.raises(S.SimulationError):
        S.Workload(1.0, warmup=-2)
