"""GPU parity of the batched serving simulator (clv_simulate, csrc/clv_sim.cu) against
the CPU restatement oracle/des.py: every SimReport field and every per-instance /
per-variant count bit-exact, the SPEC serving-sim examples through the device, and
the SPEC invariants at sizes the oracle cannot reach."""

import math

import numpy as np
import pytest

from oracle import des
from oracle.search import Pod, draw_candidate
from oracle.tables import OracleTables
from paper_2304_09781_b200 import sim as S
from paper_2304_09781_b200.errors import InfeasibleAssignmentError, SimulationError
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY, FleetConfig
from paper_2304_09781_b200.profiles import ProfileTable, ServiceRow, VariantSpec, synthetic_profile
from paper_2304_09781_b200.core import SliceType

pytestmark = pytest.mark.gpu

FIELDS = ("p95_ms", "mean_latency_ms", "completed", "counted", "throughput_rps", "energy_wh_total",
          "energy_wh_per_request", "accuracy")


def random_fleets(profile, n, count, seed):
    T = OracleTables.from_profile(profile)
    out = []
    for i in range(count):
        (parts, assign), = draw_candidate(seed, i, [Pod(T, None, n, 1.0)], DEFAULT_TOPOLOGY)
        out.append(FleetConfig(parts, assign, DEFAULT_TOPOLOGY))
    return out


def assert_same(dev: S.SimReport, ref: des.OracleReport, tag=""):
    for k in FIELDS:
        a, b = getattr(dev, k), getattr(ref, k)
        assert a == b, "%s %s: device %r oracle %r" % (tag, k, a, b)
    assert [dev.per_instance_counts[j] for j in range(len(ref.per_instance_counts))] == ref.per_instance_counts, tag
    assert [dev.per_variant_counts[v + 1] for v in range(len(ref.per_variant_counts))] == ref.per_variant_counts, tag


def _flat(mean_ms, energy=0.001, idle=0.0):
    vs = [VariantSpec(1, 0.8, 1.0)]
    service = {(1, s): ServiceRow(mean_ms, "deterministic", 0.0, energy) for s in SliceType}
    return ProfileTable("flat%g_%g_%g" % (mean_ms, energy, idle), vs, service, {s: idle for s in SliceType})


def test_spec_periodic_examples_on_device(engine):
    p = _flat(10.0)
    fc = FleetConfig([1], [1], p.topology)
    r = S.simulate(fc, p, S.Workload(50.0, 2.0, 1, periodic=True, warmup=0), engine=engine)
    assert (r.completed, r.p95_ms, r.throughput_rps) == (100, 10.0, 50.0)
    r = S.simulate(fc, p, S.Workload(200.0, 0.5, 1, periodic=True, warmup=0), engine=engine)
    assert (r.completed, r.p95_ms) == (100, 480.0)
    pe = _flat(10.0, energy=0.25)
    r = S.simulate(FleetConfig([1], [1], pe.topology), pe, S.Workload(50.0, 2.0, 1, periodic=True, warmup=0),
                   engine=engine)
    assert r.energy_wh_total == 25.0


@pytest.mark.parametrize("family,n,rate,dur", [("efficientnet", 2, 60.0, 40.0), ("resnet", 4, 300.0, 30.0),
                                               ("bert", 3, 90.0, 60.0), ("tiny3", 1, 40.0, 100.0)])
def test_parity_random_fleets(engine, family, n, rate, dur):
    p = synthetic_profile(family)
    fleets = random_fleets(p, n, 6, 77 + n)
    w = S.Workload(rate, dur, 1234 + n)
    l_tail = 150.0
    reps = S.simulate_fleets(fleets, p, w, l_tail_ms=l_tail, engine=engine)
    sim = des.sim_input(p)
    for c, fc in enumerate(fleets):
        ref = des.simulate(des.fleet_edges(fc), sim, rate, dur, 1234 + n, l_tail_ms=l_tail)
        assert_same(reps[c], ref, "%s fleet %d" % (family, c))
        assert reps[c].sla_met == ref.sla_met


def test_parity_saturated_and_warmup_variants(engine):
    p = synthetic_profile("resnet")
    fleets = random_fleets(p, 1, 4, 5)
    sim = des.sim_input(p)
    for warm in (0, 7, None, 1500):
        w = S.Workload(400.0, 8.0, 99, warmup=warm)           # overloaded: queue grows
        reps = S.simulate_fleets(fleets, p, w, engine=engine)
        for c, fc in enumerate(fleets):
            ref = des.simulate(des.fleet_edges(fc), sim, 400.0, 8.0, 99, warmup=warm)
            assert_same(reps[c], ref, "warmup %r fleet %d" % (warm, c))


def test_batch_is_order_free_and_deterministic(engine):
    p = synthetic_profile("bert")
    fleets = random_fleets(p, 8, 20, 3)
    w = S.Workload(500.0, 20.0, 8)
    a = S.simulate_fleets(fleets, p, w, engine=engine)
    b = S.simulate_fleets(list(reversed(fleets)), p, w, engine=engine)
    assert [x.to_json() for x in a] == [x.to_json() for x in reversed(b)]
    assert all(x.completed == sum(x.per_instance_counts.values()) == sum(x.per_variant_counts.values()) for x in a)


def test_errors(engine):
    big = synthetic_profile("bert")
    with pytest.raises(InfeasibleAssignmentError):
        S.simulate(FleetConfig([19], [6] * 7, big.topology), big, S.Workload(10.0, 10.0), engine=engine)
    p = synthetic_profile("tiny3")
    with pytest.raises(SimulationError):      # 10 requests, default warm-up 100 -> nothing counted
        S.simulate(FleetConfig([1], [1], p.topology), p, S.Workload(1.0, 10.0), engine=engine)


def test_throughput_share_and_sla_from_base(engine):
    # SPEC:380 on the device at >= 10^4 requests
    vs = [VariantSpec(1, 0.7, 1.0), VariantSpec(2, 0.8, 1.0)]
    service = {}
    for s in SliceType:
        service[(1, s)] = ServiceRow(10.0, "deterministic", 0.0, 0.0)
        service[(2, s)] = ServiceRow(25.0, "deterministic", 0.0, 0.0)
    p = ProfileTable("share", vs, service, {s: 0.0 for s in SliceType})
    r = S.simulate(FleetConfig([1, 1], [1, 2], p.topology), p, S.Workload(200.0, 60.0, 2), engine=engine)
    assert r.completed >= 10_000
    assert abs(r.per_variant_counts[1] / r.per_variant_counts[2] / 2.5 - 1.0) < 0.05
    # sla_from_base: deterministic 100 ms instances, light load -> l_tail = 100 ms
    p100 = _flat(100.0)
    assert S.sla_from_base(4, p100, S.Workload(2.0, 600.0, 1), engine=engine) == 100.0
    lo = S.sla_from_base(4, p100, S.Workload(20.0, 300.0, 1), engine=engine)
    hi = S.sla_from_base(4, p100, S.Workload(36.0, 300.0, 1), engine=engine)
    assert hi >= lo


def test_large_fleet_properties(engine):
    # n = 64 fleets (up to 448 instances), 10 simulated minutes at 0.7 x BASE capacity
    p = synthetic_profile("efficientnet")
    from paper_2304_09781_b200.search import base_config
    rate = S.calibrate_arrival_rate(base_config(64, p), p, 0.7)
    fleets = random_fleets(p, 64, 16, 21) + [base_config(64, p)]
    w = S.Workload(rate, 600.0, 5)
    reps = S.simulate_fleets(fleets, p, w, engine=engine)
    for r, fc in zip(reps, fleets):
        assert r.completed == reps[0].completed
        assert r.completed == sum(r.per_instance_counts.values())
        assert len(r.per_instance_counts) == fc.n_instances
        assert r.energy_wh_per_request * r.completed <= r.energy_wh_total
        assert abs(S.overall_accuracy(r, p) - r.accuracy) <= 1e-15
    base = reps[-1]
    assert abs(base.accuracy - p.accuracy(p.variant_count)) <= 1e-15


def test_run_trace_with_des_confirmation(engine, tmp_path):
    """SPEC acceptance 6 analogue with the simulator as the judge: every steady-state tick of the
    DES-confirmed Clover controller serves a fleet whose simulated p95 meets L_tail_DES."""
    from paper_2304_09781_b200.controller import ControllerParams, run_trace
    from paper_2304_09781_b200.objective import AnnealParams
    from paper_2304_09781_b200.profiles import synthetic_trace
    from paper_2304_09781_b200 import reports as R
    prof = synthetic_profile("efficientnet")
    tr = synthetic_trace(hours=2.0)
    ap = AnnealParams(proposal="uniform", max_steps=16)
    rep = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=3, chains=16,
                    des_window_s=120.0, des_top=8, log_evals=True)
    assert rep.summary["des_l_tail_ms"] > 0 and rep.summary["des_simulations"] >= 1
    assert all(r["des_sla_met"] for r in rep.rows)
    assert rep.summary["replans"] >= 1 and rep.evals_log is not None
    R.write_trace_run(str(tmp_path), rep)
    lines = open(tmp_path / "evals.csv").read().splitlines()
    assert lines[0] == ",".join(R.EVAL_FIELDS) and len(lines) == 1 + rep.evals_steps[0]
    again = run_trace(engine, tr, "clover", 8, prof, 0.5, ap, ControllerParams(), seed=3, chains=16,
                      des_window_s=120.0, des_top=8)
    R.write_timeline_csv(str(tmp_path / "t2.csv"), again)
    assert open(tmp_path / "t2.csv").read() == open(tmp_path / "timeline.csv").read()


def test_parity_ties_and_many_sigma_classes(engine):
    """Deterministic service on identical instances (every dispatch is a tie on free time,
    broken by instance order) and a catalog whose lognormal rows use several sigmas
    (one multiplier class each)."""
    vs = [VariantSpec(v, 0.7 + 0.03 * v, 1.0) for v in range(1, 5)]
    det = {(v, s): ServiceRow(12.0, "deterministic", 0.0, 0.002) for v in range(1, 5) for s in SliceType}
    pd = ProfileTable("ties", vs, det, {s: 3.0 for s in SliceType})
    fc = FleetConfig([19, 19], [1, 2, 3, 4, 1, 2, 3] * 2, pd.topology)
    sim = des.sim_input(pd)
    for periodic, rate in ((True, 400.0), (False, 300.0)):
        w = S.Workload(rate, 5.0, 4, periodic=periodic, warmup=13)
        r = S.simulate(fc, pd, w, engine=engine)
        ref = des.simulate(des.fleet_edges(fc), sim, rate, 5.0, 4, periodic=periodic, warmup=13)
        assert_same(r, ref, "ties periodic=%s" % periodic)
    sig = {}
    for v in range(1, 5):
        for s in SliceType:
            sig[(v, s)] = ServiceRow(8.0 + v, "lognormal", 0.1 * v + (0.05 * (s.index % 2) if v < 3 else 0.0), 0.001)
    pl = ProfileTable("sigmas", vs, sig, {s: 2.0 for s in SliceType})
    fleets = random_fleets(pl, 3, 5, 12)
    w = S.Workload(250.0, 20.0, 9)
    reps = S.simulate_fleets(fleets, pl, w, engine=engine)
    siml = des.sim_input(pl)
    for c, f in enumerate(fleets):
        assert_same(reps[c], des.simulate(des.fleet_edges(f), siml, 250.0, 20.0, 9), "sigmas %d" % c)


def test_too_many_sigma_classes_only_blocks_simulation(engine):
    from paper_2304_09781_b200.errors import ProfileError
    vs = [VariantSpec(v, 0.7 + 0.03 * v, 1.0) for v in range(1, 5)]
    sig = {(v, s): ServiceRow(8.0 + v, "lognormal", 0.1 * v + 0.05 * (s.index % 2), 0.001)
           for v in range(1, 5) for s in SliceType}                     # 8 distinct sigmas
    p = ProfileTable("sigmas8", vs, sig, {s: 2.0 for s in SliceType})
    fc = FleetConfig([1, 1], [1, 4], p.topology)
    best, _ = engine.score_fleets([fc], p, engine.calibrate(p, 2, 300.0, 0.5))
    assert best["found"]
    with pytest.raises(ProfileError):
        S.simulate(fc, p, S.Workload(50.0, 10.0, 1), engine=engine)
