"""GPU parity: every kernel against the CPU oracle on seeded inputs (bit-exact)."""

import numpy as np
import pytest

from oracle.anneal import anneal_chain
from oracle.evaluator import calibrate, evaluate, base_graph
from oracle.search import (Pod, oracle_search, oracle_decode, select_best, sweep_evaluate,
                           draw_candidate, fleet_graph)
from oracle.tables import OracleTables
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY, FleetConfig
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile
from tests.helpers import random_fleet_graphs, perturbed_graphs

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_feasibility_tables_exhaustive_small(engine, feas64):
    for n in range(1, 7):
        vecs = [(a, b, c, d, e) for a in range(n + 1) for b in range(2 * n + 1) for c in range(3 * n + 1)
                for d in range(4 * n + 1) for e in range(7 * n + 2)
                if 7 * a + 4 * b + 3 * c + 2 * d + e <= 7 * n + 1]
        V = np.array(vecs, dtype=np.int32)
        got = engine.feasible(V, n).cpu().numpy().astype(bool)
        exp = feas64.feasible_batch(V, n)
        assert np.array_equal(got, exp), n


@pytest.mark.parametrize("n", [8, 16, 33, 64])
def test_feasibility_tables_random_large(engine, feas64, n):
    rng = np.random.default_rng(n)
    cnt = 200_000
    a = rng.integers(0, max(1, n // 4), cnt)
    b = rng.integers(0, n + 1, cnt)
    c = rng.integers(0, 2 * n + 1, cnt)
    d = rng.integers(0, 3 * n + 1, cnt)
    e = rng.integers(0, 5 * n + 1, cnt)
    V = np.stack([a, b, c, d, e], axis=1).astype(np.int32)
    got = engine.feasible(V, n).cpu().numpy().astype(bool)
    exp = feas64.feasible_batch(V, n)
    assert np.array_equal(got, exp)
    assert 0 < exp.sum() < cnt


def test_realize_matches_host_partition(engine):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    for n in (1, 2, 3, 5, 8):
        W = random_fleet_graphs(T, n, 40, seed=77 + n)
        for w in W:
            vec = w.reshape(7, 5).sum(axis=0)
            assert engine.partition(vec, n) == DEFAULT_TOPOLOGY.partition_vector(vec, n)


@pytest.mark.parametrize("family,n", [("efficientnet", 8), ("bert", 8), ("tiny3", 2), ("resnet", 64)])
def test_score_graphs_bit_exact(engine, family, n):
    prof = synthetic_profile(family)
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, n, 400.0, 0.5)
    base = random_fleet_graphs(T, n, 3000, seed=5)
    W = np.concatenate([base, perturbed_graphs(base, 3000, seed=6)])
    best, outs = engine.score_graphs(W, prof, sc)
    ev = evaluate(W, T, sc)
    from paper_2304_09781_b200.graph import ConfigGraph
    vecs = W.reshape(len(W), T.V, 5).sum(axis=1)
    mem_bad = ((W > 0) & ~T.mem_ok[None, :]).any(axis=1)
    from oracle.feasibility import FeasOracle
    fo = FeasOracle(DEFAULT_TOPOLOGY, n)
    feas = fo.feasible_batch(vecs, n) & ~mem_bad
    got_feas = outs["feasible"].cpu().numpy().astype(bool)
    assert np.array_equal(got_feas, feas)
    for key, arr in (("f", ev.f), ("h", ev.h), ("p95", ev.L)):
        assert bits_equal(outs[key].cpu().numpy()[feas], arr[feas]), key
    assert np.array_equal(outs["sla"].cpu().numpy()[feas].astype(bool), ev.sla[feas])
    h = np.where(feas, ev.h, np.inf)
    sla = ev.sla & feas
    exp_i = select_best(h, sla)
    assert best["index"] == exp_i
    assert best["valid_count"] == int(feas.sum())
    assert bits_equal([best["h"], best["f"], best["p95_ms"]], [ev.h[exp_i], ev.f[exp_i], ev.L[exp_i]])


def test_score_x_matches_oracle(engine):
    prof = synthetic_profile("bert")
    T = OracleTables.from_profile(prof)
    n = 40
    sc = calibrate(prof, T, n, 250.0, 0.3)
    pods = [Pod(T, sc, n, 1.0)]
    fleets = []
    for i in range(500):
        (parts, assign), = draw_candidate(99, i, pods, DEFAULT_TOPOLOGY)
        fleets.append(FleetConfig(parts, assign))
    best, outs = engine.score_fleets(fleets, prof, sc)
    W = np.array([fleet_graph(f.partitions, f.assignments, DEFAULT_TOPOLOGY, T) for f in fleets])
    ev = evaluate(W, T, sc)
    assert bits_equal(outs["f"].cpu().numpy(), ev.f)
    assert bits_equal(outs["h"].cpu().numpy(), ev.h)
    assert best["index"] == select_best(ev.h, ev.sla)


def test_oracle_search_c0(engine):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, 1, 400.0, 0.5)
    i, ev, W = oracle_search(DEFAULT_TOPOLOGY, T, sc, 1)
    got = engine.oracle_search(prof, sc)
    assert got["total"] == 983_899 == len(W)
    assert got["index"] == i
    assert bits_equal([got["f"], got["h"], got["p95_ms"]], [ev.f[i], ev.h[i], ev.L[i]])
    assert engine.oracle_decode(prof, i) == oracle_decode(i, DEFAULT_TOPOLOGY, T)
    assert got["sla_count"] == int(ev.sla.sum())


def _chain_compare(engine, prof, T, starts, scs, ap, seed, n, feas, cluster=0):
    batch = engine.anneal(starts, prof, scs, ap, seed, n=n, cluster=cluster, log=True)
    host = batch.host()
    for c in range(len(starts)):
        sc = scs[c] if len(scs) > 1 else scs[0]
        out = anneal_chain(starts[c], n, T, sc, ap, seed, c, feas, log=True)
        r = host["results"][c]
        assert r["status"] == out.status, c
        assert r["steps"] == out.steps, c
        assert r["evals"] == out.evals, c
        assert r["best_step"] == out.best_step, c
        assert r["best_index"] == out.best_idx, c
        assert np.array_equal(host["best_w"][c].astype(np.int64), out.best_w), c
        assert np.array_equal(host["final_w"][c].astype(np.int64), out.final_w), c
        assert bits_equal([r["f"], r["h"], r["p95_ms"]], [out.best["f"], out.best["h"], out.best["L"]]), c
        assert bool(r["sla_met"]) == out.best["sla"]
        lg = host["log"][c][: out.steps]
        assert [bool(x) for x in lg["accepted"]] == [row["accepted"] for row in out.log]
        assert bits_equal(lg["h"], [row["h"] for row in out.log])
        assert bits_equal(lg["temp"], [row["temp"] for row in out.log])


@pytest.mark.parametrize("proposal,evaluate_mode", [("best", "all"), ("uniform", "all"), ("uniform", "proposal")])
def test_anneal_c1_lambda_sweep(engine, feas64, proposal, evaluate_mode):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 8
    lams = [i / 10 for i in range(11)]
    scs = [calibrate(prof, T, n, 400.0, lam) for lam in lams]
    starts = np.repeat(base_graph(7, n)[None, :], len(lams), axis=0)
    ap = AnnealParams(proposal=proposal, evaluate=evaluate_mode, max_steps=40)
    _chain_compare(engine, prof, T, starts, scs, ap, 1234, n, feas64)


def test_anneal_random_starts_memory_limited(engine, feas64):
    prof = synthetic_profile("bert")
    T = OracleTables.from_profile(prof)
    n = 12
    sc = calibrate(prof, T, n, 300.0, 0.5)
    starts = random_fleet_graphs(T, n, 16, seed=4242)
    ap = AnnealParams(proposal="uniform", max_steps=30, stall_limit=8)
    _chain_compare(engine, prof, T, starts, [sc], ap, 99, n, feas64, cluster=2)


def test_anneal_n64_chains(engine, feas64):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 64
    sc = calibrate(prof, T, n, 400.0, 0.5)
    starts = random_fleet_graphs(T, n, 4, seed=64)
    ap = AnnealParams(max_steps=12)
    _chain_compare(engine, prof, T, starts, [sc], ap, 7, n, feas64, cluster=8)


def test_sweep_two_pods(engine):
    pr, pb = synthetic_profile("resnet"), synthetic_profile("bert")
    Tr, Tb = OracleTables.from_profile(pr), OracleTables.from_profile(pb)
    n = 16
    sr, sb = calibrate(pr, Tr, n, 300.0, 0.5), calibrate(pb, Tb, n, 300.0, 0.5)
    pods_o = [Pod(Tr, sr, n, 0.5), Pod(Tb, sb, n, 0.5)]
    pods_e = [(pr, sr, n, 0.5), (pb, sb, n, 0.5)]
    f, h, sla = sweep_evaluate(2024, 1000, 3000, pods_o, DEFAULT_TOPOLOGY)
    best, outs = engine.sweep(pods_e, 1000, 3000, 2024, outputs=True)
    assert bits_equal(outs["f"].cpu().numpy(), f)
    assert bits_equal(outs["h"].cpu().numpy(), h)
    assert np.array_equal(outs["sla"].cpu().numpy().astype(bool), sla)
    assert best["index"] == select_best(h, sla, 1000)
    fleets = engine.sweep_decode(pods_e, 2024, best["index"])
    exp = draw_candidate(2024, best["index"], pods_o, DEFAULT_TOPOLOGY)
    assert [(list(f.partitions), list(f.assignments)) for f in fleets] == [(p, a) for p, a in exp]


def test_sweep_wide_pod_direct_sums(engine):
    """A pod wider than the sweep's 16-bit edge counters allow (7 x 9,400 slices >= 2^16)
    takes the per-draw row sums; same bits as the oracle."""
    pr = synthetic_profile("resnet")
    Tr = OracleTables.from_profile(pr)
    n = 9400
    sr = calibrate(pr, Tr, n, 300.0, 0.5)
    f, h, sla = sweep_evaluate(7, 0, 3, [Pod(Tr, sr, n, 1.0)], DEFAULT_TOPOLOGY)
    best, outs = engine.sweep([(pr, sr, n, 1.0)], 0, 3, 7, outputs=True)
    assert bits_equal(outs["f"].cpu().numpy(), f)
    assert bits_equal(outs["h"].cpu().numpy(), h)


def test_run_trace_matches_oracle_controller(engine, feas64):
    from oracle.controller import run_trace_clover
    from paper_2304_09781_b200.controller import run_trace, ControllerParams
    from paper_2304_09781_b200.profiles import CarbonTrace, synthetic_trace
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    tr = synthetic_trace(hours=1.5)               # 18 ticks
    ap = AnnealParams(proposal="uniform", max_steps=8)
    n, chains = 8, 4
    rep = run_trace(engine, tr, "clover", n, prof, 0.5, ap, ControllerParams(), seed=5, chains=chains)
    ref = run_trace_clover(tr.samples, n, prof, T, 0.5, ap, 5, chains, feas64)
    assert len(rep.rows) == len(ref)
    replan_ticks = [r.tick for r in rep.replans]
    assert replan_ticks == [x["tick"] for x in ref if x["replanned"]]
    assert [r.accepted for r in rep.replans] == [x["accepted"] for x in ref if x["replanned"]]
    for row, x in zip(rep.rows, ref):
        assert row["sla_met"] == x["sla"]
        assert row["accuracy"] == x["accuracy"]
    assert rep.rows[-1]["cumulative_gco2"] == ref[-1]["cum"]


@pytest.mark.parametrize("multi", [False, True])
def test_anneal_exact_division_path(engine, feas64, multi):
    """Scenarios outside fast_div_safe's ranges (here 1 - rho_sat < 1e-12) run the kernel
    with IEEE divisions; single- and per-chain-scenario launches stay bit-exact."""
    from dataclasses import replace
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    n = 16
    base = calibrate(prof, T, n, 380.0, 0.5)
    scs = [replace(calibrate(prof, T, n, 380.0, lam), rho_sat=1.0 - 1e-13) for lam in (0.2, 0.5, 0.8)]
    if not multi:
        scs = scs[1:2]
    assert base.rho_sat != scs[0].rho_sat
    starts = random_fleet_graphs(T, n, 3, seed=77)
    ap = AnnealParams(max_steps=16)
    _chain_compare(engine, prof, T, starts, scs if multi else scs * 1, ap, 5, n, feas64, cluster=3)
