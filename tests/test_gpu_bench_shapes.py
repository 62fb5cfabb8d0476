"""Parity at the exact shapes the benchmark times (BASELINE.json configs[2..4]).

* c2: the per-GPU shard of the 8-GPU run -- 128 chains of the n = 64 EfficientNet fleet from the
  bench's incumbent perturbations, auto cluster size, max_steps 256 (chains run to the stall
  rule), the single-scenario branch-free-division instantiation -- every chain bit for bit
  against oracle/anneal.py; and the default bench launch, the whole 1024-chain
  re-plan on one GPU, its first and last 64 chains.
* c3: the trace controller at n = 64 with 128 chains per re-plan over 6 h of the synthetic
  trace (72 ticks), against oracle/controller.py.
* c4: 10^4 contiguous indices of the two-pod (ResNet / BERT) sweep at 128 GPUs per pod
  against oracle/search.py.
The oracle runs are spread over the host's cores (independent chains / index ranges)."""

import multiprocessing as mp
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_G = {}


def _pool():
    return mp.get_context("fork").Pool(max(1, min(32, len(os.sched_getaffinity(0)))))


def _chain_job(a):
    from oracle.anneal import anneal_chain
    w, n, tables, sc, ap, s, c = a
    return anneal_chain(w, n, tables, sc, ap, s, c, _G["feas"])


def test_c2_headline_launch_all_chains(engine):
    import bench
    from paper_2304_09781_b200.profiles import synthetic_profile
    prof = synthetic_profile(bench.FAMILY)
    sc = engine.calibrate(prof, bench.N_FLEET, bench.CI, bench.LAMBDA)
    ap = bench.anneal_params(256)
    starts = bench.make_starts(prof, bench.SEED, 3 * 128, 128, 0.75)      # the bench's first timed step
    seed = bench.SEED + 3
    batch = engine.anneal(starts, prof, sc, ap, seed, chain_base=0, cluster=0)
    _cpu, outs = bench.cpu_replan(starts, seed, 256)
    par = bench.chain_parity(outs, batch)
    assert par["chains"] == 128 and par["bit_exact"], par["mismatched_chains"]
    res = batch.host()["results"]
    assert (res["status"] == 1).all()                 # every chain converged (stall rule)
    assert res["sla_met"].mean() > 0.5


def test_c2_whole_replan_1024_chains(engine, feas64):
    """The default bench launch: all 1024 chains of c2 on one B200 (cluster size 1, several
    waves).  Chains from the first and the last waves (ids 0-63 and 960-1023) bit for bit
    against oracle/anneal.py."""
    import bench
    from oracle.tables import OracleTables
    from paper_2304_09781_b200.profiles import synthetic_profile
    prof = synthetic_profile(bench.FAMILY)
    T = OracleTables.from_profile(prof)
    sc = engine.calibrate(prof, bench.N_FLEET, bench.CI, bench.LAMBDA)
    from oracle.evaluator import calibrate
    osc = calibrate(prof, T, bench.N_FLEET, bench.CI, bench.LAMBDA)
    ap = bench.anneal_params(256)
    C = bench.C2_CHAINS
    starts = bench.make_starts(prof, bench.SEED, 3 * C, C, 0.75)          # the bench's first timed step
    seed = bench.SEED + 3
    h = engine.anneal(starts, prof, sc, ap, seed, chain_base=0, cluster=0).host()
    ids = list(range(64)) + list(range(C - 64, C))
    _G["feas"] = feas64
    with _pool() as pool:
        outs = pool.map(_chain_job, [(starts[c].astype(np.int64), bench.N_FLEET, T, osc, ap, seed, c) for c in ids],
                        chunksize=1)
    u64 = lambda x: np.float64(x).view(np.uint64)
    for c, o in zip(ids, outs):
        r = h["results"][c]
        assert (int(r["status"]), int(r["steps"]), int(r["evals"]), int(r["best_index"])) == \
            (o.status, o.steps, o.evals, o.best_idx), c
        assert np.array_equal(h["best_w"][c].astype(np.int64), o.best_w), c
        assert np.array_equal(h["final_w"][c].astype(np.int64), o.final_w), c
        assert u64(r["h"]) == u64(o.best["h"]) and u64(r["p95_ms"]) == u64(o.best["L"]), c


def test_c3_trace_n64_128_chains_6h(engine, feas64):
    from oracle.controller import run_trace_clover
    from oracle.tables import OracleTables
    from paper_2304_09781_b200.controller import ControllerParams, run_trace
    from paper_2304_09781_b200.objective import AnnealParams
    from paper_2304_09781_b200.profiles import synthetic_profile, synthetic_trace
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    tr = synthetic_trace(hours=6.0)
    ap = AnnealParams(proposal="uniform", evaluate="all", max_steps=64)
    n, chains, seed = 64, 128, 230409781
    rep = run_trace(engine, tr, "clover", n, prof, 0.5, ap, ControllerParams(), seed=seed, chains=chains)
    _G["feas"] = feas64
    with _pool() as pool:
        ref = run_trace_clover(tr.samples, n, prof, T, 0.5, ap, seed, chains, feas64,
                               map_fn=lambda fn, jobs: pool.map(_chain_job, [j[:7] for j in jobs]))
    assert len(rep.rows) == len(ref) == 72
    assert [r.tick for r in rep.replans] == [x["tick"] for x in ref if x["replanned"]]
    assert [r.accepted for r in rep.replans] == [x["accepted"] for x in ref if x["replanned"]]
    assert len(rep.replans) >= 5
    for row, x in zip(rep.rows, ref):
        assert row["sla_met"] == x["sla"] and row["accuracy"] == x["accuracy"]
    assert rep.rows[-1]["cumulative_gco2"] == ref[-1]["cum"]


def _sweep_job(a):
    from oracle.search import sweep_evaluate
    from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
    b, e = a
    return sweep_evaluate(_G["seed"], b, e, _G["pods"], DEFAULT_TOPOLOGY)


def test_c4_two_pod_sweep_10k_contiguous(engine):
    from oracle.evaluator import calibrate
    from oracle.search import Pod, select_best
    from oracle.tables import OracleTables
    from paper_2304_09781_b200.profiles import synthetic_profile
    pr, pb = synthetic_profile("resnet"), synthetic_profile("bert")
    Tr, Tb = OracleTables.from_profile(pr), OracleTables.from_profile(pb)
    n = 128
    sr, sb = calibrate(pr, Tr, n, 350.0, 0.5), calibrate(pb, Tb, n, 350.0, 0.5)
    seed, begin, count = 230409781, 123_456_789, 10_000
    best, outs = engine.sweep([(pr, sr, n, 0.5), (pb, sb, n, 0.5)], begin, begin + count, seed, outputs=True)
    _G["seed"], _G["pods"] = seed, [Pod(Tr, sr, n, 0.5), Pod(Tb, sb, n, 0.5)]
    cuts = np.linspace(begin, begin + count, 65).astype(np.int64)
    with _pool() as pool:
        parts = pool.map(_sweep_job, list(zip(cuts[:-1].tolist(), cuts[1:].tolist())))
    f = np.concatenate([p[0] for p in parts])
    h = np.concatenate([p[1] for p in parts])
    sla = np.concatenate([p[2] for p in parts])
    u64 = lambda x: np.asarray(x, dtype=np.float64).view(np.uint64)
    assert np.array_equal(u64(outs["f"].cpu().numpy()), u64(f))
    assert np.array_equal(u64(outs["h"].cpu().numpy()), u64(h))
    assert np.array_equal(outs["sla"].cpu().numpy().astype(bool), sla)
    assert best["index"] == select_best(h, sla, begin)
