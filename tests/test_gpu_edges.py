"""GPU edge cases: empty and ragged inputs, both score_graphs paths (TMA ring for 16-B
aligned inputs, plain loads otherwise), partial tiles, the largest device catalog
(V = 8), invalid chain starts and empty simulator batches -- all against the oracle."""

import numpy as np
import pytest
import torch

from oracle.evaluator import calibrate, evaluate
from oracle.feasibility import FeasOracle
from oracle.search import select_best
from oracle.tables import OracleTables
from paper_2304_09781_b200.core import SliceType
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import ProfileTable, ServiceRow, VariantSpec, synthetic_profile
from tests.helpers import perturbed_graphs, random_fleet_graphs

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


def profile_v8():
    """Eight variants: the largest catalog the device tables hold (E = 40 edges)."""
    vs = [VariantSpec(v, 0.60 + 0.03 * v, 0.5 + 1.5 * v) for v in range(1, 9)]
    service = {}
    for v in range(1, 9):
        for s in SliceType:
            mean = (4.0 + 6.0 * v) * (7.0 / s.compute_units) ** 0.8
            service[(v, s)] = ServiceRow(mean, "deterministic", 0.0, 1e-6 * v * mean * s.compute_units)
    return ProfileTable("v8", vs, service, {s: 9.0 * s.compute_units for s in SliceType})


def check_scores(engine, prof, W, n, W_dev=None):
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, n, 320.0, 0.5)
    best, outs = engine.score_graphs(W if W_dev is None else W_dev, prof, sc)
    if len(W) == 0:
        assert best["valid_count"] == 0
        return best
    ev = evaluate(W, T, sc)
    vecs = W.reshape(len(W), T.V, 5).sum(axis=1)
    mem_bad = ((W > 0) & ~T.mem_ok[None, :]).any(axis=1)
    feas = FeasOracle(DEFAULT_TOPOLOGY, n).feasible_batch(vecs, n) & ~mem_bad
    assert np.array_equal(outs["feasible"].cpu().numpy().astype(bool), feas)
    for key, arr in (("f", ev.f), ("h", ev.h), ("p95", ev.L)):
        assert bits_equal(outs[key].cpu().numpy()[feas], arr[feas]), key
    if feas.any():
        exp_i = select_best(np.where(feas, ev.h, np.inf), ev.sla & feas)
        assert best["index"] == exp_i
    assert best["valid_count"] == int(feas.sum())
    return best


@pytest.mark.parametrize("count", [1, 511, 512, 513, 1537])
def test_score_graphs_partial_tiles(engine, count):
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    base = random_fleet_graphs(T, 8, max(count, 2), seed=count)[:count]
    check_scores(engine, prof, base, 8)


def test_score_graphs_unaligned_input_takes_fallback_path(engine):
    prof = synthetic_profile("resnet")
    T = OracleTables.from_profile(prof)
    base = random_fleet_graphs(T, 16, 800, seed=3)
    W = np.concatenate([base, perturbed_graphs(base, 800, seed=4)])
    padded = torch.from_numpy(np.concatenate([np.zeros((1, W.shape[1]), np.int64), W]).astype(np.int16)).cuda()
    W_dev = padded.view(torch.uint16)[1:]                    # 50 B offset: not 16-B aligned
    assert W_dev.data_ptr() % 16 != 0
    check_scores(engine, prof, W, 16, W_dev=W_dev)


def test_score_graphs_empty_batch(engine):
    prof = synthetic_profile("tiny3")
    W = np.zeros((0, 15), dtype=np.int64)
    best = check_scores(engine, prof, W, 2)
    assert not best["found"] and best["valid_count"] == 0


def test_largest_catalog_v8(engine):
    prof = profile_v8()
    T = OracleTables.from_profile(prof)
    base = random_fleet_graphs(T, 12, 2000, seed=8)
    W = np.concatenate([base, perturbed_graphs(base, 2000, seed=9)])
    check_scores(engine, prof, W, 12)


def test_anneal_empty_and_invalid_starts(engine, feas64):
    from oracle.anneal import anneal_chain
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, 8, 400.0, 0.5)
    ap = AnnealParams(max_steps=10)
    good = random_fleet_graphs(T, 8, 3, seed=1)
    bad = np.zeros_like(good[0])
    bad[(T.V - 1) * 5] = 9                               # nine 7g instances cannot fit 8 GPUs
    zero = np.zeros_like(good[0])
    starts = np.stack([good[0], bad, zero, good[1]])
    out = engine.anneal(starts, prof, sc, ap, 5).host()
    st = out["results"]["status"]
    assert st[1] == -1 and st[2] == -1 and st[0] >= 0 and st[3] >= 0
    for c in (0, 3):
        ref = anneal_chain(starts[c], 8, T, sc, ap, 5, c, feas64)
        assert (int(out["results"][c]["evals"]), int(out["results"][c]["steps"])) == (ref.evals, ref.steps)
        assert np.array_equal(out["best_w"][c].astype(np.int64), ref.best_w)
    assert np.array_equal(out["best_w"][1], starts[1]) and np.array_equal(out["final_w"][2], starts[2])


def test_simulate_empty_batch(engine):
    from paper_2304_09781_b200 import sim as S
    prof = synthetic_profile("tiny3")
    reps, vc, ic, nreq = engine.simulate(np.zeros(0, np.uint8), np.zeros(1, np.int64), prof,
                                         S.Workload(100.0, 10.0, 1))
    assert len(reps) == 0 and nreq > 0
    assert S.simulate_fleets([], prof, S.Workload(100.0, 10.0, 1), engine=engine) == []


def test_score_x_error_paths(engine):
    from paper_2304_09781_b200.errors import CarbonSchedError, InfeasibleAssignmentError, InvalidConfigError
    from paper_2304_09781_b200.mig import FleetConfig
    prof = synthetic_profile("bert")                         # variant 6 (11 GB) does not fit 1g / 2g
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, 2, 300.0, 0.5)
    good = [FleetConfig([1, 19], [3] + [1] * 7), FleetConfig([5, 9], [2] * (len(DEFAULT_TOPOLOGY.config_slices(5))
                                                                        + len(DEFAULT_TOPOLOGY.config_slices(9))))]

    def csr(fleets, patch=None):
        xp = np.array([f.partitions for f in fleets], dtype=np.uint8)
        xvs = [np.array(f.assignments, dtype=np.uint8) for f in fleets]
        if patch:
            patch(xp, xvs)
        off = np.concatenate([[0], np.cumsum([len(x) for x in xvs])]).astype(np.int64)
        return xp, np.concatenate(xvs), off

    best, _ = engine.score_x(*csr(good), 2, prof, sc)
    assert best["valid_count"] == 2
    with pytest.raises(InvalidConfigError):
        engine.score_x(*csr(good, lambda xp, xv: xp.__setitem__((1, 0), 200)), 2, prof, sc)
    with pytest.raises(CarbonSchedError):
        engine.score_x(*csr(good, lambda xp, xv: xv.__setitem__(0, xv[0][:-1])), 2, prof, sc)
    with pytest.raises(InfeasibleAssignmentError):
        engine.score_x(*csr(good, lambda xp, xv: xv[0].__setitem__(1, 6)), 2, prof, sc)
