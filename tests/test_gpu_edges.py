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


def _score_rows(engine, prof, sc, rows, n):
    xp = np.array([p for p, a in rows], dtype=np.uint8).reshape(len(rows), n)
    xv = np.array([v for p, a in rows for v in a], dtype=np.uint8)
    off = np.concatenate([[0], np.cumsum([len(a) for p, a in rows])]).astype(np.int64)
    return engine.score_x(xp, xv, off, n, prof, sc)


def test_score_x_error_precedence(engine):
    """The reference's multi-defect rows (golden, FleetConfig.__init__ order), one at a time
    and as batches: the reported row is the lowest failing index, its error the first in
    the reference's order (unknown id, length, variant < 1), then the SPEC's infeasible
    assignment."""
    import json
    import os
    from oracle.search import fleet_row_error
    from paper_2304_09781_b200 import errors as E
    G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_l0.json")))
    prof = synthetic_profile("bert")
    T = OracleTables.from_profile(prof)
    EXC = {"invalid_config": E.InvalidConfigError, "length": E.CarbonSchedError,
           "variant_lt1": E.CarbonSchedError, "infeasible": E.InfeasibleAssignmentError}
    sc = {n: calibrate(prof, T, n, 300.0, 0.5) for n in range(1, 7)}
    rows = [(p, a) for p, a, _ in G["fleet_error_precedence"]]
    kinds = set()
    for p, a in rows:
        want = fleet_row_error(p, a, DEFAULT_TOPOLOGY, T)
        kinds.add(want)
        if want is None:
            best, _ = _score_rows(engine, prof, sc[len(p)], [(p, a)], len(p))
            assert best["valid_count"] == 1
        else:
            with pytest.raises(E.CarbonSchedError) as ei:
                _score_rows(engine, prof, sc[len(p)], [(p, a)], len(p))
            assert type(ei.value) is EXC[want], (p, a, want)
            assert "candidate 0:" in str(ei.value)
    assert kinds == {None, "invalid_config", "length", "variant_lt1", "infeasible"}
    for n in range(1, 7):
        batch = [r for r in rows if len(r[0]) == n]
        errs = [fleet_row_error(p, a, DEFAULT_TOPOLOGY, T) for p, a in batch]
        bad = [i for i, e in enumerate(errs) if e]
        if not bad:
            continue
        with pytest.raises(E.CarbonSchedError) as ei:
            _score_rows(engine, prof, sc[n], batch, n)
        assert type(ei.value) is EXC[errs[bad[0]]]
        assert "candidate %d:" % bad[0] in str(ei.value)


def test_score_x_lowest_failing_index_large(engine):
    """64-GPU rows, errors planted in many tiles: the lowest failing index wins."""
    from oracle.search import draw_candidate, Pod
    from paper_2304_09781_b200 import errors as E
    prof = synthetic_profile("bert")
    T = OracleTables.from_profile(prof)
    n = 64
    sc = calibrate(prof, T, n, 300.0, 0.5)
    rows = [tuple(map(list, draw_candidate(5, i, [Pod(T, sc, n, 1.0)], DEFAULT_TOPOLOGY)[0])) for i in range(3000)]
    best, _ = _score_rows(engine, prof, sc, rows, n)
    assert best["valid_count"] == 3000
    bad = [list(r) for r in rows]
    bad[2900][0][5] = 42                                    # unknown id
    bad[1777][1] = bad[1777][1][:-1]                        # length
    bad[2222][1][3] = 0                                     # variant < 1
    with pytest.raises(E.CarbonSchedError) as ei:
        _score_rows(engine, prof, sc, [tuple(r) for r in bad], n)
    assert type(ei.value) is E.CarbonSchedError and "candidate 1777:" in str(ei.value)
    bad[1200][1][0] = 9                                     # variant > V
    with pytest.raises(E.InfeasibleAssignmentError, match="candidate 1200:"):
        _score_rows(engine, prof, sc, [tuple(r) for r in bad], n)


@pytest.mark.parametrize("shape", ["wide_rows", "many_gpus", "huge_rows"])
def test_score_x_unstaged_paths(engine, shape):
    """Tiles whose x^v span overflows the shared-memory stage (64 GPUs of 7 x 1g slices),
    fleets too wide for the x^p stage (n = 320) and rows past the 16-bit slot counters
    (n = 9,500, > 65,535 slots) take the direct-load / direct-sum walks: same bits."""
    from oracle.search import fleet_graph, row_kinds
    from paper_2304_09781_b200.mig import FleetConfig
    prof = synthetic_profile("efficientnet")
    T = OracleTables.from_profile(prof)
    rng = np.random.default_rng(11)
    ids = list(DEFAULT_TOPOLOGY.config_ids)
    one_g = max(ids, key=lambda c: len(DEFAULT_TOPOLOGY.config_slices(c)))
    n = {"wide_rows": 64, "many_gpus": 320, "huge_rows": 9500}[shape]
    fleets = []
    for i in range(700 if shape != "huge_rows" else 6):
        if shape != "many_gpus":
            parts = [one_g if rng.random() < 0.9 else int(rng.choice(ids)) for _ in range(n)]
        else:
            parts = [int(rng.choice(ids)) for _ in range(n)]
        m = sum(len(DEFAULT_TOPOLOGY.config_slices(c)) for c in parts)
        fe = [[v for v in range(1, T.V + 1) if T.mem_ok[(v - 1) * 5 + k]] for k in range(5)]
        kinds = [k for c in parts for k in row_kinds(DEFAULT_TOPOLOGY, c)]
        assign = [int(rng.choice(fe[k])) for k in kinds]
        assert len(assign) == m
        fleets.append(FleetConfig(parts, assign))
    sc = calibrate(prof, T, n, 300.0, 0.5)
    best, outs = engine.score_fleets(fleets, prof, sc)
    W = np.array([fleet_graph(f.partitions, f.assignments, DEFAULT_TOPOLOGY, T) for f in fleets])
    ev = evaluate(W, T, sc)
    assert bits_equal(outs["f"].cpu().numpy(), ev.f)
    assert bits_equal(outs["h"].cpu().numpy(), ev.h)
    assert best["index"] == select_best(ev.h, ev.sla)
