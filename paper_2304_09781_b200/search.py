"""Optimiser entry points with the reference's signatures.

``anneal`` / ``oracle_search`` / ``blover_search`` / ``sample_neighbor`` /
``realize`` keep the SPEC's argument lists and return types on top of the
reference data model; ``anneal_chains`` is the batched re-plan (many chains,
one launch, optional cross-GPU winner exchange) that the benchmark and the
trace controller drive.  All scoring happens in the CUDA kernels.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .core import ObjectiveParams, SliceType, derive_seed
from .engine import AnnealBatch, CloverEngine, CHAIN_DTYPE, LOG_DTYPE, RECORD_DTYPE
from .errors import CarbonSchedError, InfeasibleGraphError, NoNeighborError
from .graph import ConfigGraph, build_graph
from .mig import FleetConfig
from .objective import AnnealParams, Scenario, strict_eq6_default
from .profiles import ProfileTable
from .sim import Workload  # noqa: F401  (re-exported)

_ENGINES: dict = {}


def default_engine(topology=None) -> CloverEngine:
    """Process-wide engine on the current CUDA device (created lazily)."""
    import torch
    from .mig import DEFAULT_TOPOLOGY
    topo = topology or DEFAULT_TOPOLOGY
    key = (torch.cuda.current_device(), id(topo))
    if key not in _ENGINES:
        _ENGINES[key] = CloverEngine(topo)
    return _ENGINES[key]


@dataclass
class EvalResult:
    """SPEC:405-408."""

    graph: ConfigGraph
    accuracy: float
    energy_wh_per_request: float
    p95_ms: float
    f_value: float
    h_value: float
    sla_met: bool


def _seed_of(rng) -> int:
    if rng is None:
        return 0
    if isinstance(rng, int):
        return rng & ((1 << 63) - 1)
    if hasattr(rng, "seed") and isinstance(getattr(rng, "seed"), int):
        return rng.seed & ((1 << 63) - 1)
    if isinstance(rng, (random.Random, np.random.Generator)) or hasattr(rng, "getrandbits"):
        return int(rng.getrandbits(63)) if hasattr(rng, "getrandbits") else int(rng.integers(0, 1 << 63))
    raise CarbonSchedError("rng must be an int seed or a seeded random source")


def scenario_for(n: int, workload: Workload, ci: float, obj: ObjectiveParams,
                 strict: Optional[bool] = None) -> Scenario:
    return Scenario(int(n), float(workload.arrival_rate_rps), float(ci), obj,
                    strict_eq6_default() if strict is None else bool(strict))


def base_config(n: int, catalog: ProfileTable) -> FleetConfig:
    """BASE: largest variant on every unpartitioned GPU."""
    V = catalog.variant_count
    if not catalog.memory_feasible(V, SliceType.S7G):
        raise CarbonSchedError("largest variant does not fit a 7g slice")
    return FleetConfig([1] * n, [V] * n, catalog.topology)


def co2opt_config(n: int, catalog: ProfileTable) -> FleetConfig:
    """CO2OPT: configuration 19 with the smallest variant everywhere."""
    if not catalog.memory_feasible(1, SliceType.S1G):
        raise CarbonSchedError("smallest variant does not fit a 1g slice")
    topo = catalog.topology
    cid = max(topo.config_ids, key=lambda c: (len(topo.config_slices(c)), c))
    return FleetConfig([cid] * n, [1] * (len(topo.config_slices(cid)) * n), topo)


def realize(g: ConfigGraph, n: int, engine: Optional[CloverEngine] = None) -> FleetConfig:
    """SPEC:206-214 (canonical partition via the device feasibility tables)."""
    return (engine or default_engine()).realize(g, n)


def _result_from_chain(row, graph: ConfigGraph) -> EvalResult:
    return EvalResult(graph, float(row["accuracy"]), float(row["energy_wh"]), float(row["p95_ms"]),
                      float(row["f"]), float(row["h"]), bool(row["sla_met"]))


@dataclass
class ChainsResult:
    best: EvalResult
    best_chain: int
    results: np.ndarray          # CHAIN_DTYPE per chain
    best_w: np.ndarray           # [chains, E]
    final_w: np.ndarray
    evals: int                   # candidates scored by all chains of this rank
    record: np.ndarray = field(default=None)   # winner record (global when exchanged)
    log: Optional[np.ndarray] = None


def exchange_record(engine: CloverEngine, record, group=None):
    """All-gather the 32-byte winner records of all ranks and reduce them in the same
    fixed order everywhere: one tiny collective per round (NCCL over NVLink;
    gloo test runs stage the record through host memory)."""
    import torch.distributed as dist
    from .distributed import gather_records
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return record
    if dist.get_world_size(group) == 1:
        return record
    if dist.get_backend(group) == "nccl":
        gathered = gather_records(record, group)
    else:
        gathered = gather_records(record.cpu(), group).to(record.device)
    return engine.reduce_records(gathered)


def share_winner(record, res, best_w, chain_base: int, group=None):
    """Every rank gets the global winner's chain-result row and best graph: the owning rank
    (the one whose chains [chain_base, chain_base + len(res)) hold record.index) contributes
    them, the others zeros, and one all-reduce (sum) of E + 10 int64 words delivers them."""
    import torch
    import torch.distributed as dist
    E = best_w.shape[1]
    local = int(record["index"]) - chain_base
    words = np.zeros(10 + E, dtype=np.int64)
    if 0 <= local < len(res):
        words[:10] = np.frombuffer(res[local:local + 1].tobytes(), dtype=np.int64)
        words[10:] = best_w[local].astype(np.int64)
    t = torch.from_numpy(words)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    words = t.cpu().numpy()
    row = np.frombuffer(words[:10].tobytes(), dtype=CHAIN_DTYPE)[0]
    return record, row, words[10:].astype(np.uint16)


def exchange_winner(engine: CloverEngine, record, res, best_w, chain_base: int, group=None):
    """Host record of this rank -> global winner record (all-gather + clv_reduce_records) ->
    the winner's result row and graph on every rank (share_winner)."""
    import torch
    import torch.distributed as dist
    raw = torch.from_numpy(np.frombuffer(np.asarray(record, dtype=RECORD_DTYPE).tobytes(), dtype=np.uint8).copy())
    if dist.get_backend(group) == "nccl":
        raw = raw.cuda()
    g = exchange_record(engine, raw.to("cuda:%d" % engine.device) if not raw.is_cuda else raw, group)
    rec = np.frombuffer(g.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)[0].copy()
    return share_winner(rec, res, best_w, chain_base, group)


def _distributed(group, exchange: bool) -> bool:
    """True when the winner record must be exchanged across ranks."""
    if not exchange:
        return False
    import torch.distributed as dist
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return False
    return dist.get_world_size(group) > 1


def anneal_chains(engine: CloverEngine, starts, profile: ProfileTable, scenarios, ap: AnnealParams,
                  seed: int, chain_base: int = 0, cluster: int = 8, log: bool = False, group=None,
                  exchange: bool = True) -> ChainsResult:
    """Batched Clover re-plan: every start graph is an independent chain.

    Host buffers in, host results out: the starts are copied H2D from pinned memory,
    all chains run to termination in one launch, the per-GPU winner is exchanged
    across ranks (if a process group is up) and the results are copied D2H.
    """
    torch = engine.torch
    if isinstance(starts, (list, tuple)) and starts and isinstance(starts[0], ConfigGraph):
        starts = np.array([g.weights for g in starts], dtype=np.uint16)
    starts = np.ascontiguousarray(np.asarray(starts, dtype=np.uint16))
    n_chains, E = starts.shape
    if not log:
        # one native call: H2D, anneal, winner selection, D2H, synchronise (clv_replan); with a
        # process group the 32-byte local record is then exchanged and reduced in fixed order
        # and the winning chain's graph and result row are shared by its owner
        res, best_w, final_w, record = engine.replan(starts, profile, scenarios, ap, seed, chain_base, cluster)
        res, best_w, final_w, record = res.copy(), best_w.copy(), final_w.copy(), record.copy()
        if _distributed(group, exchange):
            record, row, w_best = exchange_winner(engine, record, res, best_w, chain_base, group)
        else:
            local = int(record["index"]) - chain_base
            row, w_best = res[local], best_w[local]
        g = ConfigGraph(np.asarray(w_best, dtype=np.int64), profile.variant_count, profile.name)
        return ChainsResult(_result_from_chain(row, g), int(record["index"]), res, best_w,
                            final_w, int(res["evals"].sum()), record, None)
    # H2D: cached pinned staging buffer -> cached device buffer (one async copy)
    nb_in = starts.nbytes
    h_in = engine.staging("ac_in_host", nb_in, pinned=True)
    h_in.numpy()[:nb_in] = starts.view(np.uint8).reshape(-1)
    d_in = engine.staging("ac_in_dev", nb_in)
    d_in[:nb_in].copy_(h_in[:nb_in], non_blocking=True)
    dev = d_in[:nb_in].view(torch.uint16).view(n_chains, E)
    # outputs: one device buffer [results | best_w | final_w | record], one D2H copy
    r_b = n_chains * CHAIN_DTYPE.itemsize
    w_b = (n_chains * E * 2 + 15) // 16 * 16
    total = r_b + 2 * w_b + 32
    d_out = engine.staging("ac_out_dev", total)
    steps = ap.step_limit()
    batch = AnnealBatch(d_out[:r_b], d_out[r_b:r_b + n_chains * E * 2].view(torch.uint16).view(n_chains, E),
                        d_out[r_b + w_b:r_b + w_b + n_chains * E * 2].view(torch.uint16).view(n_chains, E),
                        torch.zeros(max(1, n_chains * steps * 56), dtype=torch.uint8, device=d_out.device)
                        if log else None, n_chains, chain_base, steps)
    batch = engine.anneal(dev, profile, scenarios, ap, seed, chain_base=chain_base, cluster=cluster, log=log,
                          out=batch)
    rec_dev = d_out[r_b + 2 * w_b:total]
    rec = engine.select_chains(batch, record=rec_dev)
    if exchange:
        rec = exchange_record(engine, rec, group)
        if rec.data_ptr() != rec_dev.data_ptr():
            rec_dev.copy_(rec)
    h_out = engine.staging("ac_out_host", total, pinned=True)
    h_out[:total].copy_(d_out[:total], non_blocking=True)
    log_host = batch.log.cpu() if log else None          # (synchronises; log is a debug output)
    torch.cuda.current_stream(engine.device).synchronize()
    raw = h_out.numpy()[:total].copy()
    res = np.frombuffer(raw[:r_b].tobytes(), dtype=CHAIN_DTYPE)
    best_w = raw[r_b:r_b + n_chains * E * 2].view(np.uint16).reshape(n_chains, E)
    final_w = raw[r_b + w_b:r_b + w_b + n_chains * E * 2].view(np.uint16).reshape(n_chains, E)
    record = np.frombuffer(raw[r_b + 2 * w_b:total].tobytes(), dtype=RECORD_DTYPE)[0]
    log_arr = None
    if log_host is not None:
        log_arr = np.frombuffer(log_host.numpy().tobytes(), dtype=LOG_DTYPE)[:n_chains * steps].reshape(
            n_chains, steps)
    if _distributed(group, exchange):
        _rec, row, w_best = share_winner(record, res, best_w, chain_base, group)
    else:
        local = int(record["index"]) - chain_base
        row, w_best = res[local], best_w[local]
    g = ConfigGraph(np.asarray(w_best, dtype=np.int64), profile.variant_count, profile.name)
    return ChainsResult(_result_from_chain(row, g), int(record["index"]), res, best_w,
                        final_w, int(res["evals"].sum()), record, log_arr)


def anneal(start: ConfigGraph, n: int, profile: ProfileTable, workload: Workload, ci: float,
           obj: ObjectiveParams, ap: Optional[AnnealParams] = None, rng=None,
           engine: Optional[CloverEngine] = None):
    """Clover SA: returns (best EvalResult, log rows, simulated optimisation time).

    Default AnnealParams follow the SPEC literally: one uniformly sampled neighbour
    per iteration, 45 simulated seconds per evaluation against a 300 s budget.
    """
    eng = engine or default_engine(profile.topology)
    ap = ap or AnnealParams(proposal="uniform", evaluate="proposal")
    sc = scenario_for(n, workload, ci, obj)
    res = anneal_chains(eng, [start], profile, sc, ap, _seed_of(rng), log=True, exchange=False)
    row = res.results[0]
    if row["status"] < 0:
        raise InfeasibleGraphError("start graph is not realizable on %d GPUs" % n)
    steps = int(row["steps"])
    log = [dict(zip(res.log.dtype.names, r.tolist())) for r in res.log[0][:steps]] if res.log is not None else []
    n_evals = int(row["evals"]) if ap.evaluate == "proposal" else 1 + steps
    return res.best, log, n_evals * ap.eval_cost_s


def sample_neighbor(g: ConfigGraph, n: int, profile: ProfileTable, rng=None,
                    engine: Optional[CloverEngine] = None) -> ConfigGraph:
    """A uniformly random legal GED<=4 neighbour: one chain step with an
    always-accept temperature, proposal = min-hash neighbour."""
    eng = engine or default_engine(profile.topology)
    V = profile.variant_count
    probe = Scenario(n, 1.0, 0.0, ObjectiveParams(1.0, 1.0, 1.0, 0.5))
    ap = AnnealParams(t_init=1e300, t_floor=1e300, cooling_step=1.0, max_steps=1, stall_limit=1 << 30,
                      proposal="uniform", evaluate="proposal", time_budget_s=math.inf)
    res = anneal_chains(eng, [g], profile, probe, ap, _seed_of(rng), exchange=False)
    row = res.results[0]
    if row["status"] < 0:
        raise InfeasibleGraphError("graph is not realizable on %d GPUs" % n)
    if row["status"] == 2:
        raise NoNeighborError("no legal neighbour")
    return ConfigGraph(res.final_w[0].astype(np.int64), V, profile.name)


def oracle_search(n: int, profile: ProfileTable, workload: Workload, ci: float, obj: ObjectiveParams,
                  engine: Optional[CloverEngine] = None) -> EvalResult:
    """Exhaustive standardized search on the device."""
    eng = engine or default_engine(profile.topology)
    sc = scenario_for(n, workload, ci, obj)
    best = eng.oracle_search(profile, sc)
    cid, assign = eng.oracle_decode(profile, best["index"])
    fc = FleetConfig([cid] * n, list(assign) * n, profile.topology)
    return EvalResult(build_graph(fc, profile), best["accuracy"], best["energy_wh"], best["p95_ms"],
                      best["f"], best["h"], bool(best["sla_met"]))


def blover_search(n: int, profile: ProfileTable, workload: Workload, ci: float, obj: ObjectiveParams,
                  ap: Optional[AnnealParams] = None, rng=None, engine: Optional[CloverEngine] = None):
    """Random search in x-space with anneal's termination rules."""
    eng = engine or default_engine(profile.topology)
    ap = ap or AnnealParams(proposal="uniform", evaluate="proposal")
    sc = scenario_for(n, workload, ci, obj)
    fc, best, log = blover_run(eng, profile, sc, n, ap, _seed_of(rng))
    return EvalResult(build_graph(fc, profile), best["accuracy"], best["energy_wh"], best["p95_ms"],
                      best["f"], best["h"], bool(best["sla_met"])), log


def blover_run(eng: CloverEngine, profile: ProfileTable, sc: Scenario, n: int, ap: AnnealParams, seed: int):
    """BLOVER's draws under anneal's termination rules: at most max_steps + 1
    draws (bounded by the time budget at eval_cost_s each), stop after stall_limit draws
    without a new best.  Returns (winner FleetConfig, its full score, per-draw log); the log's
    length is the evaluation count."""
    budget = ap.max_steps + 1
    if ap.eval_cost_s > 0 and math.isfinite(ap.time_budget_s):
        budget = min(budget, max(1, math.ceil(ap.time_budget_s / ap.eval_cost_s)))
    pods = [(profile, sc, n, 1.0)]
    _best, outs = eng.sweep(pods, 0, budget, seed, outputs=True)
    h = outs["h"].cpu().numpy()
    f = outs["f"].cpu().numpy()
    sla = outs["sla"].cpu().numpy().astype(bool)
    log, bi, stall = [], None, 0
    for i in range(budget):
        better = bi is None or (sla[i] and not sla[bi]) or (sla[i] == sla[bi] and h[i] < h[bi])
        if better:
            bi, stall = i, 0
        else:
            stall += 1
        log.append(dict(iter=i, f=float(f[i]), h=float(h[i]), sla_met=bool(sla[i]), new_best=bool(better)))
        if stall >= ap.stall_limit:
            break
    fc = eng.sweep_decode(pods, seed, bi)[0]
    best, _ = eng.score_fleets([fc], profile, sc)
    return fc, best, log


def random_fleets(engine: CloverEngine, profile: ProfileTable, n: int, seed: int, count: int,
                  first: int = 0) -> list[FleetConfig]:
    """Counter-RNG x-space draws (the BLOVER sampler): config id uniform per GPU,
    memory-feasible variant uniform per slice."""
    probe = Scenario(n, 1.0, 0.0, ObjectiveParams(1.0, 1.0, 1.0, 0.5))
    pods = [(profile, probe, n, 1.0)]
    return [engine.sweep_decode(pods, seed, first + i)[0] for i in range(count)]


def perturbed_fleets(incumbent: FleetConfig, profile: ProfileTable, seed: int, count: int, first: int = 0,
                     keep: float = 0.75) -> list[FleetConfig]:
    """Re-plan start points around a deployed fleet (a re-plan starts from the
    incumbent): fleet i keeps each GPU's partition and variants with probability ``keep``
    and otherwise redraws them as BLOVER does (uniform config id, uniform memory-feasible
    variant per slice).  Draws come from derive_seed(seed, i, gpu, j) (core.py:104-118),
    so the starts are reproducible on any host."""
    topo = profile.topology
    ids = list(topo.config_ids)
    feas = {s: profile.feasible_variants(s) for s in SliceType}
    inc_parts = list(incumbent.partitions)
    inc_assign = list(incumbent.assignments)
    starts = [0]
    for cid in inc_parts:
        starts.append(starts[-1] + len(topo.config_slices(cid)))
    thresh = int(keep * (1 << 20))
    out = []
    for i in range(first, first + count):
        parts, assign = [], []
        for g, cid in enumerate(inc_parts):
            if (derive_seed(seed, i, g, 0) & ((1 << 20) - 1)) < thresh:
                parts.append(cid)
                assign.extend(inc_assign[starts[g]:starts[g + 1]])
                continue
            c = ids[derive_seed(seed, i, g, 1) % len(ids)]
            parts.append(c)
            for j, s in enumerate(topo.config_slices(c)):
                lst = feas[s]
                assign.append(lst[derive_seed(seed, i, g, 2 + j) % len(lst)])
        out.append(FleetConfig(parts, assign, topo))
    return out
