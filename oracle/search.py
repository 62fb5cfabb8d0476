"""ORACLE -- TEST INFRASTRUCTURE ONLY.  ORACLE / BLOVER schemes and x-space decode.

* exhaustive standardized search: ascending config id, then the
  lexicographic product of memory-feasible variants per slice (largest slice
  first, mig.py:240-242), candidate = FleetConfig([cid]*n, assignment*n).
  Winner: SLA-meeting max f (lowest index on ties), else min p95 (lowest index).
* counter-RNG x-space candidates:
  candidate i draws from Stream(derive_seed(seed, i)); per pod, per GPU a config
  id uniform over the table, then per slice a variant uniform over the
  memory-feasible variants of that slice kind.
* FleetConfig -> graph decode (mig.py:286-299 + SPEC:165-173).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .evaluator import evaluate, epilogue, aggregates
from .rng import Stream, derive_seed

KINDS = (7, 4, 3, 2, 1)
KIND_INDEX = {7: 0, 4: 1, 3: 2, 2: 3, 1: 4}


def row_kinds(topology, cid):
    """Slice-kind indices (0..4) of a config id, largest first."""
    return [KIND_INDEX[int(s)] for s in topology.config_slices(cid)]


def feasible_lists(tables):
    return [[v for v in range(1, tables.V + 1) if tables.mem_ok[(v - 1) * 5 + s]] for s in range(5)]


def oracle_space(topology, tables):
    """[(cid, kinds, radices, count, offset)] in enumeration order."""
    fl = feasible_lists(tables)
    out, off = [], 0
    for cid in topology.config_ids:
        kinds = row_kinds(topology, cid)
        radices = [len(fl[k]) for k in kinds]
        count = int(np.prod(radices)) if all(radices) else 0
        out.append((cid, kinds, radices, count, off))
        off += count
    return out, off


def oracle_decode(index, topology, tables):
    fl = feasible_lists(tables)
    space, total = oracle_space(topology, tables)
    for cid, kinds, radices, count, off in space:
        if index < off + count:
            rem = index - off
            digits = []
            for r in reversed(radices):
                digits.append(rem % r)
                rem //= r
            digits.reverse()
            return cid, tuple(fl[k][d] for k, d in zip(kinds, digits))
    raise IndexError(index)


def oracle_graphs(topology, tables, n):
    """All standardized candidates as a (count, E) int64 weight matrix, in index order."""
    fl = feasible_lists(tables)
    space, total = oracle_space(topology, tables)
    W = np.zeros((total, tables.E), dtype=np.int64)
    for cid, kinds, radices, count, off in space:
        if count == 0:
            continue
        grids = np.array(list(itertools.product(*[range(r) for r in radices])), dtype=np.int64)
        for j, k in enumerate(kinds):
            v = np.array(fl[k])[grids[:, j]]
            np.add.at(W, (off + np.arange(count), (v - 1) * 5 + k), n)
    return W


def select_oracle(ev):
    """(SLA desc, f desc, idx asc) else (p95 asc, idx asc) -- SPEC:539, 548."""
    ok = np.nonzero(ev.sla)[0]
    if len(ok):
        return int(ok[np.lexsort((ok, -ev.f[ok]))[0]]), True
    return int(np.lexsort((np.arange(len(ev.L)), ev.L))[0]), False


def oracle_search(topology, tables, scenario, n):
    W = oracle_graphs(topology, tables, n)
    ev = evaluate(W, tables, scenario)
    i, met = select_oracle(ev)
    return i, ev, W


# -- x-space decode ------------------------------------------------------------

def fleet_graph(partitions, assignments, topology, tables):
    w = np.zeros(tables.E, dtype=np.int64)
    pos = 0
    for cid in partitions:
        for k in row_kinds(topology, cid):
            v = assignments[pos]
            pos += 1
            if not 1 <= v <= tables.V or not tables.mem_ok[(v - 1) * 5 + k]:
                raise ValueError("infeasible assignment")
            w[(v - 1) * 5 + k] += 1
    if pos != len(assignments):
        raise ValueError("assignment length mismatch")
    return w


def fleet_row_error(partitions, assignments, topology, tables):
    """First error of one FleetConfig row, in the reference's order, or None.

    FleetConfig.__init__ (reference mig.py:248-263): ``expected`` is summed over every
    partition id (``config_slices`` raises InvalidConfigError for an unknown id, mig.py:
    129-135), then the length is compared (CarbonSchedError), then ``any(v < 1)``
    (CarbonSchedError).  Evaluation then rejects a variant above V or a
    variant that does not fit its slice (InfeasibleAssignmentError).
    Returns "invalid_config" | "length" | "variant_lt1" | "infeasible" | None.
    """
    known = set(int(c) for c in topology.config_ids)
    if any(int(c) not in known for c in partitions):
        return "invalid_config"
    kinds = [k for cid in partitions for k in row_kinds(topology, int(cid))]
    if len(kinds) != len(assignments):
        return "length"
    if any(int(v) < 1 for v in assignments):
        return "variant_lt1"
    for k, v in zip(kinds, assignments):
        if int(v) > tables.V or not tables.mem_ok[(int(v) - 1) * 5 + k]:
            return "infeasible"
    return None


# -- counter-RNG sweep -----------------------------------------------------------

@dataclass
class Pod:
    tables: object
    scenario: object
    n_gpus: int
    weight: float


def draw_candidate(seed, index, pods, topology):
    """Per pod: (partitions, assignments) drawn from the candidate's stream."""
    st = Stream(derive_seed(seed, index))
    ids = topology.config_ids
    out = []
    for pod in pods:
        fl = feasible_lists(pod.tables)
        parts, assign = [], []
        for _g in range(pod.n_gpus):
            cid = ids[st.bounded(len(ids))]
            parts.append(cid)
            for k in row_kinds(topology, cid):
                lst = fl[k]
                assign.append(lst[st.bounded(len(lst))])
        out.append((parts, assign))
    return out


def sweep_evaluate(seed, begin, end, pods, topology):
    """f, h, sla of candidates [begin, end) combined over pods (weights w_p)."""
    per_pod = [[] for _ in pods]
    for i in range(begin, end):
        for p, (parts, assign) in enumerate(draw_candidate(seed, i, pods, topology)):
            per_pod[p].append(fleet_graph(parts, assign, topology, pods[p].tables))
    f = h = None
    sla = None
    for p, pod in enumerate(pods):
        ev = evaluate(np.array(per_pod[p]), pod.tables, pod.scenario)
        if f is None:
            f, h, sla = pod.weight * ev.f, pod.weight * ev.h, ev.sla.copy()
        else:
            f, h, sla = f + pod.weight * ev.f, h + pod.weight * ev.h, sla & ev.sla
    return f, h, sla


def select_best(h, sla, base_index=0):
    """(SLA desc, h asc, idx asc) -- best tracking of SPEC:464, 482-483."""
    i = int(np.lexsort((np.arange(len(h)), h, ~sla))[0])
    return base_index + i
