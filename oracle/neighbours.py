"""ORACLE -- TEST INFRASTRUCTURE ONLY.  GED<=4 neighbourhoods.

Definition-level enumeration: every pair of removal multiset R and addition
multiset A with |R| = |A| in {1, 2}, R and A disjoint, R available in g, A
memory-feasible; for |R| = 2 a perfect matching R->A whose pairs share a variant
or a slice (two elementary moves: variant swap / slice move); any single
(v,s)->(v',s') (one elementary move, or the swap+slice composition (c));
the resulting slice multiset realizable on n GPUs.  Canonical index:
  single  (r, a)               -> r * E + a
  double  ({r1<=r2}, {a1<=a2}) -> E*E + P(r1, r2) * NP + P(a1, a2)
with P the row-major index of a sorted pair and NP = E(E+1)/2.  The device
enumerates the same set by a different (adjacency-driven) route.

moves="paper" (every configuration within the GED threshold) adds
the unit instance moves that change the instance count m:
  add one instance on edge a    -> E*E + NP*NP + a        (GED 1; a memory-feasible)
  remove one instance of edge r -> E*E + NP*NP + E + r    (GED 1; r present)
each kept when the new slice multiset is realizable on n GPUs.
"""

from __future__ import annotations

import itertools

import numpy as np


def pair_index(x, y, E):
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    return x * E - (x * (x - 1)) // 2 + (y - x)


def adjacency(V: int) -> np.ndarray:
    E = V * 5
    e = np.arange(E)
    same_v = (e[:, None] // 5) == (e[None, :] // 5)
    same_s = (e[:, None] % 5) == (e[None, :] % 5)
    return (same_v | same_s) & (e[:, None] != e[None, :])


class Neighbourhood:
    __slots__ = ("idx", "W", "r1", "r2", "a1", "a2", "kind", "ged")

    def __init__(self, idx, W, r1, r2, a1, a2, kind, ged=None):
        self.idx, self.W, self.r1, self.r2, self.a1, self.a2, self.kind = idx, W, r1, r2, a1, a2, kind
        self.ged = 2 * np.asarray(kind, dtype=np.int64) if ged is None else ged

    def __len__(self):
        return len(self.idx)


def enumerate_neighbours(w, mem_ok, V: int, n: int, feas, moves: str = "spec") -> Neighbourhood:
    w = np.asarray(w, dtype=np.int64)
    E = V * 5
    NP = E * (E + 1) // 2
    adj = adjacency(V)
    present = np.nonzero(w > 0)[0]
    okA = np.nonzero(np.asarray(mem_ok, dtype=bool))[0]
    # singles
    r = np.repeat(present, len(okA))
    a = np.tile(okA, len(present))
    keep = r != a
    r, a = r[keep], a[keep]
    s_idx = r * E + a
    # doubles
    rp = [(i, j) for ii, i in enumerate(present) for j in present[ii:] if i != j or w[i] >= 2]
    ap = [(i, j) for ii, i in enumerate(okA) for j in okA[ii:]]
    if rp and ap:
        R = np.array(rp, dtype=np.int64)
        A = np.array(ap, dtype=np.int64)
        r1 = np.repeat(R[:, 0], len(A)); r2 = np.repeat(R[:, 1], len(A))
        a1 = np.tile(A[:, 0], len(R)); a2 = np.tile(A[:, 1], len(R))
        disjoint = (a1 != r1) & (a1 != r2) & (a2 != r1) & (a2 != r2)
        match = (adj[r1, a1] & adj[r2, a2]) | (adj[r1, a2] & adj[r2, a1])
        k2 = disjoint & match
        r1, r2, a1, a2 = r1[k2], r2[k2], a1[k2], a2[k2]
        d_idx = E * E + pair_index(r1, r2, E) * NP + pair_index(a1, a2, E)
    else:
        r1 = r2 = a1 = a2 = d_idx = np.zeros(0, dtype=np.int64)
    n1, n2 = len(r), len(r1)
    if moves == "paper":                         # unit add / remove (GED 1)
        u_add, u_rem = okA, present
    else:
        u_add = u_rem = np.zeros(0, dtype=np.int64)
    n3, n4 = len(u_add), len(u_rem)
    Wn = np.repeat(w[None, :], n1 + n2 + n3 + n4, axis=0)
    rows1 = np.arange(n1)
    np.subtract.at(Wn, (rows1, r), 1)
    np.add.at(Wn, (rows1, a), 1)
    rows2 = n1 + np.arange(n2)
    for col, sign in ((r1, -1), (r2, -1), (a1, 1), (a2, 1)):
        np.add.at(Wn, (rows2, col), sign)
    base = E * E + NP * NP
    np.add.at(Wn, (n1 + n2 + np.arange(n3), u_add), 1)
    np.add.at(Wn, (n1 + n2 + n3 + np.arange(n4), u_rem), -1)
    # fleet feasibility of the new slice multisets
    svec = Wn.reshape(len(Wn), V, 5).sum(axis=1)
    feas_ok = np.zeros(len(Wn), dtype=bool)
    if len(Wn):
        uniq, inv = np.unique(svec, axis=0, return_inverse=True)
        okv = feas.feasible_batch(uniq, n)
        feas_ok = okv[inv.reshape(-1)]
    none3, none4 = np.full(n3, -1), np.full(n4, -1)
    idx = np.concatenate([s_idx, d_idx, base + u_add, base + E + u_rem])
    R1 = np.concatenate([r, r1, none3, u_rem]); R2 = np.concatenate([np.full(n1, -1), r2, none3, none4])
    A1 = np.concatenate([a, a1, u_add, none4]); A2 = np.concatenate([np.full(n1, -1), a2, none3, none4])
    kind = np.concatenate([np.ones(n1, dtype=np.int8), np.full(n2, 2, dtype=np.int8), np.zeros(n3 + n4, dtype=np.int8)])
    ged = np.concatenate([np.full(n1, 2), np.full(n2, 4), np.ones(n3 + n4, dtype=np.int64)]).astype(np.int64)
    sel = np.nonzero(feas_ok)[0]
    order = sel[np.argsort(idx[sel], kind="stable")]
    return Neighbourhood(idx[order], Wn[order], R1[order], R2[order], A1[order], A2[order], kind[order], ged[order])


def brute_force_neighbours(w, mem_ok, V: int, n: int, feas) -> set:
    """All graphs reachable by one or two elementary moves (swap / slice move).

    Small graphs only; pins enumerate_neighbours' canonical definition.
    """
    w = tuple(int(x) for x in w)
    E = V * 5

    def moves(g):
        for e in range(E):
            if g[e] <= 0:
                continue
            v, s = divmod(e, 5)
            targets = [vv * 5 + s for vv in range(V) if vv != v] + [v * 5 + ss for ss in range(5) if ss != s]
            for t in targets:
                h = list(g); h[e] -= 1; h[t] += 1
                yield tuple(h)

    out = set()
    for g1 in moves(w):
        out.add(g1)
        for g2 in moves(g1):
            out.add(g2)
    res = set()
    for g in out:
        if g == w:
            continue
        if any(g[e] > 0 and not mem_ok[e] for e in range(E)):
            continue
        svec = [sum(g[v * 5 + s] for v in range(V)) for s in range(5)]
        if feas.feasible(svec, n):
            res.add(g)
    return res
