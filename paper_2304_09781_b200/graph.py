"""Configuration graphs x^g (PAPER Definition 1).

A graph is the V x 5 matrix of edge weights w[(v, s)] = number of slices of
kind s that host variant v.  It is stored as a flat tuple in the *device edge
order* ``e = (v - 1) * 5 + s.index`` (s.index = position in SLICE_ORDER), the
same order the kernels use for their uint16 graph encodings and the profile
tables, so host graphs cross the C-ABI without re-indexing.
"""

from __future__ import annotations

from typing import Iterable, Mapping, Optional, Sequence

import numpy as np

from .core import SLICE_ORDER, SliceType, VariantId
from .errors import (CarbonSchedError, IncompatibleGraphsError, InfeasibleAssignmentError)
from .mig import FleetConfig

N_KINDS = len(SLICE_ORDER)


def edge_index(v: VariantId, s: SliceType) -> int:
    return (int(v) - 1) * N_KINDS + SliceType(s).index


def edge_of(e: int) -> tuple[int, SliceType]:
    return e // N_KINDS + 1, SLICE_ORDER[e % N_KINDS]


class ConfigGraph:
    """Immutable weighted bipartite variant->slice graph."""

    __slots__ = ("_w", "_v", "_catalog")

    def __init__(self, weights: Sequence[int], variant_count: int, catalog: Optional[str] = None):
        w = tuple(int(x) for x in weights)
        if variant_count < 1:
            raise CarbonSchedError("a graph needs at least one variant")
        if len(w) != variant_count * N_KINDS:
            raise CarbonSchedError("graph over %d variants needs %d edge weights, got %d"
                                   % (variant_count, variant_count * N_KINDS, len(w)))
        if any(x < 0 for x in w):
            raise CarbonSchedError("edge weights must be non-negative")
        self._w = w
        self._v = int(variant_count)
        self._catalog = catalog

    # -- constructors ----------------------------------------------------
    @classmethod
    def from_edges(cls, edges: Mapping[tuple[int, SliceType], int], variant_count: int,
                   catalog: Optional[str] = None) -> "ConfigGraph":
        w = [0] * (variant_count * N_KINDS)
        for (v, s), weight in edges.items():
            if not 1 <= int(v) <= variant_count:
                raise CarbonSchedError("variant %r outside catalog 1..%d" % (v, variant_count))
            w[edge_index(v, s)] += int(weight)
        return cls(w, variant_count, catalog)

    @classmethod
    def empty(cls, variant_count: int, catalog: Optional[str] = None) -> "ConfigGraph":
        return cls([0] * (variant_count * N_KINDS), variant_count, catalog)

    # -- accessors -------------------------------------------------------
    @property
    def weights(self) -> tuple[int, ...]:
        return self._w

    @property
    def variant_count(self) -> int:
        return self._v

    @property
    def catalog(self) -> Optional[str]:
        return self._catalog

    def weight(self, v: VariantId, s: SliceType) -> int:
        return self._w[edge_index(v, s)]

    def edges(self) -> dict[tuple[int, SliceType], int]:
        return {edge_of(e): x for e, x in enumerate(self._w) if x > 0}

    @property
    def n_instances(self) -> int:
        return sum(self._w)

    def slice_vector(self) -> tuple[int, ...]:
        out = [0] * N_KINDS
        for e, x in enumerate(self._w):
            out[e % N_KINDS] += x
        return tuple(out)

    def to_array(self) -> np.ndarray:
        return np.asarray(self._w, dtype=np.uint16)

    def to_json_dict(self) -> dict:
        """Debug dump with stable field order."""
        return {"edges": [{"variant": v, "slice": s.label, "weight": x}
                          for (v, s), x in sorted(self.edges().items(),
                                                  key=lambda kv: edge_index(*kv[0]))]}

    def _check(self, other: "ConfigGraph") -> None:
        if self._v != other._v or (self._catalog and other._catalog
                                   and self._catalog != other._catalog):
            raise IncompatibleGraphsError("graphs over different variant catalogs")

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, ConfigGraph):
            return NotImplemented
        return self._v == other._v and self._w == other._w

    def __hash__(self) -> int:
        return hash((self._v, self._w))

    def __repr__(self) -> str:
        body = ", ".join("(v%d,%s):%d" % (v, s.label, x) for (v, s), x in self.edges().items())
        return "ConfigGraph({%s})" % body


def build_graph(fc: FleetConfig, profile=None, variant_count: Optional[int] = None) -> ConfigGraph:
    """x^g from (x^p, x^v); memory check per SPEC:169 when a profile is given."""
    if profile is not None:
        V = profile.variant_count
        catalog = profile.name
    else:
        V = variant_count if variant_count is not None else max(fc.assignments)
        catalog = None
    w = [0] * (V * N_KINDS)
    for _g, s, v in fc.instances():
        if v > V:
            raise InfeasibleAssignmentError("variant %d outside catalog 1..%d" % (v, V))
        if profile is not None and not profile.memory_feasible(v, s):
            raise InfeasibleAssignmentError("variant %d does not fit a %s slice" % (v, s.label))
        w[edge_index(v, s)] += 1
    return ConfigGraph(w, V, catalog)


def ged(a: ConfigGraph, b: ConfigGraph) -> int:
    """L1 graph edit distance over edge weights."""
    a._check(b)
    return sum(abs(x - y) for x, y in zip(a.weights, b.weights))


def merge(a: ConfigGraph, b: ConfigGraph) -> ConfigGraph:
    """Edge-wise sum."""
    a._check(b)
    return ConfigGraph([x + y for x, y in zip(a.weights, b.weights)], a.variant_count,
                       a.catalog or b.catalog)


def scale(g: ConfigGraph, k: int) -> ConfigGraph:
    """k-fold merge of g with itself (the standardized ORACLE graph is n * g_1)."""
    return ConfigGraph([x * int(k) for x in g.weights], g.variant_count, g.catalog)


def graphs_to_array(graphs: Iterable[ConfigGraph]) -> np.ndarray:
    return np.asarray([g.weights for g in graphs], dtype=np.uint16)
