"""Host-side mirrors of the reference's graph and result types.

Same names, fields and semantics as ``locmax.graph`` / ``locmax.matchers``
(``/root/reference/pkg/src/locmax/graph.py:20-237``,
``matchers.py:21-58``) so code written against the reference runs unchanged:

* :class:`Graph` -- the immutable edge-array graph.  ``offsets`` /
  ``slot_vertex`` / ``slot_edge`` (graph.py:108-115) are derived lazily: the
  device engine rebuilds its own slot layout from the edge arrays, and at
  RMAT scale the host CSR would cost seconds nobody asked for.
* :class:`Matching` -- ``edges`` (frozenset of edge ids) and ``mate``;
  equality compares both (graph.py:176-179).  The frozenset is built lazily
  from the sorted id array the engine returns (building it for millions of
  ids costs seconds, SURVEY.md §7 hard part 6).
* :class:`RoundStats`, :class:`PhaseTrace` -- per-round trace
  (matchers.py:21-58) plus ``device_millis`` (CUDA-event time of the round
  loop).

When ``locmax`` is importable these ARE the reference's types: ``RoundStats``
is ``locmax.matchers.RoundStats``, ``PhaseTrace`` and ``Matching`` subclass
``locmax.matchers.PhaseTrace`` / ``locmax.graph.Matching``, so
``trace.rounds == ref_trace.rounds`` and ``isinstance`` checks hold.
* :func:`matching_from_edge_ids`, :func:`validate_matching` -- graph.py:195-237.

Any object exposing ``num_vertices``, ``edge_u``, ``edge_v`` and
``edge_weight`` (a ``locmax.Graph`` included) is accepted by the engine.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, NamedTuple

import numpy as np

# When the reference package is importable, results are returned in ITS types
# (RoundStats, a PhaseTrace subclass, a Matching subclass), so code written
# against locmax compares them with ``==`` and ``isinstance`` unchanged.
try:
    from locmax.graph import Matching as _RefMatching
    from locmax.matchers import PhaseTrace as _RefPhaseTrace
    from locmax.matchers import RoundStats as _RefRoundStats
except Exception:   # locmax absent: this module's own mirrors
    _RefMatching = _RefPhaseTrace = _RefRoundStats = None

REFERENCE_TYPES = _RefRoundStats is not None


class Graph:
    """Undirected simple graph with nonnegative real edge weights (graph.py:20-56)."""

    __slots__ = ("num_vertices", "edge_u", "edge_v", "edge_weight", "_csr")

    def __init__(self, num_vertices: int, edge_u, edge_v, edge_weight,
                 offsets=None, slot_vertex=None, slot_edge=None):
        self.num_vertices = int(num_vertices)
        self.edge_u = _frozen(np.asarray(edge_u, dtype=np.int64))
        self.edge_v = _frozen(np.asarray(edge_v, dtype=np.int64))
        self.edge_weight = _frozen(np.asarray(edge_weight, dtype=np.float64))
        if not (self.edge_u.shape == self.edge_v.shape == self.edge_weight.shape):
            raise ValueError("edge arrays must have equal length")
        self._csr = None
        if offsets is not None:
            self._csr = (_frozen(np.asarray(offsets, dtype=np.int64)),
                         _frozen(np.asarray(slot_vertex, dtype=np.int64)),
                         _frozen(np.asarray(slot_edge, dtype=np.int64)))

    @classmethod
    def from_reference(cls, g) -> "Graph":
        """Wrap any reference-shaped graph (e.g. ``locmax.Graph``) without copying."""
        return cls(g.num_vertices, g.edge_u, g.edge_v, g.edge_weight)

    # -- graph.py:108-115, lazily
    def _layout(self):
        if self._csr is None:
            m = self.edge_u.size
            n = self.num_vertices
            slot_vertex = np.concatenate([self.edge_u, self.edge_v]) if m else np.empty(0, np.int64)
            slot_eid = np.concatenate([np.arange(m), np.arange(m)]).astype(np.int64)
            order = np.lexsort((slot_eid, slot_vertex))
            slot_vertex = slot_vertex[order]
            slot_eid = slot_eid[order]
            degrees = np.bincount(slot_vertex, minlength=n).astype(np.int64)
            offsets = np.concatenate([[0], np.cumsum(degrees)]).astype(np.int64)
            self._csr = (_frozen(offsets), _frozen(slot_vertex), _frozen(slot_eid))
        return self._csr

    @property
    def offsets(self) -> np.ndarray:
        return self._layout()[0]

    @property
    def slot_vertex(self) -> np.ndarray:
        return self._layout()[1]

    @property
    def slot_edge(self) -> np.ndarray:
        return self._layout()[2]

    @property
    def num_edges(self) -> int:
        return int(self.edge_u.size)

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def incident_edges(self, v: int) -> np.ndarray:
        return self.slot_edge[self.offsets[v]:self.offsets[v + 1]]

    def endpoints(self, edge_id: int) -> tuple[int, int]:
        return int(self.edge_u[edge_id]), int(self.edge_v[edge_id])

    def other_endpoint(self, edge_id: int, v: int) -> int:
        u = int(self.edge_u[edge_id])
        return int(self.edge_v[edge_id]) if u == v else u

    def total_weight(self, edge_ids: Iterable[int]) -> float:
        """graph.py:54-56: sum over the ascending ids (bit-identical to the reference)."""
        if isinstance(edge_ids, np.ndarray):
            ids = np.sort(edge_ids.astype(np.int64))
        else:
            ids = np.fromiter(sorted(int(k) for k in edge_ids), dtype=np.int64)
        return float(self.edge_weight[ids].sum()) if ids.size else 0.0


def _frozen(a: np.ndarray) -> np.ndarray:
    if a.flags.writeable:
        try:
            a.setflags(write=False)
        except ValueError:
            a = a.copy()
            a.setflags(write=False)
    return a


class Matching(_RefMatching if _RefMatching is not None else object):
    """Matched edge ids plus the induced mate table (graph.py:166-192).

    A subclass of ``locmax.Matching`` when the reference is importable.  The
    frozenset ``edges`` is built lazily from the sorted id array the engine
    returns (building it for millions of ids costs seconds)."""

    def __init__(self, edge_ids, mate: np.ndarray):
        if isinstance(edge_ids, (frozenset, set)):
            edges = frozenset(edge_ids)
            ids = np.fromiter(sorted(edges), dtype=np.int64, count=len(edges))
        else:
            ids = np.sort(np.asarray(edge_ids, dtype=np.int64))
            edges = None
        ids.setflags(write=False)
        object.__setattr__(self, "_ids", ids)
        object.__setattr__(self, "_edges", edges)
        object.__setattr__(self, "mate", _frozen(np.asarray(mate, dtype=np.int64)))

    @property
    def edges(self) -> frozenset:
        if self._edges is None:
            object.__setattr__(self, "_edges", frozenset(self._ids.tolist()))
        return self._edges

    def __eq__(self, other: object) -> bool:
        if isinstance(other, Matching):
            return np.array_equal(self._ids, other._ids) and np.array_equal(self.mate, other.mate)
        if hasattr(other, "edges") and hasattr(other, "mate"):
            return self.edges == other.edges and np.array_equal(self.mate, other.mate)
        return NotImplemented

    def __hash__(self) -> int:
        return hash(self.edges)

    def __repr__(self) -> str:
        return f"Matching(size={self.size}, n={self.mate.size})"

    @property
    def size(self) -> int:
        return int(self._ids.size)

    def sorted_edge_ids(self) -> np.ndarray:
        return self._ids

    def weight(self, g) -> float:
        """graph.py:54-56,191-192: the sum over the ascending ids."""
        ids = self._ids
        return float(np.asarray(g.edge_weight)[ids].sum()) if ids.size else 0.0


def matching_from_edge_ids(g, edge_ids) -> Matching:
    """graph.py:195-203."""
    ids = np.asarray(list(edge_ids) if not isinstance(edge_ids, np.ndarray) else edge_ids,
                     dtype=np.int64)
    mate = np.full(g.num_vertices, -1, dtype=np.int64)
    if ids.size:
        eu = np.asarray(g.edge_u)
        ev = np.asarray(g.edge_v)
        mate[eu[ids]] = ev[ids]
        mate[ev[ids]] = eu[ids]
    return Matching(ids, mate)


class MatchingCheck(NamedTuple):
    valid: bool
    maximal: bool
    detail: str


def validate_matching(g, m) -> MatchingCheck:
    """graph.py:212-237 semantics, vectorised (never raises)."""
    n = g.num_vertices
    mate = np.asarray(m.mate)
    if mate.shape != (n,):
        return MatchingCheck(False, False, "mate table has wrong length")
    ids = m.sorted_edge_ids() if hasattr(m, "sorted_edge_ids") else np.array(sorted(m.edges), dtype=np.int64)
    eu = np.asarray(g.edge_u)
    ev = np.asarray(g.edge_v)
    if ids.size and (ids.min() < 0 or ids.max() >= eu.size):
        return MatchingCheck(False, False, "edge id out of range")
    ends = np.concatenate([eu[ids], ev[ids]])
    if np.unique(ends).size != ends.size:
        return MatchingCheck(False, False, "vertex shared by two matched edges")
    if ids.size and (np.any(mate[eu[ids]] != ev[ids]) or np.any(mate[ev[ids]] != eu[ids])):
        return MatchingCheck(False, False, "mate table disagrees with a matched edge")
    seen = np.zeros(n, dtype=bool)
    seen[ends] = True
    if np.any(mate[~seen] != -1):
        return MatchingCheck(False, False, "mate entry set for an unmatched vertex")
    addable = bool(np.any((mate[eu] == -1) & (mate[ev] == -1)))
    return MatchingCheck(True, not addable, "")


if _RefRoundStats is not None:
    RoundStats = _RefRoundStats

    @dataclass
    class PhaseTrace(_RefPhaseTrace):
        """locmax.PhaseTrace (matchers.py:28-58) plus the device time of the round loop."""

        device_millis: float = 0.0
else:
    @dataclass(frozen=True, eq=False)
    class RoundStats:
        """matchers.py:21-25.  Equal to any object with the same three fields
        (e.g. a locmax.RoundStats), so traces compare with ``==``."""

        edges_before: int
        edges_matched: int
        edges_removed: int

        def _key(self):
            return (self.edges_before, self.edges_matched, self.edges_removed)

        def __eq__(self, other: object) -> bool:
            try:
                return self._key() == (other.edges_before, other.edges_matched, other.edges_removed)
            except AttributeError:
                return NotImplemented

        def __hash__(self) -> int:
            return hash(self._key())

    @dataclass
    class PhaseTrace:
        """matchers.py:28-58, plus device timing of the B200 round loop."""

        rounds: list = field(default_factory=list)
        wall_millis: float = 0.0
        messages: list | None = None
        slot_ops: int | None = None
        write_log: object | None = None
        device_millis: float = 0.0

        @property
        def total_rounds(self) -> int:
            return len(self.rounds)

        def removed_fractions(self) -> list[float]:
            return [r.edges_removed / r.edges_before for r in self.rounds if r.edges_before]

        def survivor_fractions(self) -> list[float]:
            return [(r.edges_before - r.edges_removed) / r.edges_before
                    for r in self.rounds if r.edges_before]

        def mean_removed_fraction(self) -> float:
            fr = self.removed_fractions()
            return sum(fr) / len(fr) if fr else 0.0
