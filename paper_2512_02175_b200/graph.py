"""Metric graphs and their packed incidence (host side of the drop-in boundary).

Same public surface and error behaviour as the reference ``graphsde.graph``
(``/root/reference/pkg/src/graphsde/graph.py``): :func:`build_graph` validates
``(init, term, length)`` triples and per-vertex jump weights, and produces the
packed CSR incidence (``v_off``/``v_edges``/``v_orient``/``v_cumw``) that the
device simulator samples exit slots from.

Differences are internal only:

* construction is vectorised numpy (a 1e5-edge vascular graph builds in well
  under a second instead of seconds), while reproducing the reference's
  arrays bit-for-bit -- slots are sorted by (vertex, edge id)
  (``graph.py:208-213``) and cumulative weights are sequential prefix sums of
  ``w / sum(w)`` or ``1/deg`` (``graph.py:236-248``);
* ``incidence`` is a lazy sequence so huge graphs do not materialise one
  Python object per vertex unless asked;
* :attr:`MetricGraph.v_thresh` holds the 53-bit integer form of ``v_cumw``
  used by the device's exact inverse-CDF slot pick (SURVEY.md §8 note 1).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EdgeId = int
VertexId = int

#: Sentinel vertex id used as the terminal endpoint of semi-infinite edges
#: (reference ``graph.py:26``).
INFINITY_VERTEX: VertexId = -1

#: Orientation of an incident edge slot (reference ``graph.py:30-31``).
AT_INIT = 0
AT_TERM = 1

#: Tolerance for user jump weights whose sum is off (reference ``graph.py:34``).
WEIGHT_SUM_TOLERANCE = 1e-9

_TWO53 = float(2.0**53)


class GraphBuildError(ValueError):
    """Base class for metric-graph construction failures."""


class NonPositiveLength(GraphBuildError):
    pass


class WeightSimplexViolation(GraphBuildError):
    pass


class DanglingVertexReference(GraphBuildError):
    pass


class DisconnectedGraph(GraphBuildError):
    pass


class SelfLoopError(GraphBuildError):
    pass


class InfinityVertex(ValueError):
    """Raised when an operation requires a finite vertex but got the sentinel."""


@dataclass(frozen=True)
class Edge:
    """Oriented edge ``[0, length]`` from ``init`` to ``term`` (``graph.py:65-79``)."""

    init: VertexId
    term: VertexId
    length: float

    @property
    def is_semi_infinite(self) -> bool:
        return math.isinf(self.length)


@dataclass(frozen=True)
class VertexIncidence:
    """Incident slots of one finite vertex, increasing edge id (``graph.py:82-99``)."""

    edges: np.ndarray
    orientations: np.ndarray
    jump_weights: np.ndarray
    cum_weights: np.ndarray

    @property
    def degree(self) -> int:
        return int(self.edges.shape[0])


class _IncidenceView:
    """Read-only sequence of :class:`VertexIncidence`, built on first access."""

    __slots__ = ("_g", "_cache")

    def __init__(self, g: "MetricGraph"):
        self._g = g
        self._cache: dict[int, VertexIncidence] = {}

    def __len__(self) -> int:
        return int(self._g.v_off.shape[0] - 1)

    def __getitem__(self, v):
        if isinstance(v, slice):
            return tuple(self[i] for i in range(*v.indices(len(self))))
        v = int(v)
        n = len(self)
        if v < 0:
            v += n
        if not 0 <= v < n:
            raise IndexError("vertex index out of range")
        inc = self._cache.get(v)
        if inc is None:
            g = self._g
            lo, hi = int(g.v_off[v]), int(g.v_off[v + 1])
            inc = VertexIncidence(
                _frozen(g.v_edges[lo:hi].copy()),
                _frozen(g.v_orient[lo:hi].copy()),
                _frozen(g.v_weights[lo:hi].copy()),
                _frozen(g.v_cumw[lo:hi].copy()),
            )
            self._cache[v] = inc
        return inc

    def __iter__(self):
        for v in range(len(self)):
            yield self[v]


@dataclass(frozen=True, eq=False)
class MetricGraph:
    """Validated metric graph plus packed arrays (``graph.py:102-147``)."""

    edges: tuple
    is_star: bool
    edge_init: np.ndarray
    edge_term: np.ndarray
    edge_length: np.ndarray
    v_off: np.ndarray
    v_edges: np.ndarray
    v_orient: np.ndarray
    v_cumw: np.ndarray
    v_weights: np.ndarray
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def incidence(self) -> _IncidenceView:
        view = self._device.get("_incidence")
        if view is None:
            view = _IncidenceView(self)
            self._device["_incidence"] = view
        return view

    @property
    def n_edges(self) -> int:
        return int(self.edge_length.shape[0])

    @property
    def n_vertices(self) -> int:
        return int(self.v_off.shape[0] - 1)

    @property
    def has_semi_infinite_edges(self) -> bool:
        return bool(np.isinf(self.edge_length).any())

    @property
    def v_thresh(self) -> np.ndarray:
        """``floor(v_cumw * 2**53)`` as uint64, saturated at ``2**53``.

        ``u = (r >> 11) * 2**-53 <= cumw`` iff ``(r >> 11) <= v_thresh``
        (the scale by 2**53 is exact), so the device picks the reference's
        slot with integer compares only.
        """
        t = self._device.get("_thresh")
        if t is None:
            c = np.minimum(np.floor(self.v_cumw * _TWO53), _TWO53)
            t = _frozen(np.maximum(c, 0.0).astype(np.uint64))
            self._device["_thresh"] = t
        return t

    def degree(self, v: VertexId) -> int:
        return int(self.v_off[v + 1] - self.v_off[v])

    def finite_vertices(self) -> range:
        return range(self.n_vertices)

    def vertex_position(self, e: EdgeId, orientation: int) -> float:
        return 0.0 if orientation == AT_INIT else float(self.edge_length[e])


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def _validate_edges(triples):
    """Per-edge checks in the reference's order (``graph.py:188-207``)."""
    inits, terms, lengths = [], [], []
    for idx, (init, term, length) in enumerate(triples):
        if term is None:
            term = INFINITY_VERTEX
        init = int(init)
        term = int(term)
        length = float(length)
        if not length > 0.0:
            raise NonPositiveLength(f"edge {idx}: length {length!r} must be positive")
        if math.isinf(length) != (term == INFINITY_VERTEX):
            raise GraphBuildError(
                f"edge {idx}: semi-infinite edges must pair length=inf with the "
                f"infinity-vertex sentinel (got term={term}, length={length})"
            )
        if init == INFINITY_VERTEX:
            raise GraphBuildError(f"edge {idx}: init endpoint cannot be the infinity vertex")
        if init < 0 or (term < 0 and term != INFINITY_VERTEX):
            raise DanglingVertexReference(f"edge {idx}: negative vertex id")
        if init == term:
            raise SelfLoopError(f"edge {idx}: self-loops are not supported")
        inits.append(init)
        terms.append(term)
        lengths.append(length)
    return (
        np.asarray(inits, dtype=np.int64),
        np.asarray(terms, dtype=np.int64),
        np.asarray(lengths, dtype=np.float64),
    )


def _segmented_prefix_sum(w: np.ndarray, v_off: np.ndarray, rank: np.ndarray) -> np.ndarray:
    """Left-to-right prefix sums inside each vertex segment.

    Evaluated level by level (rank 0, 1, ...) so every partial sum is the
    same sequence of IEEE additions as ``np.cumsum`` on the segment.
    """
    cum = np.empty_like(w)
    first = rank == 0
    cum[first] = w[first]
    max_rank = int(rank.max()) if rank.size else 0
    for r in range(1, max_rank + 1):
        idx = np.flatnonzero(rank == r)
        cum[idx] = cum[idx - 1] + w[idx]
    return cum


def build_graph(edges, jump_weights: dict | None = None) -> MetricGraph:
    """Build and validate a :class:`MetricGraph` (reference ``graph.py:155-282``).

    Raises the reference's error classes in the reference's order:
    NonPositiveLength, GraphBuildError, DanglingVertexReference, SelfLoopError,
    WeightSimplexViolation, DisconnectedGraph.
    """
    init, term, length = _validate_edges(edges)
    return build_graph_arrays(init, term, length, jump_weights)


def _edges_valid(init: np.ndarray, term: np.ndarray, length: np.ndarray) -> bool:
    """Vectorised form of the per-edge checks of :func:`_validate_edges`."""
    inf_len = np.isinf(length)
    return bool(
        np.all(length > 0.0)
        and np.array_equal(inf_len, term == INFINITY_VERTEX)
        and np.all(init >= 0)
        and np.all((term >= 0) | (term == INFINITY_VERTEX))
        and not np.any(init == term)
    )


def build_graph_arrays(init, term, length, jump_weights: dict | None = None) -> MetricGraph:
    """:func:`build_graph` from edge arrays (int64 init/term with -1 for the
    vertex at infinity, float64 lengths).  Arrays that fail the per-edge
    checks are re-validated edge by edge for the reference's error."""
    init = np.ascontiguousarray(init, dtype=np.int64)
    term = np.ascontiguousarray(term, dtype=np.int64)
    length = np.ascontiguousarray(length, dtype=np.float64)
    if not _edges_valid(init, term, length):
        init, term, length = _validate_edges(zip(init.tolist(), term.tolist(), length.tolist()))
    m = int(init.shape[0])
    if m == 0:
        raise GraphBuildError("a metric graph needs at least one edge")

    finite = term != INFINITY_VERTEX
    n_vertices = int(max(init.max(), term[finite].max() if finite.any() else -1)) + 1

    # slots: one per (finite endpoint, edge); sorted by (vertex, edge id)
    eid = np.arange(m, dtype=np.int64)
    s_vert = np.concatenate([init, term[finite]])
    s_edge = np.concatenate([eid, eid[finite]])
    s_orient = np.concatenate(
        [np.full(m, AT_INIT, np.int8), np.full(int(finite.sum()), AT_TERM, np.int8)]
    )
    order = np.lexsort((s_edge, s_vert))
    s_vert, s_edge, s_orient = s_vert[order], s_edge[order], s_orient[order]

    deg = np.bincount(s_vert, minlength=n_vertices).astype(np.int64)
    missing = np.flatnonzero(deg == 0)
    if missing.size:
        raise DanglingVertexReference(
            f"vertex {int(missing[0])} is never referenced by any edge (ids must be dense)"
        )
    v_off = np.zeros(n_vertices + 1, dtype=np.int64)
    np.cumsum(deg, out=v_off[1:])
    rank = np.arange(s_vert.shape[0], dtype=np.int64) - v_off[s_vert]

    jump_weights = dict(jump_weights or {})
    for v in jump_weights:
        if not (0 <= v < n_vertices):
            raise DanglingVertexReference(f"jump weights given for unknown vertex {v}")

    # default 1/deg weights, then user weights (validated per vertex in id order)
    w = (1.0 / deg.astype(np.float64))[s_vert]
    for v in sorted(jump_weights):
        d = int(deg[v])
        wv = np.asarray(jump_weights[v], dtype=np.float64)
        if wv.shape != (d,):
            got = wv.shape[0] if wv.ndim else 0
            raise WeightSimplexViolation(
                f"vertex {v}: expected {d} weights (one per incident edge), got {got}"
            )
        if np.any(wv < 0.0) or np.any(wv > 1.0):
            raise WeightSimplexViolation(f"vertex {v}: weights must lie in [0, 1]")
        total = float(wv.sum())
        if abs(total - 1.0) > WEIGHT_SUM_TOLERANCE:
            raise WeightSimplexViolation(f"vertex {v}: weights sum to {total!r}, expected 1")
        w[v_off[v] : v_off[v + 1]] = wv / total
    cumw = _segmented_prefix_sum(w, v_off, rank)

    _check_connected(n_vertices, init[finite], term[finite])

    is_star = n_vertices == 1 and bool(np.isinf(length).all()) and bool((init == 0).all())
    edge_objs = tuple(
        Edge(int(a), int(b), float(c)) for a, b, c in zip(init.tolist(), term.tolist(), length.tolist())
    )
    return MetricGraph(
        edges=edge_objs,
        is_star=is_star,
        edge_init=_frozen(init),
        edge_term=_frozen(term),
        edge_length=_frozen(length),
        v_off=_frozen(v_off),
        v_edges=_frozen(s_edge.astype(np.int64)),
        v_orient=_frozen(s_orient.astype(np.int8)),
        v_cumw=_frozen(cumw),
        v_weights=_frozen(w),
    )


def _check_connected(n_vertices: int, a: np.ndarray, b: np.ndarray) -> None:
    """Connectivity over finite vertices (reference ``graph.py:285-306``)."""
    if n_vertices == 1:
        return
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    adj = coo_matrix(
        (np.ones(a.shape[0], dtype=np.int8), (a, b)), shape=(n_vertices, n_vertices)
    )
    _, labels = connected_components(adj, directed=False)
    unreachable = np.flatnonzero(labels != labels[0])
    if unreachable.size:
        raise DisconnectedGraph(
            f"graph is not connected over finite vertices (unreachable: {unreachable.tolist()})"
        )


def sample_exit_edge(graph: MetricGraph, v: VertexId, u: float) -> tuple[EdgeId, int]:
    """First slot ``j`` at ``v`` with ``u <= cum_weights[j]``, else the last slot
    (reference ``graph.py:309-326``)."""
    if v == INFINITY_VERTEX or v < 0 or v >= graph.n_vertices:
        raise InfinityVertex(f"cannot sample an exit edge at vertex {v}")
    lo, hi = int(graph.v_off[v]), int(graph.v_off[v + 1])
    hits = np.flatnonzero(u <= graph.v_cumw[lo:hi])
    slot = lo + (int(hits[0]) if hits.size else hi - lo - 1)
    return int(graph.v_edges[slot]), int(graph.v_orient[slot])
