"""The five BASELINE.json workloads as concrete, seeded graphs.

* ``star3``     -- C1: 3 semi-infinite edges, Brownian (mu=0, sigma=1).
* ``hub64``     -- C2: 64 edges 0->i+1, lengths U[0.5,2] (seed 0), LinearDrift(-k_i),
                   k_i ~ U[1,20]; not a star (finite lengths) => general stepper.
* ``star5``     -- C3: the paper's §4.1 star, ConstantDrift(-10 i), i=1..5.
* ``vascular``  -- C4/C5: random geometric tree with loops (kNN -> MST -> +2% loops),
                   Poiseuille flux, drift from_flux, emitted through the graph-file
                   format so every consumer loads the identical graph.

All generators are deterministic functions of their arguments.  Each takes an
optional ``api`` -- a module exposing the reference's graph-construction names
(``build_graph``, ``CoefficientField``, ``ConstantDrift``, ``LinearDrift`` and a
``graphfile`` submodule): this package by default, or the reference ``graphsde``
itself, so ``bench.py``'s reference arm times the reference on the identical
graphs.
"""

from __future__ import annotations

import math

import numpy as np

import importlib
import sys


def _api(api):
    return sys.modules[__package__] if api is None else api


def _graphfile(api):
    return importlib.import_module(_api(api).__name__ + ".graphfile")


def star(n_edges: int, drift, sigma=1.0, weights=None, api=None):
    A = _api(api)
    graph = A.build_graph([(0, None, math.inf)] * n_edges, {0: weights} if weights else None)
    drift = list(drift)
    sig = [sigma] * n_edges if np.isscalar(sigma) else list(sigma)
    return graph, A.CoefficientField.for_graph(graph, drift, sig)


def star3(api=None):
    return star(3, [_api(api).ConstantDrift(0.0)] * 3, api=api)


def star5(kind: str = "linear", api=None):
    A = _api(api)
    if kind == "linear":
        drift = [A.ConstantDrift(-10.0 * i) for i in range(1, 6)]
    else:
        drift = [A.LinearDrift(-10.0 * i) for i in range(1, 6)]
    return star(5, drift, api=api)


def hub64(seed: int = 0, api=None):
    A = _api(api)
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(0.5, 2.0, 64)
    ks = rng.uniform(1.0, 20.0, 64)
    graph = A.build_graph([(0, i + 1, float(lengths[i])) for i in range(64)])
    field = A.CoefficientField.for_graph(graph, [A.LinearDrift(-float(k)) for k in ks],
                                         [1.0] * 64)
    return graph, field


def vascular_tables(n_nodes: int = 100_000, seed: int = 2512, loop_frac: float = 0.02):
    """Node and segment tables of a synthetic cortical-vascular-like network.

    Nodes uniform in a cube of side ``n^(1/3)`` (unit mean spacing); 4-NN
    graph -> minimum spanning tree -> largest component; plus ``loop_frac``
    extra kNN edges as loops.  Radii ~ LogNormal(0, 0.25); pressure
    ``p = -4 z + N(0, 0.1)``; Poiseuille-like flux ``Q = (pi/2) r^4 dp / L`` so
    the centreline drift ``Q / (pi r^2)`` is O(1) (gamma ~ 0.1 at dt = 1e-3).
    """
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components, minimum_spanning_tree
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    side = n_nodes ** (1.0 / 3.0)
    pts = rng.uniform(0.0, side, size=(n_nodes, 3))
    dist, idx = cKDTree(pts).query(pts, k=5)
    a = np.repeat(np.arange(n_nodes), 4)
    b = idx[:, 1:].reshape(-1)
    d = dist[:, 1:].reshape(-1)
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    key = np.unique(lo.astype(np.int64) * n_nodes + hi)
    ka, kb = key // n_nodes, key % n_nodes
    kd = np.linalg.norm(pts[ka] - pts[kb], axis=1)
    knn = coo_matrix((kd, (ka, kb)), shape=(n_nodes, n_nodes)).tocsr()
    mst = minimum_spanning_tree(knn).tocoo()
    ncomp, labels = connected_components(mst, directed=False)
    big = np.argmax(np.bincount(labels))
    keep = labels == big
    ta, tb = mst.row.astype(np.int64), mst.col.astype(np.int64)
    tmask = keep[ta] & keep[tb]
    ta, tb = ta[tmask], tb[tmask]
    tree = set((np.minimum(ta, tb) * n_nodes + np.maximum(ta, tb)).tolist())
    cand = np.array([k for k in key.tolist() if k not in tree], dtype=np.int64)
    cand = cand[keep[cand // n_nodes] & keep[cand % n_nodes]]
    n_loops = int(round(loop_frac * ta.shape[0]))
    extra = rng.choice(cand, size=min(n_loops, cand.shape[0]), replace=False)
    ea = np.concatenate([np.minimum(ta, tb), extra // n_nodes])
    eb = np.concatenate([np.maximum(ta, tb), extra % n_nodes])
    # dense relabelling of the kept component
    new_id = np.full(n_nodes, -1, dtype=np.int64)
    kept = np.flatnonzero(keep)
    new_id[kept] = np.arange(kept.shape[0])
    ea, eb = new_id[ea], new_id[eb]
    P = pts[kept]
    m = ea.shape[0]
    radius = np.exp(rng.normal(0.0, 0.25, size=m))
    pressure = -4.0 * P[:, 2] + rng.normal(0.0, 0.1, size=P.shape[0])
    length = np.linalg.norm(P[ea] - P[eb], axis=1)
    flux = (math.pi / 2.0) * radius**4 * (pressure[ea] - pressure[eb]) / length
    nodes = [(i, float(x), float(y), float(z)) for i, (x, y, z) in enumerate(P.tolist())]
    segs = [
        (s, int(ea[s]), int(eb[s]), float(radius[s]), float(flux[s])) for s in range(m)
    ]
    return nodes, segs


def vascular_text(n_nodes: int = 100_000, seed: int = 2512, api=None) -> str:
    return _graphfile(api).network_tables_to_graph_file(*vascular_tables(n_nodes, seed))


def vascular(n_nodes: int = 100_000, seed: int = 2512, api=None):
    return _graphfile(api).parse_graph_file(vascular_text(n_nodes, seed, api))
