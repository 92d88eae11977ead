"""Graph/field cases shared by the golden generator and the tests.

Plain data only, so the same case can be built with the reference package
(``graphsde``, in make_golden.py) or with ``paper_2512_02175_b200`` (tests).
"""

from __future__ import annotations

import math

import numpy as np

INF = math.inf


def _hub(n, seed, lo=0.5, hi=2.0, klo=1.0, khi=20.0):
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(lo, hi, n)
    ks = rng.uniform(klo, khi, n)
    return dict(
        edges=[(0, i + 1, float(lengths[i])) for i in range(n)],
        weights=None,
        drift=[("linear", -float(k)) for k in ks],
        sigma=[1.0] * n,
    )


def _random_general(n_v, n_extra, seed):
    """Connected random graph: random tree + extra edges, mixed drift kinds."""
    rng = np.random.default_rng(seed)
    edges = []
    for v in range(1, n_v):
        u = int(rng.integers(0, v))
        a, b = (u, v) if rng.random() < 0.5 else (v, u)
        edges.append((a, b, float(rng.uniform(0.3, 1.5))))
    have = {(min(a, b), max(a, b)) for a, b, _ in edges}
    while len(edges) < n_v - 1 + n_extra:
        a, b = (int(x) for x in rng.integers(0, n_v, 2))
        if a == b or (min(a, b), max(a, b)) in have:
            continue
        have.add((min(a, b), max(a, b)))
        edges.append((a, b, float(rng.uniform(0.3, 1.5))))
    drift = []
    for i, (_, _, l) in enumerate(edges):
        r = i % 3
        if r == 0:
            drift.append(("constant", float(rng.uniform(-3, 3))))
        elif r == 1:
            drift.append(("linear", float(rng.uniform(-4, 4))))
        else:
            xs = sorted(float(x) for x in rng.uniform(0, l, 3))
            drift.append(("tabulated", xs, [float(m) for m in rng.uniform(-3, 3, 3)]))
    sigma = [float(s) for s in rng.uniform(0.5, 1.5, len(edges))]
    # non-uniform weights (with a zero) at vertex 0 and 1
    deg = {}
    for a, b, _ in edges:
        deg[a] = deg.get(a, 0) + 1
        deg[b] = deg.get(b, 0) + 1
    weights = {}
    for v in (0, 1):
        d = deg[v]
        w = rng.uniform(0.1, 1.0, d)
        if d >= 3:
            w[1] = 0.0
        w = w / w.sum()
        weights[v] = [float(x) for x in w]
    return dict(edges=edges, weights=weights, drift=drift, sigma=sigma)


CASES = {
    # C1: 3-edge Brownian star
    "star3_bm": dict(edges=[(0, None, INF)] * 3, weights=None,
                     drift=[("constant", 0.0)] * 3, sigma=[1.0] * 3),
    "star3_drift": dict(edges=[(0, None, INF)] * 3, weights=None,
                        drift=[("constant", -10.0), ("constant", -20.0), ("constant", -30.0)],
                        sigma=[1.0] * 3),
    # C3 / paper §4.1 stars
    "star5_linear": dict(edges=[(0, None, INF)] * 5, weights=None,
                         drift=[("constant", -10.0 * i) for i in range(1, 6)], sigma=[1.0] * 5),
    "star5_quad": dict(edges=[(0, None, INF)] * 5, weights=None,
                       drift=[("linear", -10.0 * i) for i in range(1, 6)], sigma=[1.0] * 5),
    "star_homog": dict(edges=[(0, None, INF)] * 4, weights=None,
                       drift=[("constant", -50.0)] * 4, sigma=[1.0] * 4),
    # mixed kinds, non-uniform weights incl. a zero weight, varying sigma
    "star4_mixed": dict(edges=[(0, None, INF)] * 4,
                        weights={0: [0.1, 0.0, 0.6, 0.3]},
                        drift=[("constant", -5.0), ("linear", -8.0),
                               ("tabulated", [0.0, 0.05, 0.2], [-20.0, -2.0, 1.0]),
                               ("constant", 3.0)],
                        sigma=[1.0, 0.7, 1.3, 2.0]),
    # C2 (small hub) and general graphs
    "hub64": _hub(64, 0),
    "hub8": _hub(8, 5),
    "path3": dict(edges=[(0, 1, 1.0), (1, 2, 2.0)], weights={1: [0.3, 0.7]},
                  drift=[("constant", 0.5), ("constant", -0.3)], sigma=[1.0, 1.0]),
    "single_edge": dict(edges=[(0, 1, 1.0)], weights=None, drift=[("constant", 0.0)],
                        sigma=[1.0]),
    "cycle3": dict(edges=[(0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0)], weights=None,
                   drift=[("constant", 30.0)] * 3, sigma=[1.0] * 3),
    "random_general": _random_general(14, 6, 7),
}


def build(case, ns):
    """Build (graph, field) for ``case`` with namespace ``ns`` (a package
    exposing build_graph / CoefficientField / *Drift)."""
    spec = CASES[case] if isinstance(case, str) else case
    graph = ns.build_graph(spec["edges"], spec["weights"])
    drift = []
    for d in spec["drift"]:
        if d[0] == "constant":
            drift.append(ns.ConstantDrift(d[1]))
        elif d[0] == "linear":
            drift.append(ns.LinearDrift(d[1]))
        else:
            drift.append(ns.TabulatedDrift(tuple(d[1]), tuple(d[2])))
    field = ns.CoefficientField.for_graph(graph, drift, spec["sigma"])
    return graph, field
