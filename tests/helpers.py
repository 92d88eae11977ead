"""Shared test helpers (graph construction for golden metadata, tolerances)."""

import numpy as np

import cases
import golden_io
import paper_2512_02175_b200 as gs

#: positions: reference (numba fastmath) vs strict-IEEE paths, whole trajectories
POS_ATOL = 1e-10


_C4 = []


def vascular_c4():
    """The C4 network (workloads.vascular(): ~1.02e5 edges), built once per session."""
    if not _C4:
        _C4.append(gs.workloads.vascular())
    return _C4[0]


def graph_for(case):
    if case == "vascular_small":
        return gs.parse_graph_file(golden_io.vascular_small_text())
    if case == "vascular_c4":
        return vascular_c4()
    return cases.build(case, gs)


def graph_digest(g, f) -> str:
    """SHA-256 of a graph's packed arrays (tests/golden/make_c4_golden.py)."""
    import hashlib

    h = hashlib.sha256()
    for a in (g.edge_init, g.edge_term, g.edge_length, g.v_off, g.v_edges, g.v_orient,
              g.v_cumw) + tuple(f.packed()):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def initial_for(init):
    kind = init[0]
    if kind == "at":
        return gs.AtVertex(init[1])
    if kind == "point":
        return gs.PointStart(init[1], init[2])
    return gs.PerEdgeUniform(init[1])


def oracle_init(init, graph):
    if init[0] == "at":
        lo = int(graph.v_off[init[1]])
        e = int(graph.v_edges[lo])
        return (0, e, graph.vertex_position(e, int(graph.v_orient[lo])), 0.0)
    if init[0] == "point":
        return (0, init[1], init[2], 0.0)
    return (1, 0, 0.0, float(init[1]))


def config_for(m, rng="reference", **kw):
    g, f = graph_for(m["case"])
    init = list(m["init"])
    if m["case"] == "vascular_small":
        init = ["uniform", float(np.max(g.edge_length))]
    cfg = gs.SimulationConfig(dt=m["dt"], n_steps=m["steps"], n_particles=m["n"], seed=m["seed"],
                              max_splits_per_step=m["cap"], initial=initial_for(init),
                              reflect_at=m["reflect"], rng=rng, **kw)
    return g, f, cfg, init


def assert_positions(a, b, atol=POS_ATOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    bad = ~((a == b) | (np.abs(a - b) <= atol))
    assert not bad.any(), (np.flatnonzero(bad)[:10], a[bad][:5], b[bad][:5])


def binom_z(c1, n1, c2, n2):
    """Two-sample binomial z-score of proportions c1/n1 vs c2/n2."""
    p1, p2 = c1 / n1, c2 / n2
    p = (c1 + c2) / (n1 + n2)
    se = np.sqrt(np.maximum(p * (1 - p) * (1 / n1 + 1 / n2), 1e-300))
    return (p1 - p2) / se


def chi2_two_sample(h1, h2, min_count=20):
    """Two-sample chi-square homogeneity test on histograms; returns p-value."""
    from scipy import stats

    h1 = np.asarray(h1, np.float64)
    h2 = np.asarray(h2, np.float64)
    keep = (h1 + h2) >= min_count
    a, b = h1[keep], h2[keep]
    n1, n2 = a.sum(), b.sum()
    k1, k2 = np.sqrt(n2 / n1), np.sqrt(n1 / n2)
    chi2 = float((((k1 * a - k2 * b) ** 2) / (a + b)).sum())
    dof = int(keep.sum()) - 1
    return float(stats.chi2.sf(chi2, dof)), chi2, dof
