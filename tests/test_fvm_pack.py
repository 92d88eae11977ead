"""The vectorised FVM host path (fvm._pack, fvm._term_layout, fvm.stability_limit)
against straightforward per-edge / per-vertex restatements of the reference's loops
(fvm.py:99-103, :126-152, :209-251), on graphs with constant / linear / tabulated
drifts, mixed degrees and a hub wider than the bit-key path (CPU)."""

import math

import numpy as np
import pytest

import cases
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import fvm, workloads
from paper_2512_02175_b200.coefficients import eval_diffusion, eval_drift
from paper_2512_02175_b200.graph import AT_INIT


def _graphs():
    out = [cases.build(c, gs) for c in ("hub8", "hub64", "path3", "cycle3", "single_edge")]
    g, _ = cases.build("hub8", gs)

    def tab(e):
        L = float(g.edge_length[e])
        return gs.TabulatedDrift((0.0, 0.3 * L, 0.7 * L, L), (1.0, -2.0, 0.5, 0.1))

    drifts = [tab(e) if e % 3 == 0 else
              (gs.LinearDrift(-2.0 - e) if e % 3 == 1 else gs.ConstantDrift(0.7 * e - 2.0))
              for e in range(g.n_edges)]
    out.append((g, gs.CoefficientField.for_graph(g, drifts, [1.0 + 0.1 * e
                                                             for e in range(g.n_edges)])))
    for deg in (50, 70):  # bit-key templates / per-pattern fallback
        h = gs.build_graph([(0, i + 1, 0.5 + 0.01 * i) for i in range(deg)])
        out.append((h, gs.CoefficientField.for_graph(
            h, [gs.LinearDrift(-1.0 - 0.1 * i) if i % 2 else gs.ConstantDrift(0.3 - 0.02 * i)
                for i in range(deg)], [1.0] * deg)))
    out.append(workloads.vascular(1500, seed=4))
    return out


GRAPHS = _graphs()


def _stability_loops(graph, field, grid):
    """fvm.py:209-251 as written: per edge, then per vertex slot pair."""
    max_rate = 0.0
    for e in range(grid.n_edges):
        dx = float(grid.dx[e])
        xs = np.arange(int(grid.counts[e]) + 1) * dx
        mu_max = max(abs(eval_drift(field, e, float(x))) for x in xs)
        D = 0.5 * eval_diffusion(field, e, 0.0) ** 2
        max_rate = max(max_rate, mu_max / dx + 2.0 * D / (dx * dx))
    p = fvm._pack(graph, field, grid)
    deg = np.diff(p.v_off)
    for v in np.flatnonzero(deg >= 2):
        lo, hi = int(p.v_off[v]), int(p.v_off[v + 1])
        b, dxs, D_v = p.v_b[lo:hi], p.v_dx[lo:hi], p.v_D[lo:hi]
        for i in range(hi - lo):
            diff_rate = 0.0
            for j in range(hi - lo):
                if j != i:
                    dxh = 2.0 * dxs[i] * dxs[j] / (dxs[i] + dxs[j])
                    diff_rate += D_v[i] * b[j] / (b[i] * dxh)
            dx = float(dxs[i])
            eid = int(graph.v_edges[lo + i])
            x_v = 0.0 if graph.v_orient[lo + i] == AT_INIT else float(grid.lengths[eid])
            rate = (p.v_speed_in[lo + i] / dx + diff_rate / dx + abs(eval_drift(field, eid, x_v)) / dx
                    + 2.0 * D_v[i] / (dx * dx))
            max_rate = max(max_rate, rate)
    return math.inf if max_rate == 0.0 else 1.0 / max_rate


@pytest.mark.parametrize("k", range(len(GRAPHS)))
@pytest.mark.parametrize("cells", [1, 3, 8])
def test_vectorised_fvm_host_path(k, cells):
    g, f = GRAPHS[k]
    grid = gs.EdgeGrid.uniform(g, cells)
    fvm._PACK_MEMO.clear()
    p = fvm._pack(g, f, grid)
    # interior-face drifts and slot drifts, per edge as in the reference
    faces = [fvm._face_drift(f, e, grid) for e in range(g.n_edges)]
    np.testing.assert_array_equal(p.face_mu, np.concatenate(faces) if p.face_mu.size
                                  else p.face_mu)
    at_init = np.asarray(g.v_orient) == AT_INIT
    x_v = np.where(at_init, 0.0, np.asarray(grid.lengths)[g.v_edges])
    mu_v = np.array([eval_drift(f, int(e), float(x)) for e, x in zip(g.v_edges, x_v)])
    speed = np.where(at_init, -mu_v, mu_v)
    np.testing.assert_array_equal(p.v_speed_in, np.where(speed > 0.0, speed, 0.0))
    # exchange-term layout: bit-key templates == per-pattern templates
    if np.diff(p.v_off).max() <= 60:
        a = fvm._term_layout(p.v_off, p.v_b, p.v_speed_in, p.pslot, p.slot_vertex)
        b = fvm._term_layout(p.v_off, p.v_b, p.v_speed_in, p.pslot, p.slot_vertex, bitkey=False)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(np.asarray(x), np.asarray(y))
    # CFL limit: the reference's loops, bit for bit
    assert fvm.stability_limit(g, f, grid) == _stability_loops(g, f, grid)
