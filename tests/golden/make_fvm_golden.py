"""Golden vectors for the finite-volume baseline from the REFERENCE (graphsde/fvm.py).

    python tests/golden/make_fvm_golden.py

Runs the reference's numba stepper ``_fvm_step_loop`` on ``_pack_static``
arrays, plus ``stability_limit`` and the flux helpers, over FVM_CASES and
writes tests/golden/fvm.npz.  Graphs come from cases.py (plain data), grids
and initial densities from FVM_CASES, so tests rebuild identical inputs with
this package.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

from cases import CASES  # noqa: E402


def _counts(case, n_edges):
    c = FVM_CASES[case]["cells"]
    if isinstance(c, int):
        return np.full(n_edges, c, dtype=np.int64)
    return np.asarray(c, dtype=np.int64)


def grid_spec(case, graph_lengths):
    """(counts, lengths) of the case's grid."""
    spec = FVM_CASES[case]
    n = len(graph_lengths)
    lengths = np.asarray(spec.get("lengths") or graph_lengths, dtype=np.float64)
    if lengths.shape[0] != n:
        lengths = np.full(n, lengths[0])
    return _counts(case, n), lengths


def initial_rho(case, counts, lengths):
    kind = FVM_CASES[case].get("init", "uniform")
    dx = lengths / counts
    if kind == "uniform":
        return np.repeat(np.full(len(counts), 1.0 / lengths.sum()), counts)
    out = []
    for e, (n, h) in enumerate(zip(counts, dx)):
        x = (np.arange(n) + 0.5) * h
        out.append(1.0 + 0.5 * np.sin(3.0 * x + e))
    return np.concatenate(out)


# graph case -> grid + run parameters (dt as a fraction of the stability limit)
FVM_CASES = {
    "star5_linear": dict(graph="star5_linear", cells=20, lengths=[1.0], cfl=0.9, steps=300),
    "star5_quad": dict(graph="star5_quad", cells=16, lengths=[0.6], cfl=0.95, steps=200,
                       init="bump"),
    "star4_mixed_pos": dict(graph="star4_mixed_pos", cells=12, lengths=[0.8], cfl=0.8,
                            steps=150, init="bump"),
    "hub8": dict(graph="hub8", cells=6, cfl=0.9, steps=400),
    "path3": dict(graph="path3", cells=[3, 5], cfl=1.0, steps=250, init="bump"),
    "cycle3_single": dict(graph="cycle3", cells=[1, 1, 1], cfl=0.7, steps=100, init="bump"),
    "general_ragged": dict(graph="random_general_pos", cells=[1, 3, 2, 1, 4, 1, 2, 5, 1, 3, 2, 2,
                                                                1, 4, 3, 1, 2, 1, 6],
                           cfl=0.9, steps=300, init="bump"),
    "hub8_unstable": dict(graph="hub8", cells=6, cfl=3.0, steps=200),
}


def graph_case(name):
    if name == "star4_mixed_pos":  # star4_mixed without its zero jump weight
        c = dict(CASES["star4_mixed"])
        c["weights"] = {0: [0.1, 0.2, 0.4, 0.3]}
        return c
    if name == "random_general_pos":  # random_general with uniform weights
        c = dict(CASES["random_general"])
        c["weights"] = None
        return c
    return CASES[name]


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import graphsde as gs
    from graphsde import fvm
    from graphsde.grids import EdgeGrid

    from cases import build

    out = {}
    for name, spec in FVM_CASES.items():
        g, f = build(graph_case(spec["graph"]), gs)
        counts, lengths = grid_spec(name, g.edge_length)
        grid = EdgeGrid(counts=counts, lengths=lengths)
        rho0 = initial_rho(name, counts, lengths)
        limit = fvm.stability_limit(g, f, grid)
        dt = spec["cfl"] * limit
        packed = fvm._pack_static(g, f, grid)
        rho = rho0.copy()
        neg = fvm._fvm_step_loop(rho, spec["steps"], dt, *packed, -fvm._NEGATIVE_TOL)
        out[f"{name}/counts"] = counts
        out[f"{name}/lengths"] = lengths
        out[f"{name}/rho0"] = rho0
        out[f"{name}/rho"] = rho
        out[f"{name}/meta"] = np.array([limit, dt, spec["steps"], neg], dtype=np.float64)
        for k, a in zip(("offs", "dx_edge", "D_edge", "face_mu", "face_off", "v_off", "v_cells",
                         "v_b", "v_dx", "v_speed_in", "v_D"), packed):
            out[f"{name}/packed/{k}"] = np.asarray(a)
        st = fvm.FvmState(grid=grid, rho=rho0.copy())
        flux = fvm.fvm_interior_fluxes(st, f, grid)
        out[f"{name}/interior_flux"] = np.concatenate(flux) if flux else np.zeros(0)
        net = [fvm.fvm_vertex_fluxes(st, f, g, grid, v)[0] for v in g.finite_vertices()]
        out[f"{name}/vertex_net"] = np.concatenate(net) if net else np.zeros(0)
        # the reference's own fvm_run (CFL check, exceptions) where it applies
        try:
            res = fvm.fvm_run(g, f, grid, dt, spec["steps"], fvm.FvmState(grid, rho0.copy()),
                              force=spec["cfl"] > 1.0)
            out[f"{name}/run"] = np.concatenate([[res.max_cfl, res.state.t], res.state.rho])
            out[f"{name}/run_error"] = np.array("")
        except Exception as exc:  # noqa: BLE001
            out[f"{name}/run"] = np.zeros(0)
            out[f"{name}/run_error"] = np.array(f"{type(exc).__name__}: {exc}")
        print(name, "limit", limit, "neg", neg, "cells", int(counts.sum()))
    np.savez_compressed(os.path.join(HERE, "fvm.npz"), **out)


if __name__ == "__main__":
    main()
