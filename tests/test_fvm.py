"""Finite-volume baseline (reference fvm.py) -- packing, host helpers and the C
oracle against fixtures the reference produced (tests/golden/fvm.npz,
make_fvm_golden.py); the GPU stepper against both, bit for bit."""

import os
import sys

import numpy as np
import pytest

import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import fvm

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from cases import build  # noqa: E402
from make_fvm_golden import FVM_CASES, graph_case  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "fvm.npz"))
NAMES = list(FVM_CASES)


def setup(name):
    g, f = build(graph_case(FVM_CASES[name]["graph"]), gs)
    grid = gs.EdgeGrid(counts=GOLD[f"{name}/counts"], lengths=GOLD[f"{name}/lengths"])
    limit, dt, steps, neg = GOLD[f"{name}/meta"]
    return g, f, grid, GOLD[f"{name}/rho0"], float(dt), int(steps), int(neg), float(limit)


@pytest.mark.parametrize("name", NAMES)
def test_pack_and_limit_match_reference(name):
    g, f, grid, rho0, dt, steps, neg, limit = setup(name)
    p = fvm._pack(g, f, grid)
    for k, a in zip(("offs", "dx_edge", "D_edge", "face_mu", "face_off", "v_off", "v_cells",
                     "v_b", "v_dx", "v_speed_in", "v_D"), p.reference_tuple()):
        ref = GOLD[f"{name}/packed/{k}"]
        assert a.shape == ref.shape and np.array_equal(a, ref.astype(a.dtype)), k
    assert fvm.stability_limit(g, f, grid) == limit
    st = fvm.FvmState(grid=grid, rho=rho0.copy())
    fl = fvm.fvm_interior_fluxes(st, f, grid)
    got = np.concatenate(fl) if fl else np.zeros(0)
    assert np.array_equal(got, GOLD[f"{name}/interior_flux"])
    net = [fvm.fvm_vertex_fluxes(st, f, g, grid, v)[0] for v in g.finite_vertices()]
    assert np.array_equal(np.concatenate(net), GOLD[f"{name}/vertex_net"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_bitwise(name):
    from oracle import oracle

    g, f, grid, rho0, dt, steps, neg, _ = setup(name)
    rho, n = oracle.fvm_steps(rho0, steps, dt, fvm._pack(g, f, grid).reference_tuple())
    assert n == neg
    assert np.array_equal(rho, GOLD[f"{name}/rho"])


def test_ownership_split():
    g, f, grid, *_ = setup("general_ragged")
    p = fvm._pack(g, f, grid)
    assert p.vser.size > 0 and p.vpar.size > 0  # single-cell edges share cells
    deg = np.diff(p.v_off)
    assert set(p.vpar) | set(p.vser) == set(np.flatnonzero(deg >= 2))
    g, f, grid, *_ = setup("cycle3_single")
    p = fvm._pack(g, f, grid)
    assert list(p.vser) == [0, 1, 2] and p.vpar.size == 0 and p.owned.all()


def test_validation_errors():
    g, f, grid, rho0, dt, steps, _, limit = setup("hub8")
    st = fvm.FvmState(grid=grid, rho=rho0.copy())
    with pytest.raises(ValueError):
        fvm.fvm_run(g, f, grid, 0.0, 1, st)
    with pytest.raises(fvm.UnstableTimestep):
        fvm.fvm_run(g, f, grid, 2.0 * limit, 1, st)
    other = gs.EdgeGrid(counts=grid.counts + 1, lengths=grid.lengths)
    with pytest.raises(ValueError):
        fvm.fvm_run(g, f, other, dt, 1, st)
    g0, f0 = build("star4_mixed", gs)  # a zero jump weight at the hub
    grid0 = gs.EdgeGrid.uniform(g0, 4, lengths=[0.5] * 4)
    with pytest.raises(fvm.ZeroJumpWeightAtVertex):
        fvm.stability_limit(g0, f0, grid0)


def test_state_helpers():
    g, f, grid, rho0, *_ = setup("path3")
    st = fvm.FvmState.uniform(grid, mass=2.0)
    assert abs(st.mass() - 2.0) < 1e-15
    bump = fvm.FvmState.from_function(grid, lambda e, x: 1.0 + 0.5 * np.sin(3.0 * x + e))
    assert np.array_equal(bump.rho, rho0)
    assert np.array_equal(bump.edge_density(1), rho0[3:])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_stepper_bitwise_vs_reference(name):
    g, f, grid, rho0, dt, steps, neg, _ = setup(name)
    rho, n = fvm.fvm_steps_device(g, f, grid, rho0, steps, dt)
    assert n == neg
    assert np.array_equal(rho, GOLD[f"{name}/rho"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_fvm_run_matches_reference_run(name):
    g, f, grid, rho0, dt, steps, neg, _ = setup(name)
    err = str(GOLD[f"{name}/run_error"])
    st = fvm.FvmState(grid=grid, rho=rho0.copy())
    force = FVM_CASES[name]["cfl"] > 1.0
    if err:
        kind = err.split(":")[0]
        with pytest.raises(getattr(fvm, kind)) as ei:
            fvm.fvm_run(g, f, grid, dt, steps, st, force=force)
        assert str(ei.value) == err.split(": ", 1)[1]
    else:
        res = fvm.fvm_run(g, f, grid, dt, steps, st, force=force)
        run = GOLD[f"{name}/run"]
        assert res.max_cfl == run[0] and res.state.t == run[1]
        assert np.array_equal(res.state.rho, run[2:])


@pytest.mark.gpu
def test_gpu_vs_oracle_vascular_grid():
    """A 400-node vascular-style network, ragged grid (1..4 cells per edge)."""
    from oracle import oracle

    text = open(os.path.join(HERE, "golden", "vascular_small.graph")).read()
    g, f = gs.parse_graph_file(text)
    rng = np.random.default_rng(3)
    counts = rng.integers(1, 5, g.n_edges)
    grid = gs.EdgeGrid(counts=counts, lengths=g.edge_length)
    dt = 0.9 * fvm.stability_limit(g, f, grid)
    rho0 = rng.random(grid.n_cells)
    p = fvm._pack(g, f, grid)
    assert p.vser.size > 0
    ref, n_ref = oracle.fvm_steps(rho0, 500, dt, p.reference_tuple())
    got, n = fvm.fvm_steps_device(g, f, grid, rho0, 500, dt)
    assert n == n_ref == 0
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_gpu_mass_conservation_and_two_edge_reduction():
    """SPEC fvm-baseline laws: mass drift <= 1e-12 relative per step on a
    closed graph; two identical edges with uniform weights behave like one
    interval of twice the length (agreement 1e-10)."""
    g, f, grid, rho0, dt, steps, _, _ = setup("general_ragged")
    st = fvm.FvmState(grid=grid, rho=rho0.copy())
    m0 = st.mass()
    res = fvm.fvm_run(g, f, grid, dt, steps, st)
    assert abs(res.state.mass() - m0) <= 1e-12 * steps * m0
    # two identical edges 1 -> 0 <- 2 (vertex 0 in the middle) vs one interval
    L, n, D = 1.0, 16, 0.5
    g2 = gs.build_graph([(1, 0, L), (2, 0, L)])
    f2 = gs.CoefficientField.for_graph(g2, [gs.ConstantDrift(0.0)] * 2, [1.0, 1.0])
    grid2 = gs.EdgeGrid.uniform(g2, n)
    g1 = gs.build_graph([(0, 1, 2 * L)])
    f1 = gs.CoefficientField.for_graph(g1, [gs.ConstantDrift(0.0)], [1.0])
    grid1 = gs.EdgeGrid.uniform(g1, 2 * n)
    x = (np.arange(2 * n) + 0.5) * (L / n)
    rho1 = 1.0 + 0.5 * np.cos(np.pi * x / (2 * L)) ** 2
    rho2 = rho1.copy()  # edge 1->0 = left half (x increasing towards 0), edge 2->0 mirrored
    rho2[n:] = rho1[n:][::-1]
    dt1 = 0.5 * min(fvm.stability_limit(g1, f1, grid1), fvm.stability_limit(g2, f2, grid2))
    r1 = fvm.fvm_run(g1, f1, grid1, dt1, 400, fvm.FvmState(grid1, rho1)).state.rho
    r2 = fvm.fvm_run(g2, f2, grid2, dt1, 400, fvm.FvmState(grid2, rho2)).state.rho
    assert np.max(np.abs(r2[:n] - r1[:n])) < 1e-10
    assert np.max(np.abs(r2[n:][::-1] - r1[n:])) < 1e-10
    assert D > 0


@pytest.mark.gpu
def test_gpu_vs_oracle_high_degree_hub():
    """A 64-edge hub (one vertex of degree 64) with linear drifts: the per-slot
    exchange at a high-degree vertex, bit for bit against the C oracle."""
    from oracle import oracle

    g, f = build("hub64", gs)
    grid = gs.EdgeGrid.uniform(g, 5)
    dt = 0.8 * fvm.stability_limit(g, f, grid)
    rho0 = np.random.default_rng(9).random(grid.n_cells)
    p = fvm._pack(g, f, grid)
    ref, n_ref = oracle.fvm_steps(rho0, 300, dt, p.reference_tuple())
    got, n = fvm.fvm_steps_device(g, f, grid, rho0, 300, dt)
    assert n == n_ref == 0
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", ["hub8", "general_ragged", "star4_mixed_pos"])
def test_term_layout_is_a_permutation(name):
    """Every exchange term has exactly one writer row and one reader cell."""
    g, f, grid, *_ = setup(name)
    p = fvm._pack(g, f, grid)
    assert p.tstart[0] == 0 and p.tstart[-1] == p.n_terms
    assert np.all(np.diff(p.tstart) >= 0)
    written = np.sort(p.rpos)
    assert np.array_equal(written, np.arange(p.n_terms))  # each position written once
    # a cell of degree-n vertex receives: its n-1 own exports if active, one share of every
    # other active row, and one term per diffusion pair it belongs to (n-1)
    for t, sl in enumerate(p.pslot):
        v = p.slot_vertex[sl]
        lo, hi = p.v_off[v], p.v_off[v + 1]
        n = hi - lo
        active = (p.v_speed_in[lo:hi] > 0) & (1.0 - p.v_b[lo:hi] > 0)
        k = sl - lo
        want = (n - 1) * active[k] + (active.sum() - active[k]) + (n - 1)
        assert p.tstart[t + 1] - p.tstart[t] == want


@pytest.mark.gpu
def test_gpu_vs_oracle_multiblock_path():
    """A grid above the single-block threshold (two kernels per step, CUDA-graph
    replay, stop test in the last block): bit for bit against the oracle, and a
    forced-unstable run stops at the oracle's step."""
    from oracle import oracle

    text = open(os.path.join(HERE, "golden", "vascular_small.graph")).read()
    g, f = gs.parse_graph_file(text)
    rng = np.random.default_rng(4)
    grid = gs.EdgeGrid(counts=rng.integers(30, 60, g.n_edges), lengths=g.edge_length)
    p = fvm._pack(g, f, grid)
    assert p.pslot.size + grid.n_cells > 16384  # csrc/gsde_fvm.cu kSmallItems
    dt = 0.9 * fvm.stability_limit(g, f, grid)
    rho0 = rng.random(grid.n_cells)
    ref, n_ref = oracle.fvm_steps(rho0, 150, dt, p.reference_tuple())
    got, n = fvm.fvm_steps_device(g, f, grid, rho0, 150, dt)
    assert n == n_ref == 0
    assert np.array_equal(got, ref)
    ref, n_ref = oracle.fvm_steps(rho0, 150, 4.0 * dt, p.reference_tuple())
    got, n = fvm.fvm_steps_device(g, f, grid, rho0, 150, 4.0 * dt)
    assert n_ref > 0 and n == n_ref
    assert np.array_equal(got, ref)
