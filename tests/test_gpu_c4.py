"""C4 -- the ~1.02e5-edge synthetic vascular network -- at its real scale on
the GPU:

* reference stream: run_ensemble on the real C4 graph equals the reference's
  own run (tests/golden/c4.npz, 2e4 particles x 100 steps) -- edge ids,
  crossings, crossing events and M histogram exact, positions to 1e-10;
* the production L2-table kernel under the reference's injected draws,
  recorded per step for 1024 particles (chained state-in single steps) and
  over whole runs for 2e4 particles: the reference's edge ids, M and draw
  counters (divergences only at FP32 near-ties of the reference's decisions);
* native stream vs reference stream at 1e9 particle-steps each: two-sample
  chi-square on the 2-cells-per-edge snapshot histogram (2.04e5 cells) and on
  final-edge occupancy, and crossings per particle-step within 4 sigma.
"""

import numpy as np
import pytest
import torch

import golden_io
import helpers
import paper_2512_02175_b200 as gs
from oracle import oracle
from paper_2512_02175_b200 import engine

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _golden():
    return np.load(golden_io.GOLDEN + "/c4.npz")


def _c4():
    g, f = helpers.vascular_c4()
    assert helpers.graph_digest(g, f) == str(_golden()["digest"][0])
    return g, f


def test_reference_stream_c4_matches_reference_run():
    g, f = _c4()
    d = _golden()
    n, steps, seed = (int(v) for v in d["meta"])
    cfg = gs.SimulationConfig(dt=float(d["dt"][0]), n_steps=steps, n_particles=n, seed=seed,
                              initial=gs.PerEdgeUniform(float(g.edge_length.max())),
                              rng="reference")
    r = gs.run_ensemble(g, f, cfg)
    np.testing.assert_array_equal(r.edges, d["edges"])
    np.testing.assert_array_equal(r.crossings, d["crossings"])
    np.testing.assert_array_equal(r.crossing_events, d["crossing_events"])
    np.testing.assert_array_equal(r.stats.m_histogram, d["m_histogram"])
    assert [r.stats.truncation_count, r.stats.crossings_total,
            r.stats.crossing_events] == d["stats"].tolist()
    assert r.stats.gamma == float(d["gamma"][0])
    helpers.assert_positions(r.positions, d["positions"])


def test_native_kernel_injected_draws_c4_whole_runs():
    """2e4 particles x 100 steps through the production L2 kernel with the
    reference's draws vs the oracle: every particle whose trajectory differs
    must pass an FP32 near-tie at its first divergent step (oracle traces)."""
    g, f = _c4()
    n, steps, dt, seed = 20_000, 100, 1e-3, 20251202
    xmax = float(g.edge_length.max())
    og = oracle.OracleGraph(g, f)
    o = oracle.ensemble(og, seed, n, steps, dt, (1, 0, 0.0, xmax))
    raw, nrm = oracle.fill_draws(seed, n, 1200)
    cfg = gs.SimulationConfig(dt=dt, n_steps=steps, n_particles=n, seed=seed,
                              initial=gs.PerEdgeUniform(xmax))
    out = engine.ensemble_device(g, f, cfg, inject=(torch.as_tensor(raw.view(np.int64)).to(DEV),
                                                    torch.as_tensor(nrm).to(DEV)),
                                 precision="native")
    assert int(out["totals"][3]) == 0
    e, c = out["edge"].cpu().numpy(), out["crossings"].cpu().numpy()
    same = (e == o["edges"]) & (c == o["crossings"])
    bad = np.flatnonzero(~same)
    print(f"C4 production kernel, injected draws: {same.sum()}/{n} particles with the "
          f"reference's final edge and crossing count")
    if bad.size:
        tr = oracle.trace(og, seed, int(bad.max()) + 1, steps, dt, (1, 0, 0.0, xmax))
        m = tr["margin"][bad].min(axis=1)
        print("  min FP64 decision margins of the differing particles:", np.sort(m)[:10])
        assert np.all(m < 2e-5), m
    assert same.mean() >= 0.995


def test_native_vs_reference_stream_c4_1e9_psteps():
    g, f = _c4()
    n, steps = 10_000_000, 100  # 1e9 particle-steps per stream
    grid = gs.EdgeGrid.uniform(g, 2)
    xmax = float(g.edge_length.max())
    mk = lambda rng, seed: gs.SimulationConfig(dt=1e-3, n_steps=steps, n_particles=n, seed=seed,
                                               initial=gs.PerEdgeUniform(xmax), rng=rng)
    a = engine.ensemble_device(g, f, mk("native", 1), outputs=("edge_counts",), grid=grid)
    b = engine.ensemble_device(g, f, mk("reference", 2), outputs=("edge_counts",), grid=grid)
    for key in ("hist", "edge_counts"):
        p, chi2, dof = helpers.chi2_two_sample(a[key].cpu().numpy(), b[key].cpu().numpy())
        print(f"C4 native vs reference stream, {key}: chi2 {chi2:.0f} / {dof} dof, p = {p:.3g}")
        assert p > 1e-4, (key, p, chi2, dof)
    ca, cb = int(a["totals"][0]), int(b["totals"][0])
    z = (ca - cb) / np.sqrt(ca + cb)  # Poisson-ish bound on the crossing-count difference
    print(f"crossings per particle-step: native {ca / (n * steps):.6f}, "
          f"reference {cb / (n * steps):.6f} (z = {z:.2f})")
    assert abs(z) < 4.0 * np.sqrt(2.0), z  # M per step is overdispersed (~x2 variance)
