"""Host-side validators and the drop-in namespace, pinned to vectors the
REFERENCE produced (tests/golden/make_validator_golden.py, make_golden.py):

* SteadyStateOracle: B, D, closed-form / printed normalisers, self_check,
  masses, densities, truncation lengths (analysis.py:82-206);
* l2_error of a Histogram, an FvmState, raw arrays and a callable
  (analysis.py:224-245);
* crossing_bound at 40 (k, gamma) points and check_crossing_bound reports,
  including the reference's own report on 2e5 vertex trials
  (analysis.py:275-319);
* rng.u64_to_uniform / u64_to_normal / norm_ppf (rng.py:69-143);
* every public name of every reference module exists here.

No GPU: these are host computations (the rng scalars evaluate the kernels'
__host__ __device__ code through libgsde.so).
"""

import importlib
import json
import os

import numpy as np
import pytest

import golden_io
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, engine, fvm, rng

HERE = os.path.dirname(os.path.abspath(__file__))
V = json.load(open(os.path.join(HERE, "golden", "validators.json")))
RTOL = 1e-13  # host float64 (scipy quad / brentq on the same integrands)


def close(a, b, rtol=RTOL, atol=0.0):
    np.testing.assert_allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=rtol,
                               atol=atol)


@pytest.mark.parametrize("mod", sorted(V["namespace"]))
def test_namespace_covers_reference(mod):
    ours = importlib.import_module(mod.replace("graphsde", "paper_2512_02175_b200"))
    missing = [n for n in V["namespace"][mod]["names"] if not hasattr(ours, n)]
    assert not missing, (mod, missing)


@pytest.mark.parametrize("i", range(len(V["steady_state"])))
def test_steady_state_oracle(i):
    r = V["steady_state"][i]
    if "from_field" in r:
        g = gs.build_graph([(0, None, float("inf"))] * 3)
        f = gs.CoefficientField.for_graph(g, [gs.LinearDrift(-2.0), gs.LinearDrift(-5.0),
                                              gs.LinearDrift(-9.0)], [1.3] * 3)
        o = analysis.SteadyStateOracle.from_field(g, f)
        assert o.kind == r["kind"]
        close(o.rates, r["rates"])
        close([o.B, o.D], [r["B"], r["D"]])
        return
    o = analysis.SteadyStateOracle.create(r["kind"], r["rates"], r["sigma"])
    close([o.B, o.D], [r["B"], r["D"]])
    close(o.closed_form_normalizer(), r["closed_form"])
    close(o.as_printed_normalizer(), r["as_printed"])
    sc = o.self_check()
    assert sc["kind"] == r["self_check"]["kind"]
    for k in ("quadrature_B", "closed_form_B", "as_printed_B", "total_mass"):
        close(sc[k], r["self_check"][k])
    n = len(r["rates"])
    close([o.edge_mass(e) for e in range(n)], r["edge_mass"])
    close([[o.tail_mass(e, L) for L in (0.0, 0.05, 0.5, 2.0)] for e in range(n)], r["tail_mass"],
          atol=1e-300)
    xs = np.array([0.0, 0.013, 0.1, 0.77, 3.0])
    close([np.atleast_1d(o.density(e, xs)) for e in range(n)], r["density"], atol=1e-300)
    close([float(analysis.steady_state_density(o, e, 0.25)) for e in range(n)],
          r["density_scalar"], atol=1e-300)
    close(o.truncation_lengths(1e-8), r["trunc_8"], rtol=1e-10)
    close(o.truncation_lengths(1e-4), r["trunc_4"], rtol=1e-10)


def test_steady_state_oracle_errors():
    with pytest.raises(ValueError):
        analysis.SteadyStateOracle.create("cubic", [1.0], 1.0)
    with pytest.raises(ValueError):
        analysis.SteadyStateOracle.create("linear", [1.0, 0.0], 1.0)
    g = gs.build_graph([(0, None, float("inf"))] * 2)
    for drift, sig, in (([gs.ConstantDrift(-1.0), gs.LinearDrift(-1.0)], [1.0, 1.0]),
                        ([gs.ConstantDrift(-1.0), gs.ConstantDrift(1.0)], [1.0, 1.0]),
                        ([gs.ConstantDrift(-1.0), gs.ConstantDrift(-1.0)], [1.0, 2.0])):
        with pytest.raises(gs.CoefficientError):
            analysis.SteadyStateOracle.from_field(g, gs.CoefficientField.for_graph(g, drift, sig))
    gp = gs.build_graph([(0, 1, 1.0)])
    with pytest.raises(gs.CoefficientError):
        analysis.SteadyStateOracle.from_field(
            gp, gs.CoefficientField.for_graph(gp, [gs.ConstantDrift(-1.0)], [1.0]))


def _grid(c):
    return gs.EdgeGrid(counts=np.full(len(c["lengths"]), c["cells"], np.int64),
                       lengths=np.array(c["lengths"]))


@pytest.mark.parametrize("i", range(len(V["l2"])))
def test_l2_error(i):
    c = V["l2"][i]
    grid = _grid(c)
    lin = analysis.SteadyStateOracle.create("linear", [10.0, 20.0, 30.0], 1.0)
    quad = analysis.SteadyStateOracle.create("quadratic", [10.0, 20.0, 30.0], 1.0)
    if c["kind"] == "histogram":
        est = analysis.Histogram(grid=grid, counts=np.array(c["counts"], np.int64),
                                 total=c["total"])
        got = analysis.l2_error(est, lin)
    elif c["kind"] == "fvm_state":
        got = analysis.l2_error(fvm.FvmState(grid=grid, rho=np.array(c["rho"]), t=0.5), lin)
    elif c["kind"] == "raw":
        got = analysis.l2_error(np.array(c["rho"]), lin, grid=grid)
    elif c["kind"] == "raw_quadratic":
        got = analysis.l2_error(np.array(c["rho"]), quad, grid=grid)
    else:
        got = analysis.l2_error(np.array(c["rho"]), lambda e, x: np.exp(-(e + 1) * x), grid=grid)
    close(got, c["l2"], rtol=1e-12)


def test_l2_error_mismatches():
    c = V["l2"][0]
    grid = _grid(c)
    lin = analysis.SteadyStateOracle.create("linear", [10.0, 20.0, 30.0], 1.0)
    rho = np.ones(grid.n_cells)
    with pytest.raises(analysis.GridMismatch):
        analysis.l2_error(rho, lin)  # raw array without a grid
    with pytest.raises(analysis.GridMismatch):
        analysis.l2_error(rho[:-1], lin, grid=grid)
    other = gs.EdgeGrid(counts=grid.counts, lengths=grid.lengths * 2.0)
    with pytest.raises(analysis.GridMismatch):
        analysis.l2_error(fvm.FvmState(grid=grid, rho=rho), lin, grid=other)


def test_crossing_bound_points():
    for row in golden_io.load_json("solvers.json")["crossing_bound"]:
        assert analysis.crossing_bound(row["k"], row["g"]) == pytest.approx(row["bound"],
                                                                            rel=1e-15, abs=0)


@pytest.mark.parametrize("i", range(len(V["crossing"])))
def test_check_crossing_bound_reports(i):
    c = V["crossing"][i]
    m = np.array(c["m_hist"], np.int64)
    b = engine.BounceStats(m_histogram=m, gamma=c["gamma0"], truncation_count=0,
                           crossings_total=int((m * np.arange(m.size)).sum()),
                           crossing_events=int(m.sum()))
    rep = analysis.check_crossing_bound(b, gamma=c["gamma"], k_max=c["k_max"],
                                        homogeneous=c["homogeneous"])
    assert rep.gamma == c["rep_gamma"] and rep.n_steps == c["n_steps"]
    assert rep.any_bound_violation == c["any_bound"] and rep.any_chi2_deviation == c["any_chi2"]
    assert len(rep.rows) == len(c["rows"])
    for r, g in zip(rep.rows, c["rows"]):
        assert r.k == g[0] and r.bound_violated == g[5] and r.chi2_deviates == g[6]
        close([r.empirical, r.bound, r.chi2_tail, r.std_error], g[1:5], rtol=1e-12)


def test_reference_crossing_report_on_its_trials():
    """The reference's own check_crossing_bound report of 2e5 vertex trials
    (make_golden.py: star_homog, dt 1e-3, seed 3), recomputed from its M
    histogram through this package's VertexTrials-free BounceStats path."""
    st = golden_io.meta()["stats"]["crossing_bound"]
    m = np.array(st["m_hist"], np.int64)
    b = engine.BounceStats(m_histogram=m, gamma=st["gamma"], truncation_count=0,
                           crossings_total=int((m * np.arange(m.size)).sum()),
                           crossing_events=int(m[1:].sum()))
    rep = analysis.check_crossing_bound(b)
    for r, g in zip(rep.rows, st["rows"]):
        assert r.k == g[0] and r.bound_violated == g[5] and r.chi2_deviates == g[6]
        close([r.empirical, r.bound, r.chi2_tail, r.std_error], g[1:5], rtol=1e-12)


def test_rng_scalar_functions():
    """Including the far upper tail: the reference's compiled u64_to_normal
    uses 1 - p = (2^53 - n) 2^-53 above the median (fastmath reassociation),
    which the kernels and the oracle restate -- the top lattice points give
    8.2095, 8.1259, 8.0766, ... (not the mirror of the lower tail)."""
    s = V["rng_scalars"]
    words = [int(w) for w in s["u64"]]
    assert [rng.u64_to_uniform(w) for w in words] == s["u64_to_uniform"]
    # ulp-level differences only (the reference's polynomials are FMA-contracted)
    close([rng.u64_to_normal(w) for w in words], s["u64_to_normal"], rtol=1e-15)
    close([rng.norm_ppf(p) for p in s["p"]], s["norm_ppf"], rtol=1e-15)


def test_available_workers():
    assert isinstance(engine.available_workers(), int) and engine.available_workers() >= 1
