"""Host-side mirror of the reference API (CPU only): graph packing, errors,
coefficients, grids, graph files -- checked against the reference's own
outputs (tests/golden/graphs.npz) and SPEC examples."""

import math

import numpy as np
import pytest

import cases
import golden_io
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import coefficients, engine, graphfile, workloads
from paper_2512_02175_b200.graph import INFINITY_VERTEX


def _built(case):
    if case == "vascular_small":
        return gs.parse_graph_file(golden_io.vascular_small_text())
    return cases.build(case, gs)


@pytest.mark.parametrize("case", list(cases.CASES) + ["vascular_small"])
def test_packed_graph_matches_reference(case):
    g, f = _built(case)
    ref = golden_io.load_npz_groups("graphs.npz")[case]
    for k in ("edge_init", "edge_term", "edge_length", "v_off", "v_edges", "v_orient", "v_cumw"):
        np.testing.assert_array_equal(getattr(g, k), ref[k], err_msg=k)
        assert getattr(g, k).dtype == ref[k].dtype, k
    assert g.is_star == bool(ref["is_star"][0])
    for k, a in zip(("dkind", "dcoef", "tab_off", "tab_x", "tab_mu", "sigma"), f.packed()):
        np.testing.assert_array_equal(a, ref[k], err_msg=k)
    assert coefficients.graph_gamma(f, g, 1e-3) == ref["graph_gamma"][0]


def test_v_thresh_exact_inverse_cdf():
    g, _ = cases.build("star4_mixed", gs)
    t = g.v_thresh
    rng = np.random.default_rng(0)
    for r in rng.integers(0, 2**63, 20000, dtype=np.int64).astype(np.uint64) * np.uint64(2):
        n53 = int(r) >> 11
        u = n53 * 2.0**-53
        slot_f = next((j for j in range(4) if u <= g.v_cumw[j]), 3)
        slot_i = next((j for j in range(4) if n53 <= int(t[j])), 3)
        assert slot_f == slot_i


def test_spec_examples_graph():
    g = gs.build_graph([(0, None, math.inf)] * 5, {0: [0.2] * 5})
    assert g.is_star
    g1 = gs.build_graph([(0, 1, 1.0)])
    assert list(g1.incidence[0].jump_weights) == [1.0]
    assert list(g1.incidence[1].jump_weights) == [1.0]
    with pytest.raises(gs.WeightSimplexViolation):
        gs.build_graph([(0, 1, 1.0), (0, 2, 1.0)], {0: [0.5, 0.6]})
    with pytest.raises(gs.NonPositiveLength):
        gs.build_graph([(0, 1, 0.0)])
    with pytest.raises(gs.NonPositiveLength):
        gs.build_graph([(0, 1, float("nan"))])
    with pytest.raises(gs.SelfLoopError):
        gs.build_graph([(0, 0, 1.0)])
    with pytest.raises(gs.DanglingVertexReference):
        gs.build_graph([(0, 2, 1.0)])
    with pytest.raises(gs.DanglingVertexReference):
        gs.build_graph([(0, 1, 1.0)], {5: [1.0]})
    with pytest.raises(gs.DisconnectedGraph):
        gs.build_graph([(0, 1, 1.0), (2, 3, 1.0)])
    with pytest.raises(gs.GraphBuildError):
        gs.build_graph([(0, None, 1.0)])
    with pytest.raises(gs.GraphBuildError):
        gs.build_graph([])
    with pytest.raises(gs.WeightSimplexViolation):
        gs.build_graph([(0, 1, 1.0), (0, 2, 1.0)], {0: [1.0]})


def test_sample_exit_edge_spec():
    for row in golden_io.load_json("solvers.json")["sample_exit_edge"]:
        if row["graph"] == "star5":
            g, _ = cases.build("star5_linear", gs)
        else:
            g = gs.build_graph([(0, 1, 1.0), (0, 2, 1.0)], {0: [0.1, 0.9]})
        assert list(gs.sample_exit_edge(g, row["v"], row["u"])) == row["out"]
    g, _ = cases.build("star5_linear", gs)
    with pytest.raises(gs.InfinityVertex):
        gs.sample_exit_edge(g, INFINITY_VERTEX, 0.5)


def test_gamma_and_coefficients():
    for row in golden_io.load_json("solvers.json")["gamma"]:
        g, f = cases.build(row["case"], gs)
        assert gs.gamma(f, g, row["v"], row["dt"]) == row["gamma"]
        assert coefficients.graph_gamma(f, g, row["dt"]) == row["graph_gamma"]
    f = gs.drift_from_flux([2.0, 0.0], [0.5, 1.0])
    assert f == [gs.ConstantDrift(4.0), gs.ConstantDrift(0.0)]
    with pytest.raises(gs.NonPositiveArea):
        gs.drift_from_flux([1.0], [0.0])
    with pytest.raises(gs.ZeroDiffusion):
        gs.ConstantDiffusion(0.0)
    with pytest.raises(gs.CoefficientError):
        gs.TabulatedDrift((0.0, 0.0), (1.0, 2.0))
    g, _ = cases.build("star5_quad", gs)
    fq = gs.CoefficientField.for_graph(g, [gs.LinearDrift(-10.0 * i) for i in range(1, 6)], [1.0] * 5)
    assert gs.eval_drift(fq, 2, 0.5) == -15.0
    ft = gs.CoefficientField.for_graph(g, [gs.TabulatedDrift((0.0, 1.0), (0.0, 2.0))] * 5, [1.0] * 5)
    assert gs.eval_drift(ft, 0, 0.25) == 0.5


def test_solve_alpha_spec():
    for row in golden_io.load_json("solvers.json")["solve_alpha"]:
        if row["alpha"] is None:
            with pytest.raises(gs.NoRootInUnitInterval):
                gs.solve_alpha(row["a"], row["b"], row["c"])
        else:
            assert gs.solve_alpha(row["a"], row["b"], row["c"]) == row["alpha"]


def test_config_validation():
    g, _ = cases.build("star3_bm", gs)
    ok = gs.SimulationConfig(dt=1e-3, n_steps=1, n_particles=1, seed=1)
    assert ok.validated(g) is ok
    bad = [
        dict(dt=0.0), dict(dt=float("inf")), dict(n_steps=-1), dict(max_splits_per_step=0),
        dict(workers=0), dict(reflect_at=-1.0), dict(initial=gs.AtVertex(3)),
        dict(initial=gs.PointStart(7, 0.0)), dict(initial=gs.PerEdgeUniform(float("inf"))),
        dict(rng="fast"),
    ]
    for kw in bad:
        args = dict(dt=1e-3, n_steps=1, n_particles=1, seed=1)
        args.update(kw)
        with pytest.raises(gs.ConfigInvalid):
            gs.SimulationConfig(**args).validated(g)


def test_run_ensemble_shape_errors_before_dispatch():
    g, f = cases.build("star3_bm", gs)
    with pytest.raises(gs.ConfigInvalid):
        gs.run_ensemble(g, f, gs.SimulationConfig(dt=-1.0, n_steps=1, n_particles=1, seed=1))
    gp, fp = cases.build("path3", gs)
    with pytest.raises(gs.ConfigInvalid):
        gs.run_ensemble(gp, fp, gs.SimulationConfig(dt=1e-3, n_steps=1, n_particles=1, seed=1,
                                                    reflect_at=0.5))
    # n_particles = 0 needs no device
    r = gs.run_ensemble(g, f, gs.SimulationConfig(dt=1e-3, n_steps=10, n_particles=0, seed=1))
    assert r.edges.shape == (0,) and r.stats.m_histogram.shape == (101,)
    with pytest.raises(gs.ConfigInvalid):
        gs.vertex_crossing_trials(g, f, 0.0, 10, 1)


def test_rng_stream_matches_reference_grid():
    for row in golden_io.load_json("rng.json")["raw64_grid"][:60]:
        s, st, k = int(row["seed"]), int(row["stream"]), int(row["index"])
        assert gs.rng.raw64(s, st, k) == int(row["raw"])
        assert gs.rng.uniform01(s, st, k) == row["uniform"]
        assert abs(gs.rng.normal(s, st, k) - row["normal"]) <= 1e-15 + 1e-14 * abs(row["normal"])
    rs = gs.RngStream(7, 3, 10)
    rs.normal()
    rs.uniform()
    assert rs.counter == 12


def test_graphfile_roundtrip_and_errors():
    g, f = gs.parse_graph_file(golden_io.vascular_small_text())
    text = gs.serialize_graph_file(g, f)
    g2, f2 = gs.parse_graph_file(text)
    np.testing.assert_array_equal(g.v_cumw, g2.v_cumw)
    np.testing.assert_array_equal(g.edge_length, g2.edge_length)
    assert [d.c for d in f.drift] == [d.c for d in f2.drift]
    with pytest.raises(gs.ParseError) as ei:
        gs.parse_graph_file("metric-graph v1\nedge 0 0 inf inf\nweights inf 1.0\n")
    assert ei.value.line == 3
    with pytest.raises(gs.ParseError) as ei:
        gs.parse_graph_file("metric-graph v1\nedge 0 0 1 1.0\ndrift 0 from_flux 1.0 0.0\n")
    assert ei.value.line == 3 and "NonPositiveArea" in str(ei.value)
    with pytest.raises(gs.ParseError):
        gs.parse_graph_file("not a header\n")


def test_edge_grid():
    g, _ = cases.build("hub8", gs)
    grid = gs.EdgeGrid.uniform(g, 4)
    assert grid.n_cells == 32
    np.testing.assert_array_equal(grid.offsets, np.arange(9) * 4)
    with pytest.raises(ValueError):
        gs.EdgeGrid.uniform(cases.build("star3_bm", gs)[0], 4)


def test_workloads_deterministic():
    g1, f1 = workloads.hub64()
    assert not g1.is_star and g1.n_edges == 64
    t1 = workloads.vascular_text(300, 5)
    t2 = workloads.vascular_text(300, 5)
    assert t1 == t2
    g, f = gs.parse_graph_file(t1)
    assert g.n_edges >= g.n_vertices - 1


def _same_graph(a, b):
    (g1, f1), (g2, f2) = a, b
    for k in ("edge_init", "edge_term", "edge_length", "v_off", "v_edges", "v_orient", "v_cumw"):
        np.testing.assert_array_equal(getattr(g1, k), getattr(g2, k), err_msg=k)
    assert g1.is_star == g2.is_star
    for x, y in zip(f1.packed(), f2.packed()):
        np.testing.assert_array_equal(x, y)
    assert f1.drift == f2.drift and f1.diffusion == f2.diffusion


@pytest.mark.parametrize("case", list(cases.CASES) + ["vascular_small"])
def test_native_graph_reader_matches_python_reader(case):
    g, f = _built(case)
    text = gs.serialize_graph_file(g, f)
    fast = graphfile._parse_native(text)
    assert fast is not None, "native reader should accept serialized files"
    _same_graph(fast, graphfile._parse_python(text))


BAD_DOCS = [
    "",
    "metric-graph  v1\nedge 0 0 1 1.0\n",                  # header spacing
    "metric-graph v1\nedge 0 0 1\n",                         # arity
    "metric-graph v1\nedge 0 0 1 1.0\nedge 0 1 2 1.0\n",     # duplicate id
    "metric-graph v1\nedge 1 0 1 1.0\n",                     # ids not dense
    "metric-graph v1\nedge 0 0 1 -1.0\n",                    # NonPositiveLength
    "metric-graph v1\nedge 0 0 0 1.0\n",                     # self loop
    "metric-graph v1\nedge 0 0 inf inf\nweights inf 1.0\n",  # weights at infinity
    "metric-graph v1\nedge 0 0 1 1.0\ndrift 0 from_flux 1.0 0.0\n",
    "metric-graph v1\nedge 0 0 1 1.0\ndrift 0 tabulated 0.5:1 0.2:3\n",
    "metric-graph v1\nedge 0 0 1 1.0\ndrift 0 tabulated 0.5:1 2.0:3\n",  # beyond edge
    "metric-graph v1\nedge 0 0 1 1.0\nsigma 0 0.0\n",        # ZeroDiffusion
    "metric-graph v1\nvertex 0\nedge 0 0 1 1.0\n",           # undeclared vertex 1
    "metric-graph v1\nedge 0 0 1 1.0\nweights 0 0.5 0.5\n",  # weight arity
    "metric-graph v1\nedge 0 0 1 1.0\nfoo 1\n",              # unknown directive
    "metric-graph v1\nedge 0 0 1 1_0.0\n",                   # python-only number syntax
    "metric-graph v1\nedge 0 0 1 0x1p3\n",                   # hex float (python rejects)
    "metric-graph v1\nedge 0 0 1 1.0\x0bedge 1 1 2 1.0\n",   # \v is a line break in python
]


@pytest.mark.parametrize("doc", BAD_DOCS)
def test_reader_errors_and_fallbacks_are_the_python_readers(doc):
    try:
        want = graphfile._parse_python(doc)
    except gs.ParseError as err:
        with pytest.raises(gs.ParseError) as got:
            gs.parse_graph_file(doc)
        assert (got.value.line, str(got.value)) == (err.line, str(err))
    else:
        _same_graph(gs.parse_graph_file(doc), want)
