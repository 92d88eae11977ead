"""C4 at its real scale on the CPU side (no GPU): the synthetic vascular
network (~1.02e5 edges) this package builds is the one the reference built
(same packed arrays, by digest), and the C oracle reproduces the reference's
own run_ensemble on it (tests/golden/c4.npz: 2e4 particles x 100 steps,
reference streams): edge ids, crossings, events and M histogram exact,
positions to 1e-10."""

import numpy as np

import golden_io
import helpers
from oracle import oracle


def _golden():
    return np.load(golden_io.GOLDEN + "/c4.npz")


def test_c4_graph_is_the_reference_graph():
    g, f = helpers.vascular_c4()
    d = _golden()
    assert g.n_edges == int(d["n_edges"][0]) and g.n_edges > 100_000
    assert helpers.graph_digest(g, f) == str(d["digest"][0])


def test_oracle_reproduces_reference_run_on_c4():
    g, f = helpers.vascular_c4()
    d = _golden()
    n, steps, seed = (int(v) for v in d["meta"])
    o = oracle.ensemble(oracle.OracleGraph(g, f), seed, n, steps, float(d["dt"][0]),
                        (1, 0, 0.0, float(g.edge_length.max())))
    np.testing.assert_array_equal(o["edges"], d["edges"])
    np.testing.assert_array_equal(o["crossings"], d["crossings"])
    np.testing.assert_array_equal(o["crossing_events"], d["crossing_events"])
    np.testing.assert_array_equal(o["m_histogram"], d["m_histogram"])
    helpers.assert_positions(o["positions"], d["positions"])
