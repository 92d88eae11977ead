"""Pin the C oracle against the reference's own outputs (CPU, no GPU).

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Integer outputs (edge ids, crossing counts,
draw counters, M histograms, truncations, histograms) must match exactly.
Doubles: the reference is numba ``fastmath=True`` (LLVM contracts/reassociates
the AS241 polynomials and the EM update), the oracle strict IEEE C, so single
steps agree to a few ulp and whole trajectories (hundreds of steps) to
POS_ATOL = 1e-10 absolute (measured max 8e-12).
"""

import numpy as np
import pytest

import cases
import golden_io
import paper_2512_02175_b200 as gs
from oracle import oracle

RTOL = 1e-12
POS_ATOL = 1e-10


def close(a, b, rtol=RTOL, atol=1e-300):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    same_nan = np.isnan(a) & np.isnan(b)
    return np.all((a == b) | same_nan | (np.abs(a - b) <= rtol * np.maximum(np.abs(a), np.abs(b)) + atol))


RANDOM123_KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,out", RANDOM123_KAT)
def test_philox_random123_kat(ctr, key, out):
    assert oracle.philox4x32_10(ctr, key) == out


def test_philox_matches_reference_kat():
    for row in golden_io.load_json("rng.json")["philox_kat"]:
        assert oracle.philox4x32_10(row["ctr"], row["key"]) == row["out"]


def test_raw64_uniform_normal_grid():
    for row in golden_io.load_json("rng.json")["raw64_grid"]:
        s, st, k = int(row["seed"]), int(row["stream"]), int(row["index"])
        r = oracle.raw64(s, st, k)
        assert r == int(row["raw"])
        assert oracle.uniform01(s, st, k) == row["uniform"]
        # numba fastmath may skip the rounding of p = (n + 0.5) 2^-53 when the
        # scalar entry point is compiled standalone: allow one ulp of p.
        assert close(oracle.normal(s, st, k), row["normal"], 1e-14, 1e-15)


def test_norm_ppf_values():
    data = golden_io.load_json("rng.json")
    for row in data["norm_ppf"]:
        assert close(oracle.norm_ppf(row["p"]), row["value"], 1e-14), row
    for row in data["normal_extremes"]:
        r = int(row["raw"])
        v = oracle.lib().orc_u64_to_normal(r)
        # incl. the top lattice points: the reference's fastmath build forms
        # min(p, 1-p) above the median as (2^53 - n) 2^-53, and so does the oracle
        assert close(v, row["normal"], 1e-14, 1e-15), row


def test_first_passage_vectors():
    for row in golden_io.load_json("solvers.json")["first_passage"]:
        s = oracle.solve_first_passage_s(row["a"], row["b"], row["c"])
        assert close(s, row["s"], 1e-13, 1e-300), row


STEP_CASES = list(cases.CASES)


@pytest.mark.parametrize("case", STEP_CASES)
def test_step_tuples(case):
    g, f = cases.build(case, gs)
    og = oracle.OracleGraph(g, f)
    d = golden_io.load_npz_groups("steps.npz")[case]
    for i in range(d["edge"].shape[0]):
        e, x, M, tr, k = oracle.step(og, int(d["edge"][i]), float(d["x"][i]), float(d["dt"][i]),
                                     int(d["seed"][i]), int(d["pid"][i]), int(d["k"][i]),
                                     int(d["cap"][i]), float(d["refl"][i]))
        assert e == d["o_edge"][i] and M == d["o_M"][i] and tr == d["o_trunc"][i], (case, i)
        assert k == int(d["o_k"][i]), (case, i)
        assert close(x, d["o_x"][i], RTOL, 1e-14), (case, i, x, d["o_x"][i])


def _init_tuple(init, graph):
    kind = init[0]
    if kind == "at":
        v = init[1]
        lo = int(graph.v_off[v])
        e = int(graph.v_edges[lo])
        x = graph.vertex_position(e, int(graph.v_orient[lo]))
        return (0, e, x, 0.0)
    if kind == "point":
        return (0, init[1], init[2], 0.0)
    return (1, 0, 0.0, float(init[1]))


def _graph_for(m):
    if m["case"] == "vascular_small":
        return gs.parse_graph_file(golden_io.vascular_small_text())
    return cases.build(m["case"], gs)


@pytest.mark.parametrize("m", golden_io.meta()["ensembles"], ids=lambda m: m["name"])
def test_ensembles(m):
    g, f = _graph_for(m)
    d = golden_io.load_npz_groups("ensembles.npz")[m["name"]]
    og = oracle.OracleGraph(g, f)
    out = oracle.ensemble(og, m["seed"], m["n"], m["steps"], m["dt"], _init_tuple(m["init"], g),
                          m["cap"], m["reflect"])
    np.testing.assert_array_equal(out["edges"], d["edges"])
    np.testing.assert_array_equal(out["crossings"], d["crossings"])
    np.testing.assert_array_equal(out["crossing_events"], d["crossing_events"])
    np.testing.assert_array_equal(out["m_histogram"], d["m_histogram"])
    assert int(out["truncs"].sum()) == int(d["stats"][0])
    assert close(out["positions"], d["positions"], 0.0, POS_ATOL)


@pytest.mark.parametrize("m", golden_io.meta()["trials"], ids=lambda m: m["name"])
def test_trials(m):
    g, f = cases.build(m["case"], gs)
    d = golden_io.load_npz_groups("trials.npz")[m["name"]]
    og = oracle.OracleGraph(g, f)
    lo = int(g.v_off[m["vertex"]])
    e0 = int(g.v_edges[lo])
    x0 = g.vertex_position(e0, int(g.v_orient[lo]))
    out = oracle.vertex_trials(og, m["seed"], m["n"], m["dt"], e0, x0, m["cap"])
    for k in ("M", "exit_edges", "truncated"):
        np.testing.assert_array_equal(out[k], d[k])
    assert close(out["exit_positions"], d["exit_positions"], 0.0, POS_ATOL)


def test_histogram_star3():
    st = golden_io.meta()["stats"]["hist_star3"]
    d = golden_io.load_npz_groups("ensembles.npz")["c1_star3_bm"]
    counts = np.full(3, st["cells"], np.int64)
    lengths = np.asarray(st["lengths"])
    offsets = np.concatenate([[0], np.cumsum(counts)])
    h = oracle.histogram(d["edges"], d["positions"], offsets, counts, lengths / counts)
    np.testing.assert_array_equal(h, st["counts"])
