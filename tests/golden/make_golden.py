"""Generate golden vectors by running the REFERENCE package in this container.

    python tests/golden/make_golden.py

Imports ``graphsde`` from /root/reference/pkg/src (read-only; numba cache
redirected to /tmp) and writes small fixtures next to this script.  The
fixtures pin the C oracle (tests/test_oracle_golden.py) and are compared with
the CUDA path directly (tests/test_gpu_parity.py).  /root/reference does not
exist on the GPU box; only the committed fixtures travel.
"""

from __future__ import annotations

import json
import math
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import graphsde as gs  # noqa: E402
from graphsde import analysis, engine, graphfile, kernels, rng  # noqa: E402
from graphsde.grids import EdgeGrid  # noqa: E402

from cases import CASES, build  # noqa: E402

U64 = (1 << 64) - 1


def rng_vectors():
    kats = [
        ([0, 0, 0, 0], [0, 0]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]),
    ]
    kat_out = []
    for ctr, key in kats:
        out = rng._philox4x32_10(*[np.uint32(c) for c in ctr], *[np.uint32(k) for k in key])
        kat_out.append(dict(ctr=ctr, key=key, out=[int(x) for x in out]))
    grid = []
    seeds = [0, 1, 20251202, 0xDEADBEEFCAFEF00D, U64]
    streams = [0, 1, 12345, (1 << 40) + 3, U64]
    idxs = [0, 1, 2, 3, 63, 64, 65, (1 << 33) + 1, U64 - 1, U64]
    for s in seeds:
        for st in streams:
            for k in idxs:
                r = int(rng.raw64(np.uint64(s), np.uint64(st), np.uint64(k)))
                grid.append(dict(seed=str(s), stream=str(st), index=str(k), raw=str(r),
                                 uniform=float(rng.u64_to_uniform(np.uint64(r))),
                                 normal=float(rng.u64_to_normal(np.uint64(r)))))
    ps = [1e-300, 1e-100, 1e-20, 1e-12, 1e-9, 2.5e-7, 1e-3, 0.02, 0.07, 0.075, 0.0751,
          0.3, 0.5, 0.5 + 1e-12, 0.924, 0.925, 0.93, 0.99, 1 - 1e-9, 1 - 2 ** -53]
    ppf = [dict(p=p, value=float(rng.norm_ppf(p))) for p in ps]
    # lattice extremes of u64_to_normal
    extremes = [dict(raw=str(r), normal=float(rng.u64_to_normal(np.uint64(r))))
                for r in (0, 1 << 11, (1 << 63), U64 - (1 << 11), U64)]
    return dict(philox_kat=kat_out, raw64_grid=grid, norm_ppf=ppf, normal_extremes=extremes)


def solver_vectors():
    r = np.random.default_rng(1)
    triples = []
    # fuzzed overshoot triples (c >= 0, a + b + c <= 0) + branch specials
    for _ in range(3000):
        c = float(r.exponential(0.5)) if r.random() > 0.05 else 0.0
        a = float(r.normal(0, 3)) if r.random() > 0.1 else 0.0
        b = float(-(a + c) - abs(r.normal(0, 2)))
        triples.append((a, b, c))
    specials = [(0.0, -2.0, 1.0), (-1.0, -1.0, 1.0), (-4.0, 0.0, 1.0), (1.0, -3.0, 1.0),
                (0.0, 1.0, 1.0), (2.0, 1.0, 0.0), (-2.0, 1.0, 0.0), (-2.0, 3.0, 0.0),
                (1.0, -1.0, -0.5), (0.0, 0.0, 1.0), (1e-300, -1.0, 1e-300), (3.0, -2.0, 0.5),
                (-1e-12, -1e-6, 1e-7), (5.0, -1.0, 1.0)]
    triples += specials
    fp = [dict(a=a, b=b, c=c, s=float(kernels.solve_first_passage_s(a, b, c)))
          for a, b, c in triples]
    alpha = []
    for a, b, c in [(0.0, -2.0, 1.0), (-1.0, -1.0, 1.0), (-4.0, 0.0, 1.0), (0.0, 1.0, 1.0)]:
        try:
            alpha.append(dict(a=a, b=b, c=c, alpha=engine.solve_alpha(a, b, c)))
        except engine.NoRootInUnitInterval:
            alpha.append(dict(a=a, b=b, c=c, alpha=None))
    g5, _ = build("star5_linear", gs)
    g2 = gs.build_graph([(0, 1, 1.0), (0, 2, 1.0)], {0: [0.1, 0.9]})
    exits = [dict(graph="star5", v=0, u=u, out=list(gs.sample_exit_edge(g5, 0, u)))
             for u in (0.0, 0.2, 0.2 + 1e-16, 0.55, 0.999999, 1.0)]
    exits += [dict(graph="w19", v=0, u=u, out=list(gs.sample_exit_edge(g2, 0, u)))
              for u in (0.1 - 1e-12, 0.1, 0.1 + 1e-12, 1.0 + 1e-9)]
    gam = []
    for case in ("star5_linear", "star5_quad", "star3_bm", "star4_mixed", "hub64", "path3",
                 "random_general"):
        g, f = build(case, gs)
        for dt in (1e-3, 0.37):
            gam.append(dict(case=case, dt=dt, v=0, gamma=gs.gamma(f, g, 0, dt),
                            graph_gamma=engine._graph_gamma(g, f, dt)))
    oracles = []
    rates = [10.0, 20.0, 30.0, 40.0, 50.0]
    for kind in ("linear", "quadratic"):
        o = analysis.SteadyStateOracle.create(kind, rates, 1.0)
        oracles.append(dict(kind=kind, rates=rates, B=o.B, D=o.D,
                            trunc=o.truncation_lengths(1e-8).tolist(),
                            dens=[float(o.density(e, 0.01 * (e + 1))) for e in range(5)]))
    bounds = [dict(k=k, g=g, bound=analysis.crossing_bound(k, g))
              for k in range(1, 11) for g in (0.0, 0.5, 2.5, 10.0)]
    return dict(first_passage=fp, solve_alpha=alpha, sample_exit_edge=exits, gamma=gam,
                steady_state=oracles, crossing_bound=bounds)


def step_vectors():
    out = {}
    r = np.random.default_rng(2)
    for case in CASES:
        g, f = build(case, gs)
        n = 400
        rows = []
        for _ in range(n):
            e = int(r.integers(0, g.n_edges))
            l = float(g.edge_length[e])
            u = r.random()
            if g.is_star:
                x = 0.0 if u < 0.3 else float(r.exponential(10 ** r.uniform(-3, -0.3)))
            else:
                x = 0.0 if u < 0.15 else (l if u < 0.3 else float(r.uniform(0, l)))
            dt = float(10 ** r.uniform(-4.5, -0.5))
            seed = int(r.integers(0, 2**63))
            pid = int(r.integers(0, 2**62))
            k = int(r.integers(0, 2**40))
            cap = int(r.choice([100, 100, 3, 1]))
            refl = float(r.choice([0.0, 0.0, 0.05])) if g.is_star else 0.0
            st = engine.ParticleState(edge=e, x=x)
            rs = gs.RngStream(seed, pid, k)
            if g.is_star:
                o = engine.em_step_star(g, f, st, dt, rs, max_splits=cap, reflect_at=refl)
            else:
                o = engine.em_step_general(g, f, st, dt, rs, max_splits=cap)
            rows.append((e, x, dt, seed, pid, k, cap, refl, o.state.edge, o.state.x,
                         o.crossings_this_step, int(o.truncated), rs.counter))
        a = list(zip(*rows))
        out[case] = dict(
            edge=np.array(a[0], np.int64), x=np.array(a[1]), dt=np.array(a[2]),
            seed=np.array(a[3], np.uint64), pid=np.array(a[4], np.uint64),
            k=np.array(a[5], np.uint64), cap=np.array(a[6], np.int64), refl=np.array(a[7]),
            o_edge=np.array(a[8], np.int64), o_x=np.array(a[9]), o_M=np.array(a[10], np.int64),
            o_trunc=np.array(a[11], np.int64), o_k=np.array(a[12], np.uint64),
        )
    return out


def _init(kind, *args):
    return {"at": gs.AtVertex, "point": gs.PointStart, "uniform": gs.PerEdgeUniform}[kind](*args)


ENSEMBLES = [
    # name, case, n, steps, dt, seed, init, cap, reflect
    ("c1_star3_bm", "star3_bm", 3000, 300, 1e-3, 20251202, ("at", 0), 100, 0.0),
    ("star3_drift_unif", "star3_drift", 2000, 150, 1e-3, 5, ("uniform", 0.5), 100, 0.0),
    ("star5_linear_point", "star5_linear", 2000, 200, 1e-4, 6, ("point", 2, 0.01), 100, 0.0),
    ("star5_quad_reflect", "star5_quad", 2000, 200, 1e-3, 7, ("at", 0), 100, 0.3),
    ("star4_mixed_cap3", "star4_mixed", 2000, 100, 1e-2, 8, ("uniform", 0.2), 3, 0.0),
    ("star_homog_cap5", "star_homog", 2000, 100, 1e-3, 9, ("at", 0), 5, 0.0),
    ("hub64_unif", "hub64", 3000, 200, 1e-3, 10, ("uniform", 2.0), 100, 0.0),
    ("hub8_at3", "hub8", 2000, 200, 1e-2, 11, ("at", 3), 100, 0.0),
    ("path3_point", "path3", 2000, 200, 5e-3, 12, ("point", 1, 0.5), 100, 0.0),
    ("single_edge_at0", "single_edge", 2000, 300, 1e-3, 13, ("at", 0), 100, 0.0),
    ("cycle3_cap4", "cycle3", 2000, 100, 1e-2, 14, ("at", 1), 4, 0.0),
    ("random_general_unif", "random_general", 3000, 200, 2e-3, 15, ("uniform", 1.0), 10, 0.0),
    ("star3_drift_zero_steps", "star3_drift", 1000, 0, 1e-3, 16, ("uniform", 0.5), 100, 0.0),
    ("hub8_zero_particles", "hub8", 0, 10, 1e-3, 17, ("at", 0), 100, 0.0),
    ("ragged_4097", "star5_quad", 4097, 20, 1e-3, 18, ("uniform", 0.3), 100, 0.0),
]


def vascular_small():
    from paper_2512_02175_b200 import workloads

    return workloads.vascular_text(n_nodes=400, seed=3)


def ensemble_vectors():
    out = {}
    meta = []
    vtext = vascular_small()
    entries = list(ENSEMBLES) + [
        ("vascular_small", "vascular_small", 2000, 100, 1e-3, 19, ("uniform", None), 100, 0.0)]
    for name, case, n, steps, dt, seed, init, cap, refl in entries:
        if case == "vascular_small":
            g, f = graphfile.parse_graph_file(vtext)
            init = ("uniform", float(np.max(g.edge_length)))
        else:
            g, f = build(case, gs)
        cfg = gs.SimulationConfig(dt=dt, n_steps=steps, n_particles=n, seed=seed,
                                  max_splits_per_step=cap, initial=_init(*init), workers=8,
                                  reflect_at=refl)
        res = gs.run_ensemble(g, f, cfg)
        out[name] = dict(edges=res.edges, positions=res.positions, crossings=res.crossings,
                         crossing_events=res.crossing_events, m_histogram=res.stats.m_histogram,
                         stats=np.array([res.stats.truncation_count, res.stats.crossings_total,
                                         res.stats.crossing_events], np.int64))
        meta.append(dict(name=name, case=case, n=n, steps=steps, dt=dt, seed=seed,
                         init=list(init), cap=cap, reflect=refl, gamma=res.stats.gamma))
    return out, meta, vtext


TRIALS = [
    ("star5_linear_1e-2", "star5_linear", 5000, 1e-2, 21, 0, 100),
    ("star_homog_1e-3", "star_homog", 5000, 1e-3, 22, 0, 100),
    ("star4_mixed_cap2", "star4_mixed", 5000, 1e-1, 23, 0, 2),
    ("hub8_v0", "hub8", 5000, 1e-2, 24, 0, 100),
    ("random_general_v1", "random_general", 5000, 5e-3, 25, 1, 100),
    ("star3_bm_1e-3", "star3_bm", 5000, 1e-3, 26, 0, 100),
]


def trial_vectors():
    out, meta = {}, []
    for name, case, n, dt, seed, v, cap in TRIALS:
        g, f = build(case, gs)
        tr = gs.vertex_crossing_trials(g, f, dt, n, seed, vertex=v, max_splits=cap, workers=8)
        out[name] = dict(M=tr.M, exit_edges=tr.exit_edges, exit_positions=tr.exit_positions,
                         truncated=tr.truncated)
        meta.append(dict(name=name, case=case, n=n, dt=dt, seed=seed, vertex=v, cap=cap,
                         gamma=tr.gamma))
    return out, meta


def stat_vectors(ens):
    """Histograms, exit-probability reports and a crossing-bound report."""
    g, f = build("star3_bm", gs)
    grid = EdgeGrid.uniform(g, 16, lengths=[0.5, 0.5, 0.5])
    e = ens["c1_star3_bm"]
    h1 = analysis.histogram_accumulate(e["edges"], e["positions"], grid)
    gh, fh = build("hub64", gs)
    gridh = EdgeGrid.uniform(gh, 8)
    eh = ens["hub64_unif"]
    h2 = analysis.histogram_accumulate(eh["edges"], eh["positions"], gridh)
    g5, f5 = build("star5_linear", gs)
    rep = analysis.exit_probability_experiment(g5, f5, [1e-2, 1e-3, 1e-4, 1e-5], 200_000, 11,
                                               workers=8)
    gh_, fh_ = build("star_homog", gs)
    tr = gs.vertex_crossing_trials(gh_, fh_, 1e-3, 200_000, 3, workers=8)
    cb = analysis.check_crossing_bound(tr)
    return dict(
        hist_star3=dict(counts=h1.counts.tolist(), total=h1.total, lengths=[0.5] * 3, cells=16),
        hist_hub64=dict(counts=h2.counts.tolist(), total=h2.total, cells=8),
        exit_prob=dict(trials=200_000, seed=11, dts=[1e-2, 1e-3, 1e-4, 1e-5],
                       freqs=[r.frequencies.tolist() for r in rep.rows],
                       maxdev=rep.max_deviations,
                       mean_M=[r.mean_crossings for r in rep.rows]),
        crossing_bound=dict(m_hist=tr.stats().m_histogram.tolist(), gamma=cb.gamma,
                            rows=[[r.k, r.empirical, r.bound, r.chi2_tail, r.std_error,
                                   bool(r.bound_violated), bool(r.chi2_deviates)]
                                  for r in cb.rows]),
    )


def graph_vectors():
    """Packed arrays + gamma of every case as built by the reference."""
    out = {}
    vtext = vascular_small()
    for case in list(CASES) + ["vascular_small"]:
        if case == "vascular_small":
            g, f = graphfile.parse_graph_file(vtext)
        else:
            g, f = build(case, gs)
        kind, coef, tab_off, tab_x, tab_mu, sigma = f.packed()
        out[case] = dict(edge_init=g.edge_init, edge_term=g.edge_term, edge_length=g.edge_length,
                         v_off=g.v_off, v_edges=g.v_edges, v_orient=g.v_orient, v_cumw=g.v_cumw,
                         is_star=np.array([g.is_star]), dkind=kind, dcoef=coef, tab_off=tab_off,
                         tab_x=tab_x, tab_mu=tab_mu, sigma=sigma,
                         graph_gamma=np.array([engine._graph_gamma(g, f, 1e-3)]))
    return out


def main():
    os.makedirs(HERE, exist_ok=True)
    gv = graph_vectors()
    np.savez_compressed(os.path.join(HERE, "graphs.npz"),
                        **{f"{c}/{k}": v for c, d in gv.items() for k, v in d.items()})
    if "--only-graphs" in sys.argv:
        return
    with open(os.path.join(HERE, "rng.json"), "w") as fh:
        json.dump(rng_vectors(), fh, indent=0)
    with open(os.path.join(HERE, "solvers.json"), "w") as fh:
        json.dump(solver_vectors(), fh, indent=0)
    steps = step_vectors()
    np.savez_compressed(os.path.join(HERE, "steps.npz"),
                        **{f"{c}/{k}": v for c, d in steps.items() for k, v in d.items()})
    ens, meta, vtext = ensemble_vectors()
    np.savez_compressed(os.path.join(HERE, "ensembles.npz"),
                        **{f"{c}/{k}": v for c, d in ens.items() for k, v in d.items()})
    with open(os.path.join(HERE, "vascular_small.graph"), "w") as fh:
        fh.write(vtext)
    tr, tmeta = trial_vectors()
    np.savez_compressed(os.path.join(HERE, "trials.npz"),
                        **{f"{c}/{k}": v for c, d in tr.items() for k, v in d.items()})
    stats = stat_vectors(ens)
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(dict(ensembles=meta, trials=tmeta, stats=stats,
                       reference="graphsde " + gs.__version__), fh, indent=0)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
