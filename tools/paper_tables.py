"""Paper-scale experiment tables on one B200, written with the CSV emitters.

    python tools/paper_tables.py [outdir]      (default: gpurun_out/)

1. Exit-probability dt sweep (SPEC §4.1 star, paper §4.1): exit frequencies vs the
   jump weights at dt = 1e-2 .. 1e-5 with 1e10 vertex trials per dt (native stream,
   fused exit counts) -> exit_prob.csv.  The reference reports the same table at
   2e5 trials per dt.
2. EM vs FVM at matched discretisation (SPEC acceptance 7): L2 error of the
   steady-state density against the analytic oracle on the §4.1 linear and
   quadratic stars, EM with 1e8 particles x 1e5 steps (dt = 1e-4, T = 10, snapshot
   histogram) and the FVM baseline run to T = 10 at its stability limit, 50 / 100 /
   200 cells per edge -> error_table.csv.
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, fvm, report, workloads

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs(out, exist_ok=True)

ONLY = os.environ.get("TABLES_ONLY", "")

# 1. exit probabilities
g, f = workloads.star5("linear")
rep = None
t0 = time.time()
if not ONLY or ONLY == "1":
    rep = analysis.exit_probability_experiment(g, f, [1e-2, 1e-3, 1e-4, 1e-5], 10_000_000_000,
                                               11)
    report.write_exit_prob_csv(os.path.join(out, "exit_prob.csv"), rep)
    print(f"exit-probability sweep: {time.time() - t0:.1f} s")
for r in (rep.rows if rep else ()):
    print(f"  dt={r.dt:g} max|freq-b|={r.max_deviation:.3e} se={r.binomial_se.max():.1e} "
          f"mean M={r.mean_crossings:.3f}")

# 2. EM vs FVM
rows = []
for kind in (("linear", "quadratic") if not ONLY or ONLY == "2" else ()):
    g, f = workloads.star5(kind)
    orc = analysis.SteadyStateOracle.from_field(g, f)
    lengths = orc.truncation_lengths(1e-8)
    for cells in (50, 100, 200):
        grid = gs.EdgeGrid.uniform(g, cells, lengths=lengths)
        t0 = time.time()
        cfg = gs.SimulationConfig(dt=1e-4, n_steps=100_000, n_particles=100_000_000, seed=5)
        h, st = analysis.run_ensemble_histogram(g, f, cfg, grid)
        em = analysis.l2_error(h, orc)
        t_em = time.time() - t0
        t0 = time.time()
        dt_f = 0.9 * fvm.stability_limit(g, f, grid)
        n_f = int(np.ceil(10.0 / dt_f))
        res = fvm.fvm_run(g, f, grid, dt_f, n_f, fvm.FvmState.uniform(grid))
        fv = analysis.l2_error(res.state.rho, orc, grid)
        t_fv = time.time() - t0
        rows += [dict(method=f"em_{kind}", dt=1e-4, cells_per_edge=cells, l2_error=em),
                 dict(method=f"fvm_{kind}", dt=dt_f, cells_per_edge=cells, l2_error=fv)]
        print(f"{kind} cells={cells}: EM L2={em:.4f} ({t_em:.1f} s, 1e13 psteps, "
              f"truncations {st.truncation_count}); FVM L2={fv:.4f} ({n_f} steps, {t_fv:.1f} s)")
if rows:
    report.write_error_table_csv(os.path.join(out, "error_table.csv"), rows)

# 3. Crossing statistics vs Thm 3.1 / the chi-squared law (homogeneous star, 1e10 trials
#    per stream): M histogram of vertex trials, fused on the device
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests", "golden"))
import cases  # noqa: E402
from paper_2512_02175_b200.engine import BounceStats  # noqa: E402

g, f = cases.build("star_homog", gs)
for rng, n in ((("native", 10_000_000_000), ("reference", 1_000_000_000))
               if not ONLY or ONLY == "3" else ()):
    t0 = time.time()
    ec = analysis.vertex_exit_counts(g, f, 1e-3, n, 21, rng=rng)
    bs = BounceStats(m_histogram=ec.m_histogram, gamma=ec.gamma,
                     truncation_count=ec.truncation_count, crossings_total=ec.crossings_total,
                     crossing_events=ec.crossing_events)
    cb = analysis.check_crossing_bound(bs)
    report.write_bounces_csv(os.path.join(out, f"bounces_{rng}.csv"), bs)
    report.write_bound_check_csv(os.path.join(out, f"bound_check_{rng}.csv"), cb)
    worst = max(abs(r.empirical - r.chi2_tail) / r.std_error for r in cb.rows)
    print(f"crossing law ({rng}, {n:.0e} trials, {time.time() - t0:.1f} s): gamma={cb.gamma:.4f} "
          f"bound violated={cb.any_bound_violation} chi2 deviates={cb.any_chi2_deviation} "
          f"max |emp-chi2|/se={worst:.2f}")

# 4. Native vs reference stream at scale: snapshot densities (two-sample chi-square)
from scipy import stats as _st  # noqa: E402


def _chi2(h1, h2, min_count=20):
    h1, h2 = np.asarray(h1, np.float64), np.asarray(h2, np.float64)
    keep = (h1 + h2) >= min_count
    a, b = h1[keep], h2[keep]
    k1, k2 = np.sqrt(b.sum() / a.sum()), np.sqrt(a.sum() / b.sum())
    chi2 = float((((k1 * a - k2 * b) ** 2) / (a + b)).sum())
    dof = int(keep.sum()) - 1
    return float(_st.chi2.sf(chi2, dof)), chi2, dof


for name, build, init, steps, n_nat, n_ref, cells in (
        ("C1 star3 (driftless kernel)", lambda: workloads.star3(), lambda g: gs.AtVertex(0), 1000,
         1_000_000_000, 100_000_000, 16),
        ("C2 hub64", workloads.hub64, lambda g: gs.PerEdgeUniform(2.0), 1000,
         1_000_000_000, 100_000_000, 8),
        ("C4 vascular", workloads.vascular,
         lambda g: gs.PerEdgeUniform(float(g.edge_length.max())), 100,
         1_000_000_000, 100_000_000, 2)):
    if ONLY and ONLY != "4":
        break
    g, f = build()
    grid = gs.EdgeGrid.uniform(g, cells, lengths=[3.0] * g.n_edges if g.is_star else None)
    res = {}
    for rng, n, seed in (("native", n_nat, 31), ("reference", n_ref, 32)):
        t0 = time.time()
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=steps, n_particles=n, seed=seed,
                                  initial=init(g), rng=rng)
        h, st = analysis.run_ensemble_histogram(g, f, cfg, grid)
        res[rng] = (h.counts, st.crossings_total / (n * steps), time.time() - t0)
    p, chi2, dof = _chi2(res["native"][0], res["reference"][0])
    print(f"{name}: native {n_nat:.0e} vs reference {n_ref:.0e} particles x {steps} steps: "
          f"density chi2 p={p:.3g} (chi2={chi2:.0f}, dof={dof}); crossings/pstep "
          f"{res['native'][1]:.6f} vs {res['reference'][1]:.6f}; "
          f"{res['native'][2]:.1f} s / {res['reference'][2]:.1f} s")
