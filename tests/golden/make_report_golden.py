"""Golden CSV files from the REFERENCE report writers (graphsde/report.py:54-182).

    python tests/golden/make_report_golden.py

The reference module imports matplotlib at top level (figures); matplotlib is
not in this image, so a stub module is registered first -- the CSV writers do
not touch it.  Inputs are built from ``report_inputs()`` below, which the test
(tests/test_report.py) rebuilds with this package's classes; outputs go to
tests/golden/report/.
"""

from __future__ import annotations

import os
import sys
import types

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "report")

import numpy as np  # noqa: E402


def report_inputs():
    """Plain-data inputs shared by the generator and the test."""
    rng = np.random.default_rng(2512)
    counts_per_edge = [4, 3, 5]
    lengths = [1.0, 0.3, 2.5]
    hist_counts = rng.integers(0, 50, size=sum(counts_per_edge))
    raw_density = rng.random(sum(counts_per_edge)) * 3.0
    m_hist = np.array([0, 812, 203, 51, 9, 2, 0, 1], dtype=np.int64)
    exit_rows = []
    for i, dt in enumerate([1e-2, 1e-3, 1e-4]):
        f = rng.dirichlet(np.ones(5))
        b = np.full(5, 0.2)
        se = np.sqrt(b * (1 - b) / (1000 * (i + 1)))
        exit_rows.append(dict(dt=dt, frequencies=f, expected=b,
                              max_deviation=float(np.max(np.abs(f - b))), binomial_se=se,
                              mean_crossings=1.0 + i / 3))
    bound_rows = [dict(k=k, empirical=1 - 0.5 ** k, bound=1 - np.exp(-(k - 0.01) ** 2 / (4 * k)),
                       chi2_tail=0.1 / k, std_error=1e-3 * k, bound_violated=(k == 3),
                       chi2_deviates=(k == 2)) for k in range(1, 7)]
    summary = {"n_particles": 10000, "dt": 1e-3, "label": "star3", "l2": 0.0123456789}
    errors = [dict(method="em", dt=1e-3, cells_per_edge=64, l2_error=0.0371),
              dict(method="fvm", dt=2.5e-5, cells_per_edge=128, l2_error=1.0 / 3)]
    return dict(counts_per_edge=counts_per_edge, lengths=lengths, hist_counts=hist_counts,
                raw_density=raw_density, m_hist=m_hist, exit_rows=exit_rows,
                bound_rows=bound_rows, summary=summary, errors=errors)


def main():
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    mpl.pyplot = types.ModuleType("matplotlib.pyplot")
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.pyplot", mpl.pyplot)
    sys.path.insert(0, REF)
    from graphsde import analysis, engine, report
    from graphsde.grids import EdgeGrid

    d = report_inputs()
    os.makedirs(OUT, exist_ok=True)
    grid = EdgeGrid(counts=np.array(d["counts_per_edge"]), lengths=np.array(d["lengths"]))
    h = analysis.Histogram(grid=grid, counts=d["hist_counts"], total=int(d["hist_counts"].sum()))
    report.write_density_csv(os.path.join(OUT, "density_hist.csv"), h)
    report.write_density_csv(os.path.join(OUT, "density_raw.csv"), d["raw_density"], grid)
    stats = engine.BounceStats(m_histogram=d["m_hist"], gamma=0.01, truncation_count=1,
                               crossings_total=int((np.arange(8) * d["m_hist"]).sum()),
                               crossing_events=int(d["m_hist"][1:].sum()))
    report.write_bounces_csv(os.path.join(OUT, "bounces.csv"), stats)
    rows = tuple(analysis.ExitProbabilityRow(**r) for r in d["exit_rows"])
    report.write_exit_prob_csv(os.path.join(OUT, "exit_prob.csv"),
                               analysis.ExitProbabilityReport(vertex=0, trials=1000, rows=rows))
    brows = tuple(analysis.CrossingBoundRow(**r) for r in d["bound_rows"])
    report.write_bound_check_csv(
        os.path.join(OUT, "bound_check.csv"),
        analysis.CrossingBoundReport(gamma=0.01, n_steps=1000, rows=brows, homogeneous=True))
    report.write_summary_csv(os.path.join(OUT, "summary.csv"), d["summary"])
    report.write_error_table_csv(os.path.join(OUT, "errors.csv"), d["errors"])
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
