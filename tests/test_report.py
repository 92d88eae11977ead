"""CSV emitters vs the reference's own output (tests/golden/report/, written by
tests/golden/make_report_golden.py from graphsde/report.py:54-182)."""

import os
import sys

import numpy as np
import pytest

import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, report
from paper_2512_02175_b200.engine import BounceStats

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "report")
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_report_golden import report_inputs  # noqa: E402


def _same(tmp_path, name, write):
    out = tmp_path / name
    write(out)
    assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read(), name


@pytest.fixture(scope="module")
def d():
    return report_inputs()


@pytest.fixture(scope="module")
def grid(d):
    return gs.EdgeGrid(counts=np.array(d["counts_per_edge"]), lengths=np.array(d["lengths"]))


def test_density_csv_matches_reference(tmp_path, d, grid):
    h = analysis.Histogram(grid=grid, counts=d["hist_counts"], total=int(d["hist_counts"].sum()))
    _same(tmp_path, "density_hist.csv", lambda p: report.write_density_csv(p, h))
    _same(tmp_path, "density_raw.csv", lambda p: report.write_density_csv(p, d["raw_density"], grid))


def test_density_csv_round_trip(tmp_path, d, grid):
    p = report.write_density_csv(tmp_path / "r.csv", d["raw_density"], grid)
    eid, idx, left, right, rho = report.read_density_csv(p)
    assert np.array_equal(rho, d["raw_density"])  # 17 significant digits: exact
    assert np.array_equal(eid, np.repeat(np.arange(3), d["counts_per_edge"]))
    assert np.array_equal(right - left > 0, np.ones(len(rho), bool))
    with pytest.raises(report.IoError):
        report.write_density_csv(tmp_path / "x.csv", d["raw_density"])  # raw needs a grid
    (tmp_path / "bad.csv").write_text("a,b\n")
    with pytest.raises(report.IoError):
        report.read_density_csv(tmp_path / "bad.csv")
    (tmp_path / "empty.csv").write_text(",".join(report.DENSITY_HEADER) + "\r\n")
    assert all(len(a) == 0 for a in report.read_density_csv(tmp_path / "empty.csv"))


def test_small_tables_match_reference(tmp_path, d):
    m = d["m_hist"]
    stats = BounceStats(m_histogram=m, gamma=0.01, truncation_count=1,
                        crossings_total=int((np.arange(8) * m).sum()),
                        crossing_events=int(m[1:].sum()))
    _same(tmp_path, "bounces.csv", lambda p: report.write_bounces_csv(p, stats))
    rows = tuple(analysis.ExitProbabilityRow(**r) for r in d["exit_rows"])
    rep = analysis.ExitProbabilityReport(vertex=0, trials=1000, rows=rows)
    _same(tmp_path, "exit_prob.csv", lambda p: report.write_exit_prob_csv(p, rep))
    brows = tuple(analysis.CrossingBoundRow(**r) for r in d["bound_rows"])
    brep = analysis.CrossingBoundReport(gamma=0.01, n_steps=1000, rows=brows, homogeneous=True)
    _same(tmp_path, "bound_check.csv", lambda p: report.write_bound_check_csv(p, brep))
    _same(tmp_path, "summary.csv", lambda p: report.write_summary_csv(p, d["summary"]))
    _same(tmp_path, "errors.csv", lambda p: report.write_error_table_csv(p, d["errors"]))


def test_format_value_round_trips():
    for v in (0.1, 1 / 3, 1e-300, 2.0 ** -1074, 1.7976931348623157e308, -0.0, 123456789.0):
        assert float(report.format_value(v)) == v


def test_figures_need_matplotlib(tmp_path, grid):
    try:
        import matplotlib  # noqa: F401
    except ImportError:
        with pytest.raises(report.IoError):
            report.save_density_figure(tmp_path / "f.png", grid, {})
