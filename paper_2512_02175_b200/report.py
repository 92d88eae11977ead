"""CSV result emission (reference ``graphsde/report.py:54-182``).

The CSV files are the machine-readable contract of the reference's
experiments: densities use the per-edge bin schema
``edge_id,bin_index,x_left,x_right,density`` and every float is written with
17 significant digits so it round-trips exactly.  Output is byte-identical
to the reference's writers (``tests/test_report.py`` against fixtures the
reference produced).  Large density tables (vascular grids, ~1e6 cells) are
formatted with numpy instead of a per-row ``csv.writer`` loop.

The reference also renders PNG figures with matplotlib
(``report.py:185-260``); figures carry no information the CSVs do not, and
matplotlib is not part of this image, so ``save_*_figure`` import it lazily
and raise :class:`IoError` when it is absent.
"""

from __future__ import annotations

import csv
from pathlib import Path

import numpy as np

from .analysis import CrossingBoundReport, ExitProbabilityReport, Histogram
from .engine import BounceStats
from .grids import EdgeGrid

DENSITY_HEADER = ["edge_id", "bin_index", "x_left", "x_right", "density"]


class IoError(OSError):
    """Malformed CSV input or a missing output dependency (``report.py:35``)."""


def format_value(x: float) -> str:
    """``%.17g``: the shortest width that reproduces every double (``report.py:39-41``)."""
    return format(float(x), ".17g")


def _density_of(obj, grid: EdgeGrid | None):
    """(grid, per-cell density) of a Histogram, an FVM-style state (``.grid`` +
    ``.rho``) or a raw array with an explicit grid (``report.py:44-51``)."""
    if isinstance(obj, Histogram):
        return obj.grid, obj.density()
    if hasattr(obj, "grid") and hasattr(obj, "rho"):
        return obj.grid, np.asarray(obj.rho, dtype=np.float64)
    if grid is None:
        raise IoError("raw density arrays need an explicit grid")
    return grid, np.asarray(obj, dtype=np.float64)


def _g17(a: np.ndarray) -> list[str]:
    return [format(float(v), ".17g") for v in a]


def write_density_csv(path, obj, grid: EdgeGrid | None = None) -> Path:
    """Histogram / FVM state / raw density -> density CSV (``report.py:54-68``).

    Bin ``i`` of edge ``e`` spans ``[i dx_e, (i+1) dx_e)`` with ``dx_e`` the
    grid's cell width, each bound computed as ``i * dx_e`` like the reference.
    """
    grid, density = _density_of(obj, grid)
    density = np.asarray(density, dtype=np.float64).reshape(-1)
    path = Path(path)
    counts = np.asarray(grid.counts, dtype=np.int64)
    eid = np.repeat(np.arange(grid.n_edges, dtype=np.int64), counts)
    starts = np.repeat(grid.offsets[:-1], counts)
    idx = np.arange(eid.shape[0], dtype=np.int64) - starts
    w = np.repeat(grid.dx, counts)
    left = idx.astype(np.float64) * w
    right = (idx + 1).astype(np.float64) * w
    n = min(eid.shape[0], density.shape[0])
    cols = (eid[:n].astype(str), idx[:n].astype(str), _g17(left[:n]), _g17(right[:n]),
            _g17(density[:n]))
    body = "".join(f"{a},{b},{c},{d},{e}\r\n" for a, b, c, d, e in zip(*cols))
    with path.open("w", newline="") as fh:
        fh.write(",".join(DENSITY_HEADER) + "\r\n")
        fh.write(body)
    return path


def read_density_csv(path):
    """Density CSV -> (edge_id, bin_index, x_left, x_right, density) arrays
    (``report.py:71-98``)."""
    with Path(path).open(newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header != DENSITY_HEADER:
            raise IoError(f"unexpected density header {header!r}")
        rows = [(int(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4])) for r in reader]
    if not rows:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), np.zeros(0), np.zeros(0), np.zeros(0)
    c = list(zip(*rows))
    return (np.asarray(c[0], dtype=np.int64), np.asarray(c[1], dtype=np.int64),
            np.asarray(c[2]), np.asarray(c[3]), np.asarray(c[4]))


def _write_rows(path, header, rows) -> Path:
    path = Path(path)
    with path.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)
    return path


def write_bounces_csv(path, stats: BounceStats) -> Path:
    """``m,count`` for m >= 1 (``report.py:101-111``)."""
    return _write_rows(path, ["m", "count"],
                       ([m, int(c)] for m, c in enumerate(stats.m_histogram) if m))


def write_summary_csv(path, entries: dict) -> Path:
    """``key,value``; floats at 17 digits (``report.py:114-123``)."""
    return _write_rows(path, ["key", "value"],
                       ([k, format_value(v) if isinstance(v, float) else v]
                        for k, v in entries.items()))


def write_error_table_csv(path, rows: list[dict]) -> Path:
    """``method,dt,cells_per_edge,l2_error`` (``report.py:126-141``)."""
    return _write_rows(path, ["method", "dt", "cells_per_edge", "l2_error"],
                       ([r["method"], format_value(r["dt"]), r["cells_per_edge"],
                         format_value(r["l2_error"])] for r in rows))


def write_exit_prob_csv(path, report: ExitProbabilityReport) -> Path:
    """One row per (dt, slot) (``report.py:144-161``)."""
    def rows():
        for r in report.rows:
            for s in range(len(r.frequencies)):
                yield [format_value(r.dt), s, format_value(r.frequencies[s]),
                       format_value(r.expected[s]), format_value(r.binomial_se[s]),
                       format_value(r.max_deviation)]
    return _write_rows(path, ["dt", "slot", "frequency", "expected", "binomial_se",
                              "max_deviation"], rows())


def write_bound_check_csv(path, report: CrossingBoundReport) -> Path:
    """Thm 3.1 check rows (``report.py:164-182``)."""
    return _write_rows(path, ["k", "empirical_cdf", "bound", "chi2_tail", "std_error",
                              "bound_violated"],
                       ([r.k, format_value(r.empirical), format_value(r.bound),
                         format_value(r.chi2_tail), format_value(r.std_error),
                         int(r.bound_violated)] for r in report.rows))


def _pyplot():
    try:
        import matplotlib

        matplotlib.use("Agg")
        import matplotlib.pyplot as plt
    except ImportError as exc:  # pragma: no cover - depends on the image
        raise IoError("figures need matplotlib, which is not installed") from exc
    return plt


def save_density_figure(path, grid: EdgeGrid, series, oracle=None) -> Path:
    """Per-edge density panels (``report.py:197-214``); needs matplotlib."""
    plt = _pyplot()
    n = grid.n_edges
    fig, axes = plt.subplots(n, 1, figsize=(6, 2.2 * n), squeeze=False)
    for e in range(n):
        ax = axes[e][0]
        x = grid.centers(e)
        for label, obj in series.items():
            _, d = _density_of(obj, grid)
            ax.step(x, d[grid.edge_slice(e)], where="mid", label=label)
        if oracle is not None:
            from .analysis import steady_state_density

            ax.plot(x, steady_state_density(oracle, e, x), "k--", label="oracle")
        ax.set_ylabel(f"edge {e}")
    axes[0][0].legend()
    fig.savefig(path)
    plt.close(fig)
    return Path(path)


def save_exit_prob_figure(path, report: ExitProbabilityReport) -> Path:
    """Max exit-frequency deviation vs dt (``report.py:217-235``); needs matplotlib."""
    plt = _pyplot()
    fig, ax = plt.subplots()
    ax.loglog([r.dt for r in report.rows], report.max_deviations, "o-")
    ax.set_xlabel("dt")
    ax.set_ylabel("max |freq - b|")
    fig.savefig(path)
    plt.close(fig)
    return Path(path)


def save_bounce_figure(path, stats: BounceStats, report: CrossingBoundReport | None = None):
    """Empirical P(M <= k) with the Thm 3.1 bound (``report.py:238-260``); needs matplotlib."""
    plt = _pyplot()
    fig, ax = plt.subplots()
    ks = np.arange(1, len(stats.m_histogram))
    ax.plot(ks, [stats.cdf(int(k)) for k in ks], "o-", label="empirical")
    if report is not None:
        ax.plot([r.k for r in report.rows], [r.bound for r in report.rows], "k--",
                label="bound")
    ax.legend()
    fig.savefig(path)
    plt.close(fig)
    return Path(path)
