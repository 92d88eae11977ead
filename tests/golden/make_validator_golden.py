"""Golden vectors for the host-side validators and the drop-in namespace,
produced by the REFERENCE package itself (graphsde, imported from
/root/reference/pkg/src or an install under baseline/_ref).

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_validator_golden.py

Writes tests/golden/validators.json:
* SteadyStateOracle (analysis.py:82-206): B, D, closed-form / printed
  normalisers, self_check, edge / tail masses, densities, truncation lengths
  for several rate sets, sigmas and tolerances;
* l2_error (analysis.py:224-245) of a Histogram, an FvmState and a raw array
  against oracles and a callable;
* check_crossing_bound (analysis.py:283-319) on synthetic M histograms
  (homogeneous and not, gamma overrides, k_max, empty);
* the public names of every reference module (the namespace-diff test).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "graphsde")):
        sys.path.insert(0, p)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsde_numba_cache")

import graphsde as gs  # noqa: E402
from graphsde import analysis, engine, fvm, graphfile, grids, rng  # noqa: E402

MODULES = ("graphsde", "graphsde.analysis", "graphsde.engine", "graphsde.rng", "graphsde.graph",
           "graphsde.coefficients", "graphsde.grids", "graphsde.graphfile", "graphsde.fvm",
           "graphsde.report")


def namespace():
    import importlib
    import types

    out = {}
    for name in MODULES:
        try:
            m = importlib.import_module(name)
        except Exception as exc:  # report.py needs matplotlib (absent here): read its source
            import ast

            src = os.path.join(os.path.dirname(gs.__file__), name.split(".")[-1] + ".py")
            tree = ast.parse(open(src).read())
            names = set()
            for node in tree.body:
                if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
                    names.add(node.name)
                elif isinstance(node, ast.Assign):
                    names.update(t.id for t in node.targets if isinstance(t, ast.Name))
                elif isinstance(node, ast.AnnAssign) and isinstance(node.target, ast.Name):
                    names.add(node.target.id)
            out[name] = {"names": sorted(n for n in names if not n.startswith("_")),
                         "from_source": repr(exc)}
            continue
        names = []
        for k, v in vars(m).items():
            if k.startswith("_") or isinstance(v, types.ModuleType):
                continue
            mod = getattr(v, "__module__", None)
            if mod is not None and not mod.startswith("graphsde"):
                continue  # re-exported third-party names (np, math helpers, numba, ...)
            names.append(k)
        out[name] = {"names": sorted(names)}
    return out


def oracles():
    rows = []
    for kind in ("linear", "quadratic"):
        for rates, sigma in (([10.0, 20.0, 30.0, 40.0, 50.0], 1.0), ([1.0, 3.5], 0.7),
                             ([0.2, 5.0, 80.0], 2.0)):
            o = analysis.SteadyStateOracle.create(kind, rates, sigma)
            xs = [0.0, 0.013, 0.1, 0.77, 3.0]
            rows.append(dict(
                kind=kind, rates=rates, sigma=sigma, B=o.B, D=o.D,
                closed_form=float(o.closed_form_normalizer()),
                as_printed=float(o.as_printed_normalizer()),
                self_check={k: (float(v) if not isinstance(v, str) else v)
                            for k, v in o.self_check().items()},
                edge_mass=[o.edge_mass(e) for e in range(len(rates))],
                tail_mass=[[o.tail_mass(e, L) for L in (0.0, 0.05, 0.5, 2.0)]
                           for e in range(len(rates))],
                density=[[float(v) for v in np.atleast_1d(o.density(e, np.array(xs)))]
                         for e in range(len(rates))],
                density_scalar=[float(o.density(e, 0.25)) for e in range(len(rates))],
                trunc_8=o.truncation_lengths(1e-8).tolist(),
                trunc_4=o.truncation_lengths(1e-4).tolist(),
            ))
    # from_field on a star graph
    g = gs.build_graph([(0, None, float("inf"))] * 3)
    f = gs.CoefficientField.for_graph(g, [gs.LinearDrift(-2.0), gs.LinearDrift(-5.0),
                                          gs.LinearDrift(-9.0)], [1.3] * 3)
    o = analysis.SteadyStateOracle.from_field(g, f)
    rows.append(dict(from_field="star3_quadratic", kind=o.kind, rates=o.rates.tolist(), B=o.B,
                     D=o.D))
    return rows


def l2_cases():
    out = []
    g = gs.build_graph([(0, None, float("inf"))] * 3)
    o = analysis.SteadyStateOracle.create("linear", [10.0, 20.0, 30.0], 1.0)
    grid = grids.EdgeGrid.uniform(g, 12, lengths=o.truncation_lengths(1e-6))
    r = np.random.default_rng(5)
    counts = r.integers(0, 1000, grid.n_cells).astype(np.int64)
    h = analysis.Histogram(grid=grid, counts=counts, total=int(counts.sum()))
    out.append(dict(kind="histogram", lengths=grid.lengths.tolist(), cells=12,
                    counts=counts.tolist(), total=int(counts.sum()),
                    l2=analysis.l2_error(h, o)))
    rho = r.uniform(0.0, 3.0, grid.n_cells)
    st = fvm.FvmState(grid=grid, rho=rho, t=0.5)
    out.append(dict(kind="fvm_state", lengths=grid.lengths.tolist(), cells=12,
                    rho=rho.tolist(), l2=analysis.l2_error(st, o)))
    out.append(dict(kind="raw", lengths=grid.lengths.tolist(), cells=12, rho=rho.tolist(),
                    l2=analysis.l2_error(rho, o, grid=grid)))
    oq = analysis.SteadyStateOracle.create("quadratic", [10.0, 20.0, 30.0], 1.0)
    out.append(dict(kind="raw_quadratic", lengths=grid.lengths.tolist(), cells=12,
                    rho=rho.tolist(), l2=analysis.l2_error(rho, oq, grid=grid)))
    out.append(dict(kind="callable", lengths=grid.lengths.tolist(), cells=12, rho=rho.tolist(),
                    l2=analysis.l2_error(rho, lambda e, x: np.exp(-(e + 1) * x), grid=grid)))
    return out


def bound_cases():
    out = []
    r = np.random.default_rng(11)
    for i, (homog, gam, kmax) in enumerate([(True, None, 10), (False, None, 10), (True, 0.0, 6),
                                            (True, 3.7, 12), (False, 0.4, 3), (True, None, 1)]):
        m = r.integers(0, 5000, 40).astype(np.int64)
        m[0] = 0
        m[25:] = 0
        g0 = float(r.uniform(0.1, 4.0))
        b = engine.BounceStats(m_histogram=m, gamma=g0, truncation_count=0,
                               crossings_total=int((m * np.arange(m.size)).sum()),
                               crossing_events=int(m.sum()))
        rep = analysis.check_crossing_bound(b, gamma=gam, k_max=kmax, homogeneous=homog)
        out.append(dict(m_hist=m.tolist(), gamma0=g0, gamma=gam, k_max=kmax, homogeneous=homog,
                        rep_gamma=rep.gamma, n_steps=rep.n_steps,
                        any_bound=rep.any_bound_violation, any_chi2=rep.any_chi2_deviation,
                        rows=[[x.k, x.empirical, x.bound, x.chi2_tail, x.std_error,
                               bool(x.bound_violated), bool(x.chi2_deviates)]
                              for x in rep.rows]))
    m = np.zeros(11, np.int64)
    b = engine.BounceStats(m_histogram=m, gamma=1.0, truncation_count=0, crossings_total=0,
                           crossing_events=0)
    rep = analysis.check_crossing_bound(b)
    out.append(dict(m_hist=m.tolist(), gamma0=1.0, gamma=None, k_max=10, homogeneous=True,
                    rep_gamma=rep.gamma, n_steps=rep.n_steps, any_bound=rep.any_bound_violation,
                    any_chi2=rep.any_chi2_deviation,
                    rows=[[x.k, x.empirical, x.bound, x.chi2_tail, x.std_error,
                           bool(x.bound_violated), bool(x.chi2_deviates)] for x in rep.rows]))
    return out


def rng_scalars():
    r = np.random.default_rng(3)
    top = (1 << 53) - 1  # 53-bit lattice index n = r >> 11
    words = [0, 1, 2047, 2048, (1 << 64) - 1, (1 << 63), (1 << 63) - 1] + [
        (top - j) << 11 for j in range(1, 9)] + [j << 11 for j in range(1, 5)] + [
        int(v) for v in r.integers(0, 1 << 63, 40, dtype=np.int64)]
    ps = [1e-300, 1e-20, 1e-12, 2.5e-7, 0.01, 0.075, 0.0751, 0.3, 0.5, 0.6, 0.925, 0.9999,
          1.0 - 1e-12]
    return dict(u64=[str(w) for w in words],
                u64_to_uniform=[float(rng.u64_to_uniform(np.uint64(w))) for w in words],
                u64_to_normal=[float(rng.u64_to_normal(np.uint64(w))) for w in words],
                p=ps, norm_ppf=[float(rng.norm_ppf(p)) for p in ps])


def main():
    out = dict(reference="graphsde " + gs.__version__, namespace=namespace(),
               steady_state=oracles(), l2=l2_cases(), crossing=bound_cases(),
               rng_scalars=rng_scalars(), available_workers_type="int")
    with open(os.path.join(HERE, "validators.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print("validators.json written")


if __name__ == "__main__":
    main()
