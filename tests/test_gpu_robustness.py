"""GPU robustness edges of the native kernels:

* ``n_steps == 0`` (placement only) counts every particle exactly once in the
  fused histogram / edge counts;
* caps whose M histogram exceeds the shared-memory bins (the reference accepts
  any ``max_splits_per_step``) run, and agree with a small cap when no step
  reaches it;
* more in-flight launches on one graph handle than its work-counter ring has
  slots, alternating between streams, equal serial launches;
* particle ids beyond the native stream's 2^48 range are refused.
"""

import numpy as np
import pytest
import torch

import cases
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import _native, analysis, engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rng", ["native", "reference"])
@pytest.mark.parametrize("case", ["star3_bm", "hub64"])
def test_placement_only_counts_each_particle_once(case, rng):
    g, f = cases.build(case, gs)
    grid = gs.EdgeGrid.uniform(g, 5, lengths=[2.0] * g.n_edges if g.is_star else None)
    init = gs.PointStart(1, 0.3) if g.is_star else gs.PerEdgeUniform(2.0)
    n = 100_003
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=0, n_particles=n, seed=4, initial=init, rng=rng)
    res = engine.ensemble_device(g, f, cfg, outputs=("all", "edge_counts"), grid=grid)
    assert int(res["hist"].sum()) == n
    assert int(res["edge_counts"].sum()) == n
    ec = np.bincount(res["edge"].cpu().numpy(), minlength=g.n_edges)
    np.testing.assert_array_equal(res["edge_counts"].cpu().numpy(), ec)
    h, _ = analysis.run_ensemble_histogram(g, f, cfg, grid)
    assert h.counts.sum() == n
    np.testing.assert_array_equal(h.counts, res["hist"].cpu().numpy())


@pytest.mark.parametrize("case", ["star5_linear", "hub64"])
def test_cap_beyond_shared_bins(case):
    """cap = 20000 -> 20001 M bins (> the 8192 kept in shared memory): bins >= 8
    go to global atomics.  No step here reaches M = 100, so a cap-100 run of
    the same streams must give the same M histogram and outputs."""
    g, f = cases.build(case, gs)
    init = gs.AtVertex(0) if g.is_star else gs.PerEdgeUniform(2.0)
    mk = lambda cap: gs.SimulationConfig(dt=1e-2, n_steps=200, n_particles=200_000, seed=8,
                                         initial=init, max_splits_per_step=cap)
    big = engine.ensemble_device(g, f, mk(20_000))
    small = engine.ensemble_device(g, f, mk(100))
    mb, ms = big["m_hist"].cpu().numpy(), small["m_hist"].cpu().numpy()
    assert mb[101:].sum() == 0 and mb.size == 20_001
    np.testing.assert_array_equal(mb[:101], ms)
    for k in ("edge", "x", "crossings", "events"):
        assert torch.equal(big[k], small[k]), k
    tb = engine.trials_device(g, f, 1e-2, 300_000, 3, max_splits=20_000, per_trial=False)
    ts = engine.trials_device(g, f, 1e-2, 300_000, 3, max_splits=100, per_trial=False)
    np.testing.assert_array_equal(tb["m_hist"].cpu().numpy()[:101], ts["m_hist"].cpu().numpy())
    assert torch.equal(tb["exit_counts"], ts["exit_counts"])


def test_more_launches_in_flight_than_work_slots():
    """80 native launches on one handle (ring of 64 work counters), queued on
    two streams without host synchronisation: each equals its serial run."""
    g, f = cases.build("hub8", gs)
    cfgs = [gs.SimulationConfig(dt=1e-2, n_steps=50, n_particles=20_000 + 37 * i, seed=i,
                                initial=gs.PerEdgeUniform(2.0)) for i in range(80)]
    serial = []
    for c in cfgs:
        r = engine.ensemble_device(g, f, c, outputs=("edge", "crossings"))
        torch.cuda.synchronize()
        serial.append(r)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    queued = []
    for i, c in enumerate(cfgs):
        st = streams[i % 2]
        with torch.cuda.stream(st):
            queued.append(engine.ensemble_device(g, f, c, outputs=("edge", "crossings"),
                                                 stream=st.cuda_stream))
    torch.cuda.synchronize()
    for a, b in zip(serial, queued):
        for k in ("edge", "crossings", "m_hist", "totals"):
            assert torch.equal(a[k], b[k]), k


def test_native_particle_ids_below_2_48():
    g, f = cases.build("star3_bm", gs)
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=1, n_particles=10, seed=1)
    engine.ensemble_device(g, f, cfg, pid_offset=(1 << 48) - 10)  # the last ten ids: fine
    with pytest.raises(_native.GsdeError):
        engine.ensemble_device(g, f, cfg, pid_offset=(1 << 48) - 9)


@pytest.mark.parametrize("cells", [8, 100])  # 64 x 8 (+64): shared bins; 64 x 100: global
def test_fused_bins_shared_and_global_paths(cells):
    """Final-edge counts and the snapshot histogram fused into the native
    ensemble kernel -- warp-aggregated shared-memory counters when the bins
    fit, global atomics otherwise -- equal the histogram of the per-particle
    outputs exactly."""
    from oracle import oracle

    g, f = cases.build("hub64", gs)
    grid = gs.EdgeGrid.uniform(g, cells)
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=100, n_particles=300_001, seed=12,
                              initial=gs.PerEdgeUniform(2.0))
    res = engine.ensemble_device(g, f, cfg, outputs=("edge", "x", "edge_counts"), grid=grid)
    e, x = res["edge"].cpu().numpy(), res["x"].cpu().numpy()
    np.testing.assert_array_equal(res["edge_counts"].cpu().numpy(),
                                  np.bincount(e, minlength=g.n_edges))
    np.testing.assert_array_equal(res["hist"].cpu().numpy(),
                                  oracle.histogram(e, x, grid.offsets, grid.counts, grid.dx))


_GLOBAL_BINS_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, engine, workloads
out = {{}}
for name, (g, f), init in (("hub64", workloads.hub64(), gs.PerEdgeUniform(2.0)),
                           ("star3", workloads.star3(), gs.AtVertex(0))):
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=300, n_particles=200_001, seed=3, initial=init,
                              max_splits_per_step=4)
    grid = gs.EdgeGrid.uniform(g, 4, lengths=[3.0] * g.n_edges if g.is_star else None)
    for lean in (True, False):
        r = engine.ensemble_device(g, f, cfg, outputs=("edge_counts",) if lean else
                                   ("all", "edge_counts"), grid=grid, occupation=(3, 1))
        for k in ("m_hist", "totals", "edge_counts", "hist", "occ"):
            out[name + ("_lean_" if lean else "_pp_") + k] = r[k].cpu().numpy()
ec = analysis.vertex_exit_counts(*workloads.star5("linear"), 1e-3, 2_000_001, 4)
out["trials_counts"], out["trials_m"] = ec.counts, ec.m_histogram
out["trials_tot"] = np.array([ec.crossings_total, ec.crossing_events, ec.truncation_count])
np.savez({path!r}, **out)
"""


def test_global_bins_path_equals_shared_counters(tmp_path):
    """Runs too large for the kernels' 32-bit shared counters (M histogram,
    occupation, final-state bins, trial exit counts) keep them in global int64
    memory (FULL kernels, no shared M bins); GSDE_FORCE_GLOBAL_BINS=1 takes that
    path at a small size.  Every estimator must equal the shared-counter run."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for force in (False, True):
        path = str(tmp_path / f"bins_{int(force)}.npz")
        env = dict(os.environ)
        env.pop("GSDE_FORCE_GLOBAL_BINS", None)
        if force:
            env["GSDE_FORCE_GLOBAL_BINS"] = "1"
        subprocess.run([sys.executable, "-c", _GLOBAL_BINS_SCRIPT.format(root=root, path=path)],
                       check=True, env=env, timeout=600)
        res[force] = np.load(path)
    a, b = res[False], res[True]
    assert sorted(a.files) == sorted(b.files) and len(a.files) == 23
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["hub64_lean_m_hist"][4] > 0  # steps at the cap are counted


_CD_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads
out = {{}}
g, f = workloads.vascular(20_000, seed=5)
grid = gs.EdgeGrid.uniform(g, 4)
for cap in (100, 3):
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=200, n_particles=300_001, seed=3,
                              initial=gs.PerEdgeUniform(float(g.edge_length.max())),
                              max_splits_per_step=cap)
    for outs in (("edge_counts",), ("all", "edge_counts")):
        r = engine.ensemble_device(g, f, cfg, outputs=outs, grid=grid, occupation=(5, 2))
        for k, v in r.items():
            if not k.startswith("_") and v is not None:
                out["c%d_%d_%s" % (cap, len(outs), k)] = v.cpu().numpy()
np.savez({path!r}, **out)
"""


def test_constant_drift_variant_equals_generic_kernel(tmp_path):
    """Graphs whose drifts are all constant in x (C4's drift from_flux) run the
    constant-drift kernel variant; it must equal the generic affine-drift kernel
    (GSDE_GENERIC_DRIFT=1) bit for bit, lean and per-particle, with occupation
    sampling and a truncating cap."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for generic in (False, True):
        path = str(tmp_path / f"cd_{int(generic)}.npz")
        env = dict(os.environ)
        env.pop("GSDE_GENERIC_DRIFT", None)
        if generic:
            env["GSDE_GENERIC_DRIFT"] = "1"
        subprocess.run([sys.executable, "-c", _CD_SCRIPT.format(root=root, path=path)],
                       check=True, env=env, timeout=600)
        res[generic] = np.load(path)
    a, b = res[False], res[True]
    assert sorted(a.files) == sorted(b.files) and len(a.files) >= 20
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


_CHUNK_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads
out = {{}}
for name, (g, f), init in (("hub64", workloads.hub64(), gs.PerEdgeUniform(2.0)),
                           ("star3", workloads.star3(), gs.AtVertex(0))):
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=150, n_particles=100_003, seed=3, initial=init,
                              max_splits_per_step=4)
    grid = gs.EdgeGrid.uniform(g, 4, lengths=[3.0] * g.n_edges if g.is_star else None)
    for outs in (("edge_counts",), ("all", "edge_counts", "counter")):
        r = engine.ensemble_device(g, f, cfg, outputs=outs, grid=grid, occupation=(3, 1))
        for k, v in r.items():
            if not k.startswith("_") and v is not None:
                out[name + "_%d_" % len(outs) + k] = v.cpu().numpy()
    # resume from state-in (per-particle edge / x / next Philox block): pointer offsets
    st = (r["edge"].to(torch.int32), r["x"].to(torch.float32), r["counter"])
    r2 = engine.ensemble_device(g, f, cfg, outputs=("all", "counter"), state=st)
    for k in ("edge", "x", "crossings", "counter", "m_hist", "totals"):
        out[name + "_resume_" + k] = r2[k].cpu().numpy()
# the reference's own streams (FP64 reference-stream kernel, its own chunking)
g, f = workloads.hub64()
cfg = gs.SimulationConfig(dt=1e-3, n_steps=60, n_particles=30_001, seed=9,
                          initial=gs.PerEdgeUniform(2.0), rng="reference")
r = engine.ensemble_device(g, f, cfg, outputs=("all",))
for k in ("edge", "x", "crossings", "events", "m_hist", "totals"):
    out["ref_" + k] = r[k].cpu().numpy()
# injected reference draws through the production kernel (row pointer offsets)
g, f = workloads.hub64()
rs = np.random.default_rng(3)
n, K = 20_001, 120
raw = torch.as_tensor(rs.integers(0, 2**63, size=(n, K), dtype=np.int64)).cuda()
nrm = torch.as_tensor(rs.standard_normal((n, K))).cuda()
cfg = gs.SimulationConfig(dt=1e-3, n_steps=40, n_particles=n, seed=3,
                          initial=gs.PerEdgeUniform(2.0))
r = engine.ensemble_device(g, f, cfg, inject=(raw, nrm), precision="native",
                           outputs=("all", "counter"))
for k in ("edge", "x", "crossings", "counter", "m_hist", "totals"):
    out["inj_" + k] = r[k].cpu().numpy()
np.savez({path!r}, **out)
"""


def test_chunked_launches_equal_one_launch(tmp_path):
    """Calls large enough to overflow a block's 32-bit shared counters run as
    consecutive launches over particle-id chunks; GSDE_CHUNK_PARTICLES forces
    small chunks.  Estimators, per-particle arrays, the native resume path
    (state-in + Philox counters) and injected-draw rows must equal one launch."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for chunk in (None, "7777"):
        path = str(tmp_path / f"chunk_{chunk}.npz")
        env = dict(os.environ)
        env.pop("GSDE_CHUNK_PARTICLES", None)
        if chunk:
            env["GSDE_CHUNK_PARTICLES"] = chunk
        subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT.format(root=root, path=path)],
                       check=True, env=env, timeout=600)
        res[chunk] = np.load(path)
    a, b = res[None], res["7777"]
    assert sorted(a.files) == sorted(b.files) and len(a.files) >= 36
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


_UNI_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads
out = {{}}
for name, (g, f) in (("vasc", workloads.vascular(20_000, seed=5)), ("hub64", workloads.hub64())):
    grid = gs.EdgeGrid.uniform(g, 4)
    for cap in (100, 3):
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=200, n_particles=200_001, seed=3,
                                  initial=gs.PerEdgeUniform(float(g.edge_length.max())),
                                  max_splits_per_step=cap)
        for outs in (("edge_counts",), ("all", "edge_counts")):
            r = engine.ensemble_device(g, f, cfg, outputs=outs, grid=grid, occupation=(5, 2))
            for k, v in r.items():
                if not k.startswith("_") and v is not None:
                    out["%s_c%d_%d_%s" % (name, cap, len(outs), k)] = v.cpu().numpy()
# star vertex trials (C3's star5: equal jump weights), fused counts and per-trial arrays
g, f = workloads.star5("linear")
for per_trial in (False, True):
    r = engine.trials_device(g, f, 1e-3, 300_001, 7, per_trial=per_trial)
    for k, v in r.items():
        if not k.startswith("_") and v is not None:
            out["trials_%d_%s" % (per_trial, k)] = v.cpu().numpy()
np.savez({path!r}, **out)
"""


def test_uniform_exit_variant_equals_alias_pick(tmp_path):
    """Graphs whose every alias column keeps its own slot (equal jump weights at
    every vertex: C2, C4, C3's star) pick exits by the column alone; the result
    must equal the alias pick (GSDE_GENERIC_EXITS=1) bit for bit -- shared-memory
    and L2-resident tables, lean and per-particle, occupation, a truncating cap,
    and the star vertex trials."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for generic in (False, True):
        path = str(tmp_path / f"uni_{int(generic)}.npz")
        env = dict(os.environ)
        env.pop("GSDE_GENERIC_EXITS", None)
        if generic:
            env["GSDE_GENERIC_EXITS"] = "1"
        subprocess.run([sys.executable, "-c", _UNI_SCRIPT.format(root=root, path=path)],
                       check=True, env=env, timeout=600)
        res[generic] = np.load(path)
    a, b = res[False], res[True]
    assert sorted(a.files) == sorted(b.files) and len(a.files) >= 46
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)

