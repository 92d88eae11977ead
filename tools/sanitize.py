"""Small runs of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
import torch
import cases
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, engine, fvm, workloads

for case, init in (("star3_bm", gs.AtVertex(0)), ("hub8", gs.PerEdgeUniform(2.0)),
                   ("random_general", gs.PerEdgeUniform(1.0)), ("star4_mixed", gs.AtVertex(0))):
    g, f = cases.build(case, gs)
    grid = gs.EdgeGrid.uniform(g, 4, lengths=None if not g.is_star else [2.0] * g.n_edges)
    for rng in ("native", "reference"):
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=60, n_particles=3000, seed=1, rng=rng,
                                  initial=init)
        engine.ensemble_device(g, f, cfg, outputs=("all", "edge_counts"), grid=grid,
                               occupation=(1, 5))
        # the lean kernel (fused estimators only)
        engine.ensemble_device(g, f, cfg, outputs=("edge_counts",), grid=grid)
    if g.is_star or not g.has_semi_infinite_edges:
        for rng in ("native", "reference"):
            engine.trials_device(g, f, 1e-3, 5000, 3, rng=rng)
            engine.trials_device(g, f, 1e-3, 5000, 3, rng=rng, per_trial=False)
g, f = workloads.vascular(3000, seed=2)
grid = gs.EdgeGrid.uniform(g, 4)
cfg = gs.SimulationConfig(dt=1e-3, n_steps=30, n_particles=20000, seed=2,
                          initial=gs.PerEdgeUniform(float(g.edge_length.max())))
engine.ensemble_device(g, f, cfg, outputs=("edge_counts",), grid=grid)
# the production kernel under injected reference draws (INJECT/NATIVE), star + L2 graph
rs = np.random.default_rng(3)  # any draws will do for memory checking
for gg, ff, init, n in ((*cases.build("star3_bm", gs), gs.AtVertex(0), 2000),
                        (g, f, gs.PerEdgeUniform(float(g.edge_length.max())), 2000)):
    raw = rs.integers(0, 2**63, size=(n, 200), dtype=np.int64).view(np.uint64)
    nrm = rs.standard_normal((n, 200))
    inj = (torch.as_tensor(raw.view(np.int64)).cuda(), torch.as_tensor(nrm).cuda())
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=60, n_particles=n, seed=3, initial=init)
    engine.ensemble_device(gg, ff, cfg, inject=inj, precision="native")
gt, ft = cases.build("random_general", gs)  # trials, incl. tabulated drifts
raw = rs.integers(0, 2**63, size=(3000, 210), dtype=np.int64).view(np.uint64)
inj = (torch.as_tensor(raw.view(np.int64)).cuda(),
       torch.as_tensor(rs.standard_normal((3000, 210))).cuda())
engine.trials_device(gt, ft, 1e-3, 3000, 3, max_splits=100, inject=inj, precision="native")
# streamed results: per-particle kernels with progress counters (batched
# stores + publication) and the copy stream waiting on them
engine._PIPELINE_MIN = 1
for gg, ff, init in ((*cases.build("star3_bm", gs), gs.AtVertex(0)),
                     (g, f, gs.PerEdgeUniform(float(g.edge_length.max())))):
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=40, n_particles=30001, seed=4, initial=init)
    engine._ensemble_to_host(gg, ff, cfg)
    prog = torch.zeros(64, dtype=torch.int32, device="cuda")
    engine.ensemble_device(gg, ff, cfg, outputs=("all", "edge_counts"), grid=gs.EdgeGrid.uniform(
        gg, 4, lengths=None if not gg.is_star else [2.0] * gg.n_edges), progress=(prog, 9))
gs5, fs5 = workloads.star5("linear")  # C3's star: uniform-exit vertex trials
for per_trial in (False, True):
    engine.trials_device(gs5, fs5, 1e-3, 20000, 5, per_trial=per_trial)
gp, fp = cases.build("path3", gs)
gridp = gs.EdgeGrid(counts=np.array([3, 1]), lengths=gp.edge_length)
fvm.fvm_steps_device(gp, fp, gridp, np.linspace(1, 2, 4), 20, 0.5 * fvm.stability_limit(gp, fp, gridp))
gridv = gs.EdgeGrid(counts=np.full(g.n_edges, 9), lengths=g.edge_length)
fvm.fvm_steps_device(g, f, gridv, np.ones(gridv.n_cells), 3, 0.5 * fvm.stability_limit(g, f, gridv))
analysis.histogram_accumulate(np.zeros(100, np.int64), np.linspace(0, 1, 100), gs.EdgeGrid.uniform(gp, 5))
torch.cuda.synchronize()
print("sanitize workload done")
