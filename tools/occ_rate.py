"""Cost of the fused time-integrated occupation histogram (sample every step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads

for name, build, n, init, grid_fn in (
        ("star3", workloads.star3, 16_000_000, gs.AtVertex(0),
         lambda g: gs.EdgeGrid.uniform(g, 16, lengths=[3.0] * 3)),
        ("hub64", workloads.hub64, 20_000_000, gs.PerEdgeUniform(2.0),
         lambda g: gs.EdgeGrid.uniform(g, 8))):
    g, f = build()
    grid = grid_fn(g)
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=1000, n_particles=n, seed=3, initial=init)
    for occ in (None, (1, 0), (10, 0)):
        kw = dict(outputs=("edge_counts",), grid=grid, occupation=occ)
        engine.ensemble_device(g, f, cfg, **kw)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.ensemble_device(g, f, cfg, **kw)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        print(f"{name} occupation={occ} {n * 1000 / ms * 1e3:.3e} psteps/s ({ms:.1f} ms)")
