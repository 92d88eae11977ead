"""Time one large hub64 call (1e9 particles x 1000 steps = 1e12 psteps): past the
32-bit shared-counter bound, so it runs as particle-id chunks (default) or, with
GSDE_CHUNK_PARTICLES=1000000000000, as one FULL launch with global counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads

g, f = workloads.hub64()
cfg = gs.SimulationConfig(dt=1e-3, n_steps=1000, n_particles=1_000_000_000, seed=1,
                          initial=gs.PerEdgeUniform(2.0))
grid = gs.EdgeGrid.uniform(g, 8)
engine.ensemble_device(g, f, gs.SimulationConfig(dt=1e-3, n_steps=10, n_particles=10**6, seed=1,
                                                 initial=gs.PerEdgeUniform(2.0)),
                       outputs=("edge_counts",), grid=grid)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = engine.ensemble_device(g, f, cfg, outputs=("edge_counts",), grid=grid)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"hub64 1e9 x 1000 ({os.environ.get('GSDE_CHUNK_PARTICLES', 'default chunks')}): "
      f"{el:.2f} s -> {1e12 / el:.4g} psteps/s; totals {r['totals'].cpu().numpy().tolist()} "
      f"hist sum {int(r['hist'].sum())}")
