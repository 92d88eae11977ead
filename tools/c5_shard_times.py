"""C5 strong-scaling proxy on one GPU: the per-rank shard of the 1e10-psteps C4
job (1e8 / N particles x 100 steps, global-id offset of rank N-1) timed alone for
N = 1, 2, 4, 8; per-rank kernel time x N / single-GPU time = the kernel's share of
strong-scaling efficiency (the one NCCL all-reduce of ~7.4 MB per step is not
included)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_02175_b200 import engine

g, f = bench._vascular_cached()
import paper_2512_02175_b200 as gs
grid = gs.EdgeGrid.uniform(g, 8)
base = None
s = torch.cuda.current_stream()
for N in (1, 2, 4, 8):
    n = 100_000_000 // N
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=100, n_particles=100_000_000, seed=20251202,
                              initial=gs.PerEdgeUniform(float(g.edge_length.max())))
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        engine.ensemble_device(g, f, cfg, pid_offset=(N - 1) * n, n_particles=n,
                               outputs=("edge_counts",), grid=grid, stream=s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts[1:])
    base = base or t
    print(f"N={N}: shard {n:.3g} particles, {t:.2f} ms -> kernel-level efficiency "
          f"{base / (N * t):.3f}", flush=True)
