"""Throughput of the bit-exact reference-stream kernels (FP64, AS241) on C1 and hub64."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads

for name, build, n, steps, init in (
        ("star3", workloads.star3, 2_000_000, 1000, gs.AtVertex(0)),
        ("hub64", workloads.hub64, 2_000_000, 1000, gs.PerEdgeUniform(2.0))):
    g, f = build()
    for rng in ("reference", "native"):
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=steps, n_particles=n, seed=3, rng=rng,
                                  initial=init)
        engine.ensemble_device(g, f, cfg, outputs=("edge_counts",))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.ensemble_device(g, f, cfg, outputs=("edge_counts",))
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        print(f"{name} {rng:9s} {n * steps / ms * 1e3:.3e} psteps/s ({ms:.1f} ms)")
