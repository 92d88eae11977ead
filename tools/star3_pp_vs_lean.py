"""star3 (C1 config): the lean kernel (fused estimators only) and the
per-particle kernel (run_ensemble's arrays), one launch each -- for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_02175_b200 import engine

wl = bench.make_workload("star3", 0, 1)
cfg = wl.cfg_single()
for outs in (("edge_counts",), ("edge", "x", "crossings", "events")):
    r = engine.ensemble_device(wl.g, wl.f, cfg, outputs=outs)
    torch.cuda.synchronize()
    del r
