"""Run a fixed set of ensembles (+ per-particle arrays) with the libgsde.so that
GSDE_LIB_PATH selects and save every output, or compare two saved runs: two
builds whose kernels must agree bit for bit (e.g. a kernel variant chosen by
graph properties vs the generic kernel it replaces).

    GSDE_LIB_PATH=a.so python tools/lib_equal.py out_a.npz
    python tools/lib_equal.py --compare out_a.npz out_b.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    assert sorted(a.files) == sorted(b.files)
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("lib_equal:", "IDENTICAL" if not bad else f"DIFFER {bad}", f"({len(a.files)} arrays)")
    sys.exit(1 if bad else 0)

import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads

out = {}
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
                out[f"c{cap}_{len(outs)}_{k}"] = v.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", len(out), "arrays")
