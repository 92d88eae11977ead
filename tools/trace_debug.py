"""Per-step trace of the production kernel (injected draws, chained state-in
single steps) vs the oracle for the particles whose trajectories diverge:
prints the steps around the first divergence (edge, x, M, draw counter, FP64
decision margin).  python tools/trace_debug.py star4_mixed 150 0.01 uniform 0.2 5 0"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import helpers  # noqa: E402
import paper_2512_02175_b200 as gs  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2512_02175_b200 import engine  # noqa: E402

case, steps, dt, ik, iv, cap, wall = sys.argv[1:8]
steps, dt, cap, wall = int(steps), float(dt), int(cap), float(wall)
init = (ik, float(iv)) if ik == "uniform" else (ik, int(iv))
g, f = helpers.graph_for(case)
n, seed = 1024, 20251202
og = oracle.OracleGraph(g, f)
ref = oracle.trace(og, seed, n, steps, dt, helpers.oracle_init(init, g), cap, wall)
K = 2 * cap + 4
inj = lambda r, m: (torch.as_tensor(r.view(np.int64)).cuda(), torch.as_tensor(m).cuda())
cfg1 = gs.SimulationConfig(dt=dt, n_steps=1, n_particles=n, seed=seed, max_splits_per_step=cap,
                           initial=helpers.initial_for(init), reflect_at=wall)
raw, nrm = oracle.fill_draws(seed, n, K + 2)
res = engine.ensemble_device(g, f, cfg1, outputs=("all", "counter"), inject=inj(raw, nrm),
                             precision="native")
E = np.zeros((n, steps), np.int64); X = np.zeros((n, steps)); M = np.zeros((n, steps), np.int64)
KK = np.zeros((n, steps), np.uint64); k = np.zeros(n, np.uint64)
for s in range(steps):
    if s:
        raw, nrm = oracle.fill_draws_rows(np.full(n, seed, np.uint64), np.arange(n, dtype=np.uint64), k, K)
        cfg = gs.SimulationConfig(dt=dt, n_steps=1, n_particles=n, seed=seed,
                                  max_splits_per_step=cap, reflect_at=wall)
        res = engine.ensemble_device(g, f, cfg, outputs=("all", "counter"), inject=inj(raw, nrm),
                                     precision="native", state=(res["edge"], res["x"]))
    k = k + res["counter"].cpu().numpy().astype(np.uint64)
    E[:, s] = res["edge"].cpu().numpy(); X[:, s] = res["x"].cpu().numpy()
    M[:, s] = res["crossings"].cpu().numpy(); KK[:, s] = k
same = (E == ref["edge"]) & (M == ref["M"]) & (KK == ref["k"])
for i in np.flatnonzero(~same.all(axis=1)):
    s0 = int(np.argmin(same[i]))
    print(f"particle {i}: first divergence at step {s0}")
    for s in range(max(0, s0 - 6), min(steps, s0 + 2)):
        print(f"  s={s}: ref e={ref['edge'][i, s]} x={ref['x'][i, s]:.9g} M={ref['M'][i, s]} "
              f"k={ref['k'][i, s]} trunc={ref['trunc'][i, s]} margin={ref['margin'][i, s]:.3g} | "
              f"gpu e={E[i, s]} x={X[i, s]:.9g} M={M[i, s]} k={KK[i, s]}")
sig = f.packed()[5]
scale = np.maximum(np.abs(ref["x"]), sig[ref["edge"]] * np.sqrt(dt))
xbad = np.abs(X - ref["x"]) > 1e-5 * scale
for i in np.flatnonzero(xbad.any(axis=1))[:6]:
    s0 = int(np.argmax(xbad[i]))
    print(f"particle {i}: first |dx| > 1e-5 at step {s0}")
    for s in range(max(0, s0 - 3), min(steps, s0 + 2)):
        print(f"  s={s}: ref e={ref['edge'][i, s]} x={ref['x'][i, s]:.9g} M={ref['M'][i, s]} "
              f"k={ref['k'][i, s]} trunc={ref['trunc'][i, s]} margin={ref['margin'][i, s]:.3g} | "
              f"gpu e={E[i, s]} x={X[i, s]:.9g} M={M[i, s]} k={KK[i, s]}")
print("particles with |dx| > 1e-5 somewhere:", int(xbad.any(axis=1).sum()), "of", n)
