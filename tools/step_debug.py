"""One reference step of one particle through the production kernel vs the
oracle (injected draws, state-in).  python tools/step_debug.py CASE STEPS DT
INITKIND INITVAL CAP WALL PARTICLE STEP"""
import os
import sys

import numpy as np
import torch

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (R, os.path.join(R, "tests"), os.path.join(R, "tests", "golden")):
    sys.path.insert(0, p)
import helpers  # noqa: E402
import paper_2512_02175_b200 as gs  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2512_02175_b200 import engine  # noqa: E402

case, steps, dt, ik, iv, cap, wall, pi, si = sys.argv[1:10]
steps, dt, cap, wall, pi, si = int(steps), float(dt), int(cap), float(wall), int(pi), int(si)
init = (ik, float(iv)) if ik == "uniform" else (ik, int(iv))
g, f = helpers.graph_for(case)
n, seed = pi + 1, 20251202
og = oracle.OracleGraph(g, f)
ref = oracle.trace(og, seed, n, steps, dt, helpers.oracle_init(init, g), cap, wall)
e0, x0, k0 = ref["edge"][pi, si - 1], ref["x"][pi, si - 1], ref["k"][pi, si - 1]
K = 2 * cap + 4
raw, nrm = oracle.fill_draws_rows(np.array([seed], np.uint64), np.array([pi], np.uint64),
                                  np.array([k0], np.uint64), K)
print("state", e0, repr(x0), "k", k0, "draws raw/normal:", [hex(int(r)) for r in raw[0, :6]],
      nrm[0, :6])
cfg = gs.SimulationConfig(dt=dt, n_steps=1, n_particles=1, seed=seed, max_splits_per_step=cap,
                          reflect_at=wall)
inj = (torch.as_tensor(raw.view(np.int64)).cuda(), torch.as_tensor(nrm).cuda())
res = engine.ensemble_device(g, f, cfg, outputs=("all", "counter"), inject=inj,
                             precision="native",
                             state=(torch.tensor([e0]), torch.tensor([x0])))
for prec in ("f32", "f64"):
    r2 = engine.step_batch(g, f, torch.tensor([e0]).cuda(), torch.tensor([x0]).cuda(), dt, None,
                           None, torch.tensor([0]).cuda(), cap, wall, inject=inj, precision=prec)
    print(f"reference-order stepper {prec}: edge {int(r2[0][0])} x {float(r2[1][0])!r} "
          f"M {int(r2[2][0])} trunc {int(r2[3][0])} k {int(r2[4][0])}")
print("oracle : edge", ref["edge"][pi, si], "x", repr(ref["x"][pi, si]), "M", ref["M"][pi, si],
      "k", ref["k"][pi, si], "margin", ref["margin"][pi, si])
print("kernel : edge", int(res["edge"][0]), "x", repr(float(res["x"][0])), "M",
      int(res["crossings"][0]), "used", int(res["counter"][0]))
