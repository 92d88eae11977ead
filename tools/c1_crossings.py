"""C1 crossing rate per particle-step: driftless kernel vs generic native kernel vs the
reference stream, batch means with standard errors (statistical check of the ZD variant)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_02175_b200 as gs

g = gs.build_graph([(0, None, float("inf"))] * 3)
for label, mu, rng, n, batches in (("native ZD", 0.0, "native", 100_000_000, 10),
                                   ("native generic (mu=1e-30)", 1e-30, "native", 100_000_000, 10),
                                   ("reference stream", 0.0, "reference", 10_000_000, 10)):
    f = gs.CoefficientField.for_graph(g, [gs.ConstantDrift(mu)] * 3, [1.0] * 3)
    rates = []
    for b in range(batches):
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=1000, n_particles=n, seed=1000 + b, rng=rng)
        r = gs.run_ensemble(g, f, cfg) if n <= 10_000_000 else None
        if r is None:
            from paper_2512_02175_b200 import engine
            d = engine.ensemble_device(g, f, cfg, outputs=())
            c = int(d["totals"][0])
        else:
            c = r.stats.crossings_total
        rates.append(c / (n * 1000))
    rates = np.array(rates)
    print(f"{label}: crossings/pstep {rates.mean():.7f} +- {rates.std(ddof=1) / np.sqrt(len(rates)):.7f}")
