"""C3 at scale, native FP32 stream vs the reference's own stream on the GPU:
the §4.1 star's dt sweep, 1e10 native trials and 1e9 reference-stream trials
per dt; per-edge exit frequencies and mean M with their z-scores (difference
over the combined binomial / sample standard error).

    python tools/trials_scale_check.py out.csv
"""
import csv
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2512_02175_b200 import analysis, workloads

g, f = workloads.star5("linear")
rows = []
worst = 0.0
for i, dt in enumerate((1e-2, 1e-3, 1e-4, 1e-5)):
    t0 = time.time()
    nat = analysis.vertex_exit_counts(g, f, dt, 10_000_000_000, 101 + i, rng="native")
    t1 = time.time()
    ref = analysis.vertex_exit_counts(g, f, dt, 1_000_000_000, 201 + i, rng="reference")
    t2 = time.time()
    pn, pr = nat.counts / nat.trials, ref.counts / ref.trials
    se = np.sqrt(pn * (1 - pn) / nat.trials + pr * (1 - pr) / ref.trials)
    z = (pn - pr) / se
    mh_n, mh_r = nat.m_histogram, ref.m_histogram
    b = np.arange(mh_n.shape[0])
    mn, mr = (b * mh_n).sum() / mh_n.sum(), (b * mh_r).sum() / mh_r.sum()
    vn = ((b - mn) ** 2 * mh_n).sum() / mh_n.sum()
    vr = ((b - mr) ** 2 * mh_r).sum() / mh_r.sum()
    zm = (mn - mr) / np.sqrt(vn / nat.trials + vr / ref.trials)
    worst = max(worst, float(np.abs(z).max()), abs(float(zm)))
    for e in range(g.n_edges):
        rows.append([dt, e, pn[e], pr[e], se[e], z[e]])
    rows.append([dt, "meanM", mn, mr, np.sqrt(vn / nat.trials + vr / ref.trials), zm])
    print(f"dt={dt:g}: native {t1 - t0:.1f} s ({nat.trials / (t1 - t0):.3g} trials/s), "
          f"reference {t2 - t1:.1f} s; max |z| exits {np.abs(z).max():.2f}, mean M z {zm:.2f}",
          flush=True)
with open(sys.argv[1] if len(sys.argv) > 1 else "trials_scale.csv", "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["dt", "edge", "native_freq", "reference_freq", "se", "z"])
    w.writerows(rows)
print(f"worst |z| over {len(rows)} comparisons: {worst:.2f}")
