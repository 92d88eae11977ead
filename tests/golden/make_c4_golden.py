"""C4 golden run at its real scale, produced by the REFERENCE package itself.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_c4_golden.py

The synthetic vascular network of BASELINE config 4 (workloads.vascular():
1e5 nodes -> kNN -> MST -> +2% loops, ~1.02e5 edges) is emitted through the
graph-file format and parsed by the reference's own parser
(graphfile.py:69-186, :269-296); graphsde.run_ensemble (engine.py:273-352)
then runs 20000 particles x 100 steps (dt 1e-3, PerEdgeUniform(max length),
seed 20251202) in its reference streams.  Writes tests/golden/c4.npz: the
per-particle outputs, the M histogram and totals, and a SHA-256 of the parsed
graph's packed arrays (the GPU test regenerates the graph and first checks it
is the same graph).
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "graphsde")):
        sys.path.insert(0, p)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsde_numba_cache")

import graphsde as R  # noqa: E402
import graphsde.graphfile  # noqa: E402,F401

from paper_2512_02175_b200 import workloads  # noqa: E402  (tables only: plain arrays)

N, STEPS, DT, SEED = 20_000, 100, 1e-3, 20251202


def graph_digest(g, f) -> str:
    h = hashlib.sha256()
    for a in (g.edge_init, g.edge_term, g.edge_length, g.v_off, g.v_edges, g.v_orient,
              g.v_cumw) + tuple(f.packed()):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    g, f = workloads.vascular(api=R)
    cfg = R.SimulationConfig(dt=DT, n_steps=STEPS, n_particles=N, seed=SEED,
                             initial=R.PerEdgeUniform(float(g.edge_length.max())), workers=8)
    r = R.run_ensemble(g, f, cfg)
    np.savez_compressed(
        os.path.join(HERE, "c4.npz"), edges=r.edges, positions=r.positions,
        crossings=r.crossings, crossing_events=r.crossing_events,
        m_histogram=r.stats.m_histogram,
        stats=np.array([r.stats.truncation_count, r.stats.crossings_total,
                        r.stats.crossing_events]),
        gamma=np.array([r.stats.gamma]), n_edges=np.array([g.n_edges]),
        digest=np.array([graph_digest(g, f)]),
        meta=np.array([N, STEPS, SEED]), dt=np.array([DT]))
    print("c4.npz:", g.n_edges, "edges,", r.stats.crossings_total, "crossings")


if __name__ == "__main__":
    main()
