"""Host-side invariants of the run_ensemble transfer pipeline (CPU)."""
import numpy as np

from paper_2512_02175_b200 import engine


def test_pipeline_chunks_cover_every_particle_once():
    """run_ensemble's particle-id chunks: positive, shrinking, contiguous, covering the run."""
    ch = np.array(engine._CHUNKS)
    assert abs(ch.sum() - 1.0) < 1e-12
    assert np.all(ch > 0) and np.all(np.diff(ch) <= 0)
    for n in (engine._PIPELINE_MIN, engine._PIPELINE_MIN + 12_345, 16_000_000, 10**9 + 7):
        b = engine._chunk_bounds(n)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) > 0)
