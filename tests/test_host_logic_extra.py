"""Host-side invariants of the run_ensemble transfer pipeline (CPU)."""
import numpy as np

from paper_2512_02175_b200 import engine


def test_pipeline_chunks_cover_every_particle_once():
    """run_ensemble's particle-id chunks: positive, contiguous, covering the run, for
    both schedules (kernel-bound: shrinking; transfer-bound: small first chunk)."""
    for ch in (np.array(engine._CHUNKS), np.array(engine._CHUNKS_TRANSFER_BOUND)):
        assert abs(ch.sum() - 1.0) < 1e-12 and np.all(ch > 0)
    assert np.all(np.diff(engine._CHUNKS) <= 0)
    assert engine._CHUNKS_TRANSFER_BOUND[0] < engine._CHUNKS[0]
    for steps in (1, 100, 255, 256, 1000):
        for n in (engine._PIPELINE_MIN, engine._PIPELINE_MIN + 12_345, 16_000_000, 10**9 + 7):
            b = engine._chunk_bounds(n, steps)
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) > 0)
