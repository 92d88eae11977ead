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


def test_streamed_copy_groups_cover_every_range_once():
    """engine._copy_groups: contiguous, complete, the last 8 ranges one by one."""
    from paper_2512_02175_b200 import engine

    for n_ranges in (1, 2, 7, 8, 9, 16, 17, 100, 256):
        groups = engine._copy_groups(n_ranges)
        flat = [r for a, b in groups for r in range(a, b)]
        assert flat == list(range(n_ranges))
        assert all(b - a == 1 for a, b in groups[-min(8, n_ranges):])
        assert all(b - a <= 8 for a, b in groups)
