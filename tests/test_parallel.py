"""N > 1 host logic on CPU: sharding + the single integer all-reduce, world
size 2 over gloo.  Each rank's shard is simulated by the oracle (test-side);
the merged estimators must equal a single-process run exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cases
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200.parallel import merge_estimators, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 10, 4097, 10**8 + 3):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (o1, c1), (o2, _) in zip(spans, spans[1:]):
                assert o1 + c1 == o2
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _estimators(g, f, seed, n, steps, dt, off, cnt, grid):
    from oracle import oracle

    o = oracle.ensemble(oracle.OracleGraph(g, f), seed, cnt, steps, dt, (1, 0, 0.0, 2.0), 100,
                        0.0, pid_offset=off)
    hist = oracle.histogram(o["edges"], o["positions"], grid.offsets, grid.counts, grid.dx)
    return dict(
        m_hist=torch.as_tensor(o["m_histogram"]),
        totals=torch.tensor([o["crossings"].sum(), o["crossing_events"].sum(),
                             o["truncs"].sum(), 0], dtype=torch.int64),
        edge_counts=torch.as_tensor(np.bincount(o["edges"], minlength=g.n_edges).astype(np.int64)),
        hist=torch.as_tensor(hist),
    )


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, f = cases.build("hub8", gs)
        grid = gs.EdgeGrid.uniform(g, 4)
        n = 5001
        off, cnt = shard_range(n, rank, world)
        parts = _estimators(g, f, 123, n, 50, 1e-2, off, cnt, grid)
        merged = merge_estimators(parts)
        q.put((rank, {k: v.numpy().copy() for k, v in merged.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_merge_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, f = cases.build("hub8", gs)
    grid = gs.EdgeGrid.uniform(g, 4)
    single = _estimators(g, f, 123, 5001, 50, 1e-2, 0, 5001, grid)
    for rank in (0, 1):
        for k, v in single.items():
            np.testing.assert_array_equal(got[rank][k], v.numpy(), err_msg=f"rank {rank} {k}")
    assert int(single["hist"].sum()) == 5001
