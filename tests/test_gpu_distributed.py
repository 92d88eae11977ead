"""The multi-GPU API at world size 2 on a real GPU: two ranks share cuda:0 over
gloo (the driver's boxes have one GPU), each simulating its own global-id
shard through ``parallel.run_ensemble_distributed`` /
``parallel.exit_counts_distributed``.  The merged estimators and the
concatenated per-particle shards must equal a single-rank run bit for bit
(every particle is a pure function of (seed, global id),
the merge is an integer sum)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(gs):
    g, f = gs.workloads.hub64()
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=200, n_particles=200_003, seed=77,
                              initial=gs.PerEdgeUniform(2.0))
    return g, f, cfg, gs.EdgeGrid.uniform(g, 8)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2512_02175_b200 as gs
    from paper_2512_02175_b200 import parallel

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, f, cfg, grid = _case(gs)
        r = parallel.run_ensemble_distributed(g, f, cfg, grid=grid, particles=True)
        s5 = gs.workloads.star5("linear")
        ec = parallel.exit_counts_distributed(*s5, 1e-3, 400_001, 9)
        q.put((rank, {
            "m_hist": r.m_histogram, "crossings": r.crossings_total,
            "events": r.crossing_events, "truncs": r.truncation_count,
            "edge_counts": r.edge_counts, "hist": r.histogram, "shard": r.shard,
            "particles": r.particles,
            "exit_counts": ec.counts, "exit_m": ec.m_histogram,
            "exit_totals": (ec.crossings_total, ec.crossing_events, ec.truncation_count),
        }))
    finally:
        dist.destroy_process_group()


def test_world2_shared_gpu_equals_single_rank():
    import torch.multiprocessing as mp

    import paper_2512_02175_b200 as gs
    from paper_2512_02175_b200 import analysis, parallel

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    g, f, cfg, grid = _case(gs)
    single = parallel.run_ensemble_distributed(g, f, cfg, grid=grid)  # world 1
    ref = gs.run_ensemble(g, f, cfg)
    ec1 = analysis.vertex_exit_counts(*gs.workloads.star5("linear"), 1e-3, 400_001, 9)
    # both shards together cover every global id once
    assert got[0]["shard"] == (0, 100_002) and got[1]["shard"] == (100_002, 100_001)
    for rank in (0, 1):
        r = got[rank]
        np.testing.assert_array_equal(r["m_hist"], single.m_histogram)
        np.testing.assert_array_equal(r["m_hist"], ref.stats.m_histogram)
        assert (r["crossings"], r["events"], r["truncs"]) == (
            single.crossings_total, single.crossing_events, single.truncation_count)
        np.testing.assert_array_equal(r["edge_counts"], single.edge_counts)
        np.testing.assert_array_equal(r["hist"], single.histogram)
        assert int(r["hist"].sum()) == cfg.n_particles
        np.testing.assert_array_equal(r["exit_counts"], ec1.counts)
        np.testing.assert_array_equal(r["exit_m"], ec1.m_histogram)
        assert r["exit_totals"] == (ec1.crossings_total, ec1.crossing_events,
                                    ec1.truncation_count)
    # the per-particle shards, concatenated, are the single-rank run_ensemble arrays
    for key, arr in (("edges", ref.edges), ("positions", ref.positions),
                     ("crossings", ref.crossings), ("crossing_events", ref.crossing_events)):
        cat = np.concatenate([got[0]["particles"][key], got[1]["particles"][key]])
        np.testing.assert_array_equal(cat, arr, err_msg=key)
    np.testing.assert_array_equal(np.bincount(ref.edges, minlength=g.n_edges), single.edge_counts)
