"""Multi-GPU ensembles: particle sharding + one integer all-reduce.

Particles are independent and every particle is a pure function of
``(seed, global particle id)`` (reference ``rng.py:1-11``, ``SPEC.md:238``),
so the path shards without any data-path exchange: rank ``r`` of ``W``
simulates the contiguous global ids :func:`shard_range` gives it (the kernel
keys its streams by ``pid_offset + local index``), then ONE all-reduce (sum,
int64) merges the estimators -- M histogram, totals, final-edge occupancy and
the snapshot histogram.  Integer sums make the merged result identical to a
1-GPU run for any world size.

Backend: NCCL over NVLink for CUDA tensors; the same code runs under gloo on
CPU tensors (tests/test_parallel.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ESTIMATORS = ("m_hist", "totals", "edge_counts", "hist", "exit_counts")


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """``(offset, count)`` of rank ``rank``'s contiguous particle-id shard."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of size {world}")
    base, extra = divmod(int(n), int(world))
    offset = rank * base + min(rank, extra)
    return offset, base + (1 if rank < extra else 0)


def merge_estimators(parts: dict, group=None) -> dict:
    """All-reduce (sum) the integer estimator tensors of one rank in a single
    collective; returns the merged tensors (same keys, same device)."""
    import torch
    import torch.distributed as dist

    keys = [k for k in ESTIMATORS if k in parts and parts[k] is not None]
    flat = torch.cat([parts[k].reshape(-1).to(torch.int64) for k in keys])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    out, o = {}, 0
    for k in keys:
        n = parts[k].numel()
        out[k] = flat[o: o + n].view_as(parts[k])
        o += n
    return out


@dataclass(frozen=True)
class DistributedResult:
    m_histogram: np.ndarray
    crossings_total: int
    crossing_events: int
    truncation_count: int
    edge_counts: np.ndarray | None
    histogram: np.ndarray | None
    n_particles: int
    shard: tuple
    #: this rank's shard of the per-particle arrays (host numpy, reference
    #: dtypes) when asked for with ``particles=True``: edges, positions,
    #: crossings, crossing_events of global ids shard[0] .. shard[0]+shard[1]-1
    particles: dict | None = None


def run_ensemble_distributed(graph, field, config, grid=None, group=None,
                             edge_counts: bool = True,
                             particles: bool = False) -> DistributedResult:
    """Run ``config.n_particles`` particles sharded over the ranks of the
    default process group (one GPU per rank), estimators merged with one
    NCCL all-reduce.  Per-particle arrays stay on each rank's GPU unless
    ``particles=True``: then each rank copies its shard to (pinned) host
    memory through ``run_ensemble``'s chunked transfer pipeline -- the
    distributed form of ``run_ensemble``'s result."""
    import torch.distributed as dist

    from .engine import _check_ensemble_shape, _ensemble_to_host, ensemble_device

    config = config.validated(graph)
    _check_ensemble_shape(graph, config)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    off, cnt = shard_range(config.n_particles, rank, world)
    host = None
    if particles:
        arrs, res = _ensemble_to_host(graph, field, config, pid_offset=off, n_particles=cnt,
                                      grid=grid, edge_counts=edge_counts, estimators=True)
        host = dict(zip(("edges", "positions", "crossings", "crossing_events"), arrs))
    else:
        res = ensemble_device(graph, field, config, pid_offset=off, n_particles=cnt,
                              outputs=("edge_counts",) if edge_counts else (), grid=grid)
    merged = merge_estimators(res, group)
    tot = merged["totals"].cpu().numpy()
    return DistributedResult(
        m_histogram=merged["m_hist"].cpu().numpy(),
        crossings_total=int(tot[0]),
        crossing_events=int(tot[1]),
        truncation_count=int(tot[2]),
        edge_counts=merged["edge_counts"].cpu().numpy() if "edge_counts" in merged else None,
        histogram=merged["hist"].cpu().numpy() if "hist" in merged else None,
        n_particles=config.n_particles,
        shard=(off, cnt),
        particles=host,
    )


def exit_counts_distributed(graph, field, dt, n_trials, seed, vertex=0, max_splits=100,
                            rng="native", group=None):
    """Vertex trials (the estimator behind ``exit_probability_experiment``,
    reference ``analysis.py:348-384``) sharded by global trial id over the
    ranks; exit counts, M histogram and totals merged with one all-reduce.
    Identical to a 1-GPU :func:`analysis.vertex_exit_counts` for any world size."""
    import torch.distributed as dist

    from .analysis import ExitCounts
    from .coefficients import gamma as vgamma
    from .engine import trials_device

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    off, cnt = shard_range(n_trials, rank, world)
    res = trials_device(graph, field, dt, cnt, seed, vertex, max_splits, rng, per_trial=False,
                        trial_offset=off)
    merged = merge_estimators(res, group)
    tot = merged["totals"].cpu().numpy()
    return ExitCounts(merged["exit_counts"].cpu().numpy(), merged["m_hist"].cpu().numpy(),
                      int(n_trials), int(tot[0]), int(tot[1]), int(tot[2]),
                      vgamma(field, graph, vertex, dt))
