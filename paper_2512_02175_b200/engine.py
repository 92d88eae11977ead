"""Public simulation API (reference ``graphsde/engine.py``), GPU-backed.

Same names, signatures, validation and exceptions as the reference:
``run_ensemble`` (``engine.py:273-352``), ``vertex_crossing_trials``
(``:391-441``), ``em_step_star`` / ``em_step_general`` (``:206-270``),
``solve_alpha`` (``:37-57``) and the config / result dataclasses.  The kernel
calls the reference makes into numba (``engine.py:309-328``, ``:411-433``,
``:221-227``, ``:255-262``) are replaced by ``libgsde.so`` calls.

Two additions, both keyword-only or defaulted so reference call sites work
unchanged:

* ``SimulationConfig.rng`` -- ``"native"`` (default; the B200 FP32 production
  stream: statistically equivalent to the reference) or ``"reference"``
  (the reference's own Philox/AS241 streams in FP64: bit-compatible edge
  ids, crossing counts and truncations, positions to ~1e-11);
* ``SimulationConfig.device`` -- CUDA device index (default: current).

``workers`` is accepted and validated for compatibility; it has no effect
(results never depended on it).
"""

from __future__ import annotations

import dataclasses
import math
import os
from dataclasses import dataclass, field as dataclass_field

import numpy as np

from . import _native
from .coefficients import CoefficientField, gamma, graph_gamma
from .graph import AT_INIT, MetricGraph, VertexId
from .rng import RngStream

DEFAULT_MAX_SPLITS = 100
RNG_MODES = ("native", "reference")


class ConfigInvalid(ValueError):
    pass


class NoRootInUnitInterval(ValueError):
    """The partial-step quadratic has no first-passage root in [0, 1]."""


def solve_alpha(a: float, b: float, c: float) -> float:
    """``alpha = s**2`` for the first-passage root of ``a s^2 + b s + c``
    (reference ``engine.py:37-57``; the root comes from the same
    ``solve_first_passage_s`` the kernels use)."""
    s = float(_native.lib().gsde_solve_first_passage_s(float(a), float(b), float(c)))
    if s < 0.0:
        raise NoRootInUnitInterval(f"no first-passage root in [0, 1] for a={a!r}, b={b!r}, c={c!r}")
    residual = abs(a * s * s + b * s + c)
    scale = max(abs(a), abs(b), abs(c), 1.0)
    if residual > 1e-6 * scale and not (s == 1.0 or s == 0.0):
        raise NoRootInUnitInterval(
            f"first-passage root failed the residual check: s={s!r}, residual={residual!r}"
        )
    return s * s


@dataclass
class ParticleState:
    edge: int
    x: float
    crossings_total: int = 0
    crossing_events: int = 0


@dataclass(frozen=True)
class StepOutcome:
    state: ParticleState
    crossings_this_step: int
    truncated: bool


@dataclass(frozen=True)
class AtVertex:
    vertex: VertexId = 0


@dataclass(frozen=True)
class PointStart:
    edge: int
    x: float


@dataclass(frozen=True)
class PerEdgeUniform:
    x_max: float


InitialDistribution = AtVertex | PointStart | PerEdgeUniform


@dataclass(frozen=True)
class SimulationConfig:
    dt: float
    n_steps: int
    n_particles: int
    seed: int
    max_splits_per_step: int = DEFAULT_MAX_SPLITS
    initial: InitialDistribution = dataclass_field(default_factory=AtVertex)
    workers: int = 1
    reflect_at: float = 0.0
    rng: str = "native"
    device: int | None = None
    #: run_ensemble only: shard the particles (by global id) over these GPUs from
    #: one process; results are identical to one device
    devices: tuple | None = None

    def validated(self, graph: MetricGraph) -> "SimulationConfig":
        """Reference checks (``engine.py:114-139``) plus the ``rng`` mode."""
        if not (self.dt > 0.0 and math.isfinite(self.dt)):
            raise ConfigInvalid(f"dt must be positive and finite, got {self.dt!r}")
        if self.n_steps < 0 or self.n_particles < 0:
            raise ConfigInvalid("n_steps and n_particles must be nonnegative")
        if self.max_splits_per_step < 1:
            raise ConfigInvalid("max_splits_per_step must be at least 1")
        if self.workers < 1:
            raise ConfigInvalid("workers must be at least 1")
        if self.reflect_at < 0.0:
            raise ConfigInvalid("reflect_at must be nonnegative")
        if self.rng not in RNG_MODES:
            raise ConfigInvalid(f"rng must be one of {RNG_MODES}, got {self.rng!r}")
        if self.devices is not None and (len(self.devices) < 1 or
                                         any(int(d) < 0 for d in self.devices)):
            raise ConfigInvalid("devices must be a non-empty sequence of device indices")
        init = self.initial
        if isinstance(init, AtVertex):
            if not (0 <= init.vertex < graph.n_vertices):
                raise ConfigInvalid(f"initial vertex {init.vertex} out of range")
        elif isinstance(init, PointStart):
            if not (0 <= init.edge < graph.n_edges):
                raise ConfigInvalid(f"initial edge {init.edge} out of range")
            if not (0.0 <= init.x <= float(graph.edge_length[init.edge])):
                raise ConfigInvalid(f"initial position {init.x!r} outside the edge")
        elif isinstance(init, PerEdgeUniform):
            if not (init.x_max > 0.0 and math.isfinite(init.x_max)):
                raise ConfigInvalid("PerEdgeUniform needs a positive finite x_max")
        else:
            raise ConfigInvalid(f"unknown initial distribution {init!r}")
        return self


@dataclass(frozen=True)
class BounceStats:
    """Vertex-crossing statistics of a run (reference ``engine.py:142-166``)."""

    m_histogram: np.ndarray
    gamma: float
    truncation_count: int
    crossings_total: int
    crossing_events: int

    @property
    def vertex_steps(self) -> int:
        return int(self.m_histogram.sum())

    def cdf(self, k: int) -> float:
        n = self.vertex_steps
        if n == 0:
            return 1.0
        return float(self.m_histogram[: k + 1].sum()) / n


@dataclass(frozen=True)
class EnsembleResult:
    edges: np.ndarray
    positions: np.ndarray
    crossings: np.ndarray
    crossing_events: np.ndarray
    stats: BounceStats
    config: SimulationConfig


def available_workers() -> int:
    """Reference ``engine.py:186-187`` (numba's thread count).  ``workers`` has
    no effect here (the GPU runs every particle at once); this reports the
    host's CPU count so reference code sizing its ``workers`` keeps working."""
    import os

    return int(os.cpu_count() or 1)


def _resolve_initial(graph: MetricGraph, init: InitialDistribution):
    """Initial distribution -> placement code (reference ``engine.py:194-203``)."""
    if isinstance(init, AtVertex):
        lo = int(graph.v_off[init.vertex])
        e = int(graph.v_edges[lo])
        return _native.GSDE_INIT_POINT, e, graph.vertex_position(e, int(graph.v_orient[lo])), 0.0
    if isinstance(init, PointStart):
        return _native.GSDE_INIT_POINT, int(init.edge), float(init.x), 0.0
    return _native.GSDE_INIT_PER_EDGE_UNIFORM, 0, 0.0, float(init.x_max)


def _stream_code(rng: str) -> int:
    return _native.GSDE_STREAM_NATIVE if rng == "native" else _native.GSDE_STREAM_REFERENCE


def _check_ensemble_shape(graph: MetricGraph, config: SimulationConfig) -> None:
    if not graph.is_star and graph.has_semi_infinite_edges:
        raise ConfigInvalid(
            "general ensembles require finite edge lengths; semi-infinite "
            "edges are only supported on star graphs"
        )
    if config.reflect_at > 0.0 and not graph.is_star:
        raise ConfigInvalid("reflect_at applies to star graphs only")


def ensemble_device(graph, field, config, *, pid_offset=0, n_particles=None, outputs=("all",),
                    grid=None, inject=None, precision="f32", stream=None, occupation=None,
                    state=None, progress=None):
    """Run an ensemble and return DEVICE tensors (no host copies).

    ``outputs``: any of ``"edge", "x", "crossings", "events", "truncs"`` or
    ``"all"``; ``m_hist`` / ``totals`` are always produced, ``edge_counts``
    when ``"edge_counts"`` is listed, the snapshot histogram when ``grid``
    (an :class:`EdgeGrid`) is given.  ``pid_offset`` / ``n_particles`` select
    a shard of global particle ids (multi-GPU).  ``inject=(raw, normal)``
    (device uint64 / float64 tensors ``[n, K]``) selects the injected-draw
    stream with ``precision`` ``"f32"`` or ``"f64"`` (the reference-order
    stepper in that precision) or ``"native"`` (the production FP32 kernel
    itself, fed one injected draw per use).  ``occupation=(every,
    start)`` (needs ``grid``) adds the time-integrated occupation histogram
    ``res["occ"]``: every particle's (edge, x) binned after every
    ``every``-th completed macro step beyond step ``start``.

    ``state=(edge, x[, counter])`` (device tensors ``[n]``) starts particle
    ``i`` from ``(edge[i], x[i])`` instead of ``config.initial`` -- the batched
    ``ParticleState`` of ``em_step_*`` (``engine.py:60-67``): the production
    kernel reads it as SoA (int32 edges, float32 positions) with coalesced
    loads.  With the native stream ``counter`` (uint64 as int64) is each
    particle's next Philox block -- ``res["counter"]`` of the run being
    resumed (``outputs`` incl. ``"counter"``); with ``inject`` and
    ``precision="native"`` the injected rows start at the state's draw and
    ``res["counter"]`` counts the draws each particle consumed.  Native /
    injected-native streams only.

    ``progress=(counters, shift)`` (a zeroed device int32 tensor) streams the
    per-particle arrays: the kernel adds 1 to ``counters[i >> shift]`` once
    particle ``i``'s outputs are stored, so a copy stream can wait for a
    range (``gsde_stream_wait_geq32``) while the launch still runs.
    """
    torch, dev = _native.torch_cuda(config.device)
    n = config.n_particles if n_particles is None else int(n_particles)
    cap = config.max_splits_per_step
    dg = _native.device_graph(graph, field, dev)
    kw = dict(device=f"cuda:{dev}")
    want = set(outputs)
    full = "all" in want
    res = {}

    def maybe(name, dtype):
        if full or name in want:
            res[name] = torch.empty(n, dtype=dtype, **kw)
            return res[name]
        return None

    e_t, x_t = maybe("edge", torch.int64), maybe("x", torch.float64)
    k_t = res["counter"] = torch.empty(n, dtype=torch.int64, **kw) if "counter" in want else None
    c_t, ev_t, tr_t = (maybe("crossings", torch.int64), maybe("events", torch.int64),
                       maybe("truncs", torch.int64))
    res["m_hist"] = torch.zeros(cap + 1, dtype=torch.int64, **kw)
    res["totals"] = torch.zeros(4, dtype=torch.int64, **kw)
    ec_t = None
    if "edge_counts" in want:
        ec_t = res["edge_counts"] = torch.zeros(graph.n_edges, dtype=torch.int64, **kw)
    o = _native.Out()
    for k, t in (("edge", e_t), ("x", x_t), ("crossings", c_t), ("events", ev_t),
                 ("truncs", tr_t), ("m_hist", res["m_hist"]), ("totals", res["totals"]),
                 ("edge_counts", ec_t), ("counter", k_t)):
        setattr(o, k, _native.ptr(t))
    if occupation is not None and grid is None:
        raise ConfigInvalid("the occupation histogram needs a grid")
    if grid is not None:
        res["hist"] = torch.zeros(grid.n_cells, dtype=torch.int64, **kw)
        g_off, g_cnt, g_dx = grid.device_arrays(torch, dev)
        res["_grid"] = (g_off, g_cnt, g_dx)
        o.hist, o.hist_offsets, o.hist_counts, o.hist_dx = (
            res["hist"].data_ptr(), g_off.data_ptr(), g_cnt.data_ptr(), g_dx.data_ptr())
        o.hist_n_cells = grid.n_cells
        if occupation is not None:
            every, start = (int(v) for v in occupation)
            if every < 1 or start < 0:
                raise ConfigInvalid("occupation needs every >= 1 and start >= 0")
            res["occ"] = torch.zeros(grid.n_cells, dtype=torch.int64, **kw)
            o.occ, o.occ_every, o.occ_start = res["occ"].data_ptr(), every, start
    init_kind, init_edge, init_x, init_xmax = _resolve_initial(graph, config.initial)
    r = _native.Run()
    r.seed = int(config.seed) & 0xFFFFFFFFFFFFFFFF
    r.n_particles = n
    r.pid_offset = int(pid_offset)
    r.n_steps = config.n_steps
    r.dt = config.dt
    r.init_kind, r.init_edge, r.init_x, r.init_xmax = init_kind, init_edge, init_x, init_xmax
    r.cap = cap
    r.reflect_len = config.reflect_at
    r.stream = _stream_code(config.rng)
    if inject is not None:
        raw, nrm = inject
        r.stream = _native.GSDE_STREAM_INJECT
        r.precision = {"f64": _native.GSDE_PREC_F64, "f32": _native.GSDE_PREC_F32,
                       "native": _native.GSDE_PREC_NATIVE}[precision]
        r.inj_raw, r.inj_normal, r.inj_stride = raw.data_ptr(), nrm.data_ptr(), raw.shape[1]
    if state is not None:
        se = state[0].to(device=f"cuda:{dev}", dtype=torch.int32).contiguous()
        sx = state[1].to(device=f"cuda:{dev}", dtype=torch.float32).contiguous()
        if se.shape[0] != n or sx.shape[0] != n:
            raise ConfigInvalid(f"state arrays must have n_particles = {n} entries")
        res["_state"] = (se, sx)  # alive until the launch is queued
        r.init_kind = _native.GSDE_INIT_STATE
        r.state_edge, r.state_x = se.data_ptr(), sx.data_ptr()
        if len(state) > 2 and state[2] is not None:
            sk = state[2].to(device=f"cuda:{dev}", dtype=torch.int64).contiguous()
            res["_state"] += (sk,)
            r.state_counter = sk.data_ptr()
    if progress is not None:
        o.progress, o.progress_base, o.progress_shift = progress[0].data_ptr(), 0, int(progress[1])
    s = stream if stream is not None else _native.cur_stream(dev)
    _native.check(_native.lib().gsde_ensemble(dg.handle, r, o, s))
    return res


def run_ensemble(graph: MetricGraph, field: CoefficientField,
                 config: SimulationConfig) -> EnsembleResult:
    """Drive ``n_particles`` independent particles for ``n_steps`` steps on
    the GPU (reference ``engine.py:273-352``).  Deterministic in
    ``(seed, config)``; with ``rng="reference"`` the edge ids, crossing counts
    and M histogram equal the reference's exactly."""
    config = config.validated(graph)
    _check_ensemble_shape(graph, config)
    n = config.n_particles
    run_gamma = graph_gamma(field, graph, config.dt)
    cap = config.max_splits_per_step
    if n == 0:
        z = np.zeros(0, np.int64)
        stats = BounceStats(np.zeros(cap + 1, np.int64), run_gamma, 0, 0, 0)
        return EnsembleResult(z, np.zeros(0), z.copy(), z.copy(), stats, config)
    if config.devices is not None and len(config.devices) > 1:
        edges, positions, crossings, events, m_hist, totals = _multi_device(graph, field,
                                                                           config)
    else:
        if config.devices is not None:
            config = dataclasses.replace(config, device=int(config.devices[0]))
        edges, positions, crossings, events, m_hist, totals = _ensemble_to_host(graph, field,
                                                                               config)
    stats = BounceStats(
        m_histogram=m_hist,
        gamma=run_gamma,
        truncation_count=int(totals[2]),
        crossings_total=int(totals[0]),
        crossing_events=int(totals[1]),
    )
    return EnsembleResult(edges, positions, crossings, events, stats, config)


#: Particle-count split of a large run_ensemble call: chunk k's device->host
#: copy of the per-particle arrays overlaps chunk k+1's kernel; chunks shrink
#: about geometrically (each copy still hides behind the next kernel: D2H moves
#: a chunk ~2.7x faster than the kernel makes it), so the exposed copy of the
#: last one is small.  C1 run_ensemble: (0.4, 0.3, 0.2, 0.1) 26.6 ms, these 25.9.
# Chunk schedules (fractions of the particle ids).  Kernel-bound runs (a
# particle's steps take longer than its 32 B of D2H at ~55 GB/s: roughly
# n_steps >= 256 at 3-7e11 psteps/s) want a large first chunk and a small last
# one (the copies hide under the next kernels); transfer-bound runs want a
# small first chunk, so the copy engine starts early.  Measured (ms per
# run_ensemble, one B200): star3 1.6e7 x 1000: 25.5 (kernel-bound schedule) vs
# 26.0; hub64 1e8 x 1000: 267.2 vs 268.2; vascular 1e8 x 100: 88.9 vs 76.7.
_CHUNKS = (0.55, 0.25, 0.12, 0.055, 0.02, 0.005)  # (0.5, .28, .14, .06, .02): +0.3%
_CHUNKS_TRANSFER_BOUND = (0.08, 0.22, 0.3, 0.25, 0.12, 0.03)
_PIPELINE_MIN = 1 << 22
_COPY_STREAMS: dict = {}  # device -> (copy stream, second launch stream)


def _chunk_bounds(n: int, n_steps: int = 1000) -> np.ndarray:
    """Particle-id boundaries of run_ensemble's chunks: [0, ..., n]."""
    fr = _CHUNKS if n_steps >= 256 else _CHUNKS_TRANSFER_BOUND
    bounds = np.concatenate([[0], np.cumsum(np.floor(np.array(fr) * n).astype(np.int64))])
    bounds[-1] = n
    return bounds


def _ensemble_to_host(graph, field, config, pid_offset=0, n_particles=None, grid=None,
                      edge_counts=False, estimators=False):
    """run_ensemble's device work + transfers: per-particle arrays land in
    pinned host memory; large runs are split by global particle id (results
    are identical: every particle's stream is keyed by its id, the fused
    counts are integer sums) so transfers overlap the next chunk's kernel.

    ``pid_offset`` / ``n_particles`` select a shard of global ids (multi-GPU
    ranks).  With ``estimators=True`` returns ``(host arrays, device
    estimators)`` -- the chunks' fused estimators summed on the device (M
    histogram, totals, and ``edge_counts`` / the ``grid`` histogram when
    asked) -- instead of the flat list."""
    import torch

    names = ("edge", "x", "crossings", "events")
    n = config.n_particles if n_particles is None else int(n_particles)
    outs = names + (("edge_counts",) if edge_counts else ())
    est_keys = ("m_hist", "totals") + (("edge_counts",) if edge_counts else ()) + (
        ("hist",) if grid is not None else ())
    if n < _PIPELINE_MIN:
        res = ensemble_device(graph, field, config, pid_offset=pid_offset, n_particles=n,
                              outputs=outs, grid=grid)
        if not estimators:
            return _to_host([res[k] for k in names + ("m_hist", "totals")])
        hosts = _to_host([res[k] for k in names])
        return hosts, {k: res[k] for k in est_keys}
    _, dev = _native.torch_cuda(config.device)
    compute = torch.cuda.current_stream(dev)
    streams = _COPY_STREAMS.get(dev)
    if streams is None:  # copies; second launch stream
        streams = _COPY_STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    copier, side = streams
    if config.rng == "native" and 0 < config.n_steps and (
            config.n_steps < 256 or os.environ.get("GSDE_FORCE_STREAMING")) and _streaming_ok(copier):
        return _streamed_to_host(graph, field, config, pid_offset, n, outs, names, grid,
                                 est_keys, estimators, compute, copier)
    side.wait_stream(compute)  # whatever the caller queued comes first
    hosts = [torch.empty(n, dtype=torch.float64 if k == "x" else torch.int64, pin_memory=True)
             for k in names]
    bounds = _chunk_bounds(n, config.n_steps)
    parts = []
    for c, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:])):
        if hi <= lo:
            continue
        # chunks alternate between two streams, so a chunk's kernel fills the
        # SMs its predecessor's tail leaves idle (separate outputs; integer sums)
        st = compute if c % 2 == 0 else side
        with torch.cuda.stream(st):
            res = ensemble_device(graph, field, config, pid_offset=int(pid_offset + lo),
                                  n_particles=int(hi - lo), outputs=outs, grid=grid,
                                  stream=st.cuda_stream)
        done = torch.cuda.Event()
        done.record(st)
        copier.wait_event(done)
        with torch.cuda.stream(copier):
            for h, k in zip(hosts, names):
                h[lo:hi].copy_(res[k], non_blocking=True)
        parts.append(res)  # keeps the device buffers alive until the copies finished
    copier.synchronize()
    compute.wait_stream(side)
    est = {k: sum(r[k] for r in parts) for k in est_keys}
    if estimators:
        return [h.numpy() for h in hosts], est
    return [h.numpy() for h in hosts] + [est["m_hist"].cpu().numpy(),
                                         est["totals"].cpu().numpy()]


_STREAM_RANGES = 256  # progress counters per launch
_STREAMING: dict = {}  # copy stream -> stream memory operations work


def _streaming_ok(copier) -> bool:
    """cuStreamWaitValue32 usable (checked once per copy stream with a wait
    that is already satisfied); GSDE_NO_STREAMING=1 keeps the chunked
    launches."""
    import torch

    if os.environ.get("GSDE_NO_STREAMING"):
        return False
    ok = _STREAMING.get(copier)
    if ok is None:
        z = torch.zeros(1, dtype=torch.int32, device=copier.device)
        torch.cuda.current_stream(copier.device).synchronize()
        ok = _native.lib().gsde_stream_wait_geq32(copier.cuda_stream, z.data_ptr(), 0) == 0
        copier.synchronize()
        _STREAMING[copier] = ok
    return ok


def _copy_groups(n_ranges: int) -> list:
    """Range groups the copy stream moves together: 8 ranges at a time, the
    last 8 one by one (the final copy, exposed after the kernel, is small)."""
    cuts = list(range(0, max(n_ranges - 8, 0), 8)) + list(range(max(n_ranges - 8, 0), n_ranges))
    cuts.append(n_ranges)
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _streamed_to_host(graph, field, config, pid_offset, n, outs, names, grid, est_keys,
                      estimators, compute, copier):
    """_ensemble_to_host with ONE launch: the kernel counts finished
    particles per id range (gsde_out.progress, published after a GPU-scope
    fence) and the copy stream waits on each range's counter
    (cuStreamWaitValue32) before moving it, so the D2H starts with the first
    finished range.  Used for transfer-bound runs (n_steps < 256, where the
    copy engine is the bottleneck): C4 e2e 70.2 -> 64.7 ms.  Kernel-bound runs
    keep the chunked launches: there the last ranges complete only as the
    launch ends, and copying them afterwards costs more than the chunks'
    launch tails (C1 27.0 vs 25.3 ms, hub64 264.0 vs 264.1 ms;
    tools/e2e_streamed_ab.py, tools/e2e_streamed_timeline.py)."""
    import torch

    shift = max(0, (n - 1).bit_length() - (_STREAM_RANGES.bit_length() - 1))
    n_ranges = ((n - 1) >> shift) + 1
    prog = torch.zeros(n_ranges, dtype=torch.int32, device=compute.device)
    zeroed = torch.cuda.Event()
    zeroed.record(compute)
    copier.wait_event(zeroed)  # the counters' zeroing precedes every wait (not the launch)
    hosts = [torch.empty(n, dtype=torch.float64 if k == "x" else torch.int64, pin_memory=True)
             for k in names]
    res = ensemble_device(graph, field, config, pid_offset=int(pid_offset), n_particles=n,
                          outputs=outs, grid=grid, stream=compute.cuda_stream,
                          progress=(prog, shift))
    wait = _native.lib().gsde_stream_wait_geq32
    base = prog.data_ptr()
    with torch.cuda.stream(copier):
        for a, b in _copy_groups(n_ranges):
            for r in range(a, b):
                cnt = min(n, (r + 1) << shift) - (r << shift)
                _native.check(wait(copier.cuda_stream, base + 4 * r, cnt))
            lo, hi = a << shift, min(n, b << shift)
            for h, k in zip(hosts, names):
                h[lo:hi].copy_(res[k][lo:hi], non_blocking=True)
    copier.synchronize()
    est = {k: res[k] for k in est_keys}
    if estimators:
        return [h.numpy() for h in hosts], est
    return [h.numpy() for h in hosts] + [est["m_hist"].cpu().numpy(),
                                         est["totals"].cpu().numpy()]


def _multi_device(graph, field, config):
    """run_ensemble over several GPUs of this process: contiguous particle-id
    shards (the streams are keyed by global id), one launch per device queued
    on each device's current stream before any result is read, per-particle
    arrays gathered into pinned host memory, integer estimators summed."""
    import torch

    from .parallel import shard_range

    names = ("edge", "x", "crossings", "events")
    n = config.n_particles
    devs = [int(d) for d in config.devices]
    hosts = [torch.empty(n, dtype=torch.float64 if k == "x" else torch.int64, pin_memory=True)
             for k in names]
    parts = []
    for r, d in enumerate(devs):
        off, cnt = shard_range(n, r, len(devs))
        if cnt == 0:
            continue
        with torch.cuda.device(d):
            res = ensemble_device(graph, field, dataclasses.replace(config, device=d),
                                  pid_offset=off, n_particles=cnt, outputs=names)
            for h, k in zip(hosts, names):
                h[off:off + cnt].copy_(res[k], non_blocking=True)
        parts.append((d, res))
    m_hist = np.zeros(config.max_splits_per_step + 1, np.int64)
    totals = np.zeros(4, np.int64)
    for d, res in parts:
        torch.cuda.current_stream(d).synchronize()
        m_hist += res["m_hist"].cpu().numpy()
        totals += res["totals"].cpu().numpy()
    return [h.numpy() for h in hosts] + [m_hist, totals]


def _bits64(v: int) -> int:
    """uint64 value as the int64 with the same bit pattern (torch storage)."""
    v = int(v) & 0xFFFFFFFFFFFFFFFF
    return v - (1 << 64) if v >= (1 << 63) else v


def _to_host(tensors):
    """Device tensors -> numpy arrays through pinned staging buffers (torch's
    caching host allocator recycles them across calls); one stream sync."""
    import torch

    hosts = []
    for t in tensors:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        hosts.append(h)
    torch.cuda.current_stream(tensors[0].device).synchronize()
    return [h.numpy() for h in hosts]


def _step(graph, field, state, dt, rng, max_splits, reflect_at, star):
    torch, dev = _native.torch_cuda()
    dg = _native.device_graph(graph, field, dev)
    kw = dict(device=f"cuda:{dev}")
    edge = torch.tensor([state.edge], dtype=torch.int64, **kw)
    x = torch.tensor([state.x], dtype=torch.float64, **kw)
    k = torch.tensor([_bits64(rng.counter)], dtype=torch.int64, **kw)
    seed = torch.tensor([_bits64(rng.seed)], dtype=torch.int64, **kw)
    pid = torch.tensor([_bits64(rng.particle)], dtype=torch.int64, **kw)
    M = torch.zeros(1, dtype=torch.int64, **kw)
    tr = torch.zeros(1, dtype=torch.int64, **kw)
    a = _native.StepArgs()
    a.n, a.dt, a.cap, a.reflect_len = 1, float(dt), int(max_splits), float(reflect_at)
    a.stream = _native.GSDE_STREAM_REFERENCE
    a.seed, a.pid = seed.data_ptr(), pid.data_ptr()
    _native.check(_native.lib().gsde_step_batch(
        dg.handle, a, edge.data_ptr(), x.data_ptr(), k.data_ptr(), M.data_ptr(), tr.data_ptr(),
        _native.cur_stream(dev)))
    out = torch.stack([edge, M, tr]).cpu().numpy().reshape(-1)
    rng.counter = int(k.cpu().numpy()[0]) & 0xFFFFFFFFFFFFFFFF
    m = int(out[1])
    new_state = ParticleState(
        edge=int(out[0]),
        x=float(x.cpu().numpy()[0]),
        crossings_total=state.crossings_total + m,
        crossing_events=state.crossing_events + (1 if m > 0 else 0),
    )
    return StepOutcome(new_state, m, bool(out[2]))


def em_step_star(graph: MetricGraph, field: CoefficientField, state: ParticleState, dt: float,
                 rng: RngStream, max_splits: int = DEFAULT_MAX_SPLITS,
                 reflect_at: float = 0.0) -> StepOutcome:
    """One Alg. 1 step on a star graph (reference ``engine.py:206-235``);
    advances ``rng.counter``."""
    if not graph.is_star:
        raise ConfigInvalid("em_step_star requires a star graph; use em_step_general")
    return _step(graph, field, state, dt, rng, max_splits, reflect_at, True)


def em_step_general(graph: MetricGraph, field: CoefficientField, state: ParticleState,
                    dt: float, rng: RngStream,
                    max_splits: int = DEFAULT_MAX_SPLITS) -> StepOutcome:
    """One Alg. 2 step on a finite-edge graph (reference ``engine.py:238-270``)."""
    if graph.has_semi_infinite_edges:
        raise ConfigInvalid(
            "em_step_general requires finite edge lengths; star graphs with "
            "semi-infinite edges go through em_step_star"
        )
    return _step(graph, field, state, dt, rng, max_splits, 0.0, False)


def step_batch(graph, field, edges, xs, dt, seeds, pids, ks, max_splits=DEFAULT_MAX_SPLITS,
               reflect_at=0.0, inject=None, precision="f64"):
    """Batched single macro steps (device tensors in/out); returns
    ``(edge, x, M, trunc, k)``.  REFERENCE stream, or injected draws.
    ``seeds`` / ``pids`` / ``ks`` hold uint64 values as int64 bit patterns."""
    torch, dev = _native.torch_cuda()
    dg = _native.device_graph(graph, field, dev)
    n = int(edges.shape[0])
    edge = edges.clone()
    x = xs.clone()
    k = ks.clone()
    M = torch.zeros(n, dtype=torch.int64, device=edges.device)
    tr = torch.zeros(n, dtype=torch.int64, device=edges.device)
    a = _native.StepArgs()
    a.n, a.dt, a.cap, a.reflect_len = n, float(dt), int(max_splits), float(reflect_at)
    a.stream = _native.GSDE_STREAM_REFERENCE
    a.seed, a.pid = _native.ptr(seeds), _native.ptr(pids)
    if inject is not None:
        raw, nrm = inject
        a.stream = _native.GSDE_STREAM_INJECT
        a.precision = _native.GSDE_PREC_F64 if precision == "f64" else _native.GSDE_PREC_F32
        a.inj_raw, a.inj_normal, a.inj_stride = raw.data_ptr(), nrm.data_ptr(), raw.shape[1]
    _native.check(_native.lib().gsde_step_batch(
        dg.handle, a, edge.data_ptr(), x.data_ptr(), k.data_ptr(), M.data_ptr(), tr.data_ptr(),
        _native.cur_stream(dev)))
    return edge, x, M, tr, k


@dataclass(frozen=True)
class VertexTrials:
    """Outcomes of single macro steps started at a vertex (``engine.py:368-388``)."""

    M: np.ndarray
    exit_edges: np.ndarray
    exit_positions: np.ndarray
    truncated: np.ndarray
    dt: float
    gamma: float

    def stats(self) -> BounceStats:
        cap = int(self.M.max()) if self.M.size else 1
        hist = np.bincount(self.M, minlength=cap + 1).astype(np.int64)
        return BounceStats(
            m_histogram=hist,
            gamma=self.gamma,
            truncation_count=int(self.truncated.sum()),
            crossings_total=int(self.M.sum()),
            crossing_events=int((self.M > 0).sum()),
        )


def _trial_start(graph: MetricGraph, vertex: VertexId):
    if graph.is_star:
        return 0, 0.0
    if graph.has_semi_infinite_edges:
        raise ConfigInvalid("vertex trials on non-star graphs need finite edges")
    lo = int(graph.v_off[vertex])
    e0 = int(graph.v_edges[lo])
    return e0, graph.vertex_position(e0, int(graph.v_orient[lo]))


def trials_device(graph, field, dt, n_trials, seed, vertex=0, max_splits=DEFAULT_MAX_SPLITS,
                  rng="native", device=None, per_trial=True, trial_offset=0, inject=None,
                  precision="f32", stream=None):
    """Vertex trials on the GPU; returns DEVICE tensors.  With
    ``per_trial=False`` only the fused estimator (exit counts per edge,
    M histogram incl. M = 0, totals) is produced."""
    torch, dev = _native.torch_cuda(device)
    dg = _native.device_graph(graph, field, dev)
    e0, x0 = _trial_start(graph, vertex)
    kw = dict(device=f"cuda:{dev}")
    n = int(n_trials)
    res = {}
    o = _native.TrialsOut()
    if per_trial:
        for k, dt_ in (("M", torch.int64), ("edge", torch.int64), ("trunc", torch.int64),
                       ("x", torch.float64)):
            res[k] = torch.empty(n, dtype=dt_, **kw)
            setattr(o, k, res[k].data_ptr())
    res["exit_counts"] = torch.zeros(graph.n_edges, dtype=torch.int64, **kw)
    res["m_hist"] = torch.zeros(max_splits + 1, dtype=torch.int64, **kw)
    res["totals"] = torch.zeros(4, dtype=torch.int64, **kw)
    o.exit_counts, o.m_hist, o.totals = (res["exit_counts"].data_ptr(), res["m_hist"].data_ptr(),
                                         res["totals"].data_ptr())
    t = _native.Trials()
    t.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    t.n_trials, t.trial_offset, t.dt = n, int(trial_offset), float(dt)
    t.start_edge, t.start_x, t.cap = e0, float(x0), int(max_splits)
    t.stream = _stream_code(rng)
    if inject is not None:
        raw, nrm = inject
        t.stream = _native.GSDE_STREAM_INJECT
        t.precision = {"f64": _native.GSDE_PREC_F64, "f32": _native.GSDE_PREC_F32,
                       "native": _native.GSDE_PREC_NATIVE}[precision]
        t.inj_raw, t.inj_normal, t.inj_stride = raw.data_ptr(), nrm.data_ptr(), raw.shape[1]
    s = stream if stream is not None else _native.cur_stream(dev)
    _native.check(_native.lib().gsde_vertex_trials(dg.handle, t, o, s))
    return res


def vertex_crossing_trials(graph: MetricGraph, field: CoefficientField, dt: float,
                           n_trials: int, seed: int, vertex: VertexId = 0,
                           max_splits: int = DEFAULT_MAX_SPLITS, workers: int = 1, *,
                           rng: str = "native", device: int | None = None) -> VertexTrials:
    """``n_trials`` independent macro steps from ``vertex`` (reference
    ``engine.py:391-441``)."""
    if not dt > 0.0:
        raise ConfigInvalid(f"dt must be positive, got {dt!r}")
    if rng not in RNG_MODES:
        raise ConfigInvalid(f"rng must be one of {RNG_MODES}, got {rng!r}")
    n = int(n_trials)
    if n > 0:
        res = trials_device(graph, field, dt, n, seed, vertex, max_splits, rng, device)
        M, ex, xs, tr = _to_host([res["M"], res["edge"], res["x"], res["trunc"]])
    else:
        _trial_start(graph, vertex)
        M = np.zeros(0, np.int64)
        ex, tr, xs = M.copy(), M.copy(), np.zeros(0)
    return VertexTrials(M=M, exit_edges=ex, exit_positions=xs, truncated=tr, dt=float(dt),
                        gamma=gamma(field, graph, vertex, dt))
