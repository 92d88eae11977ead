#!/usr/bin/env python
"""Benchmark: particle-steps/s of the timestep-splitting EM simulator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload star3|hub64|star5_trials|vascular] [--no-extras]

One bench "step" = one pass of the hot path over the workload's batch: one
``run_ensemble``-equivalent launch (all particles x all macro steps, fused
M-histogram / occupancy / snapshot-histogram estimators) plus, for N > 1, the
NCCL all-reduce that merges the estimators.  Default workload = C1 throughput
variant: 3-edge Brownian star, 1.6e7 particles per GPU x
1000 steps, dt = 1e-3 -- the configuration the north-star target
(>= 1e11 psteps/s per B200) is quoted on.  Particles shard by global id
(weak scaling); no data-path collective.

Rank 0 prints ONE JSON line.  ``value`` is device-timed (CUDA events, max
over ranks) with inputs resident; ``e2e`` goes through the public API
(``run_ensemble``: graph upload + kernel + D2H of the reference-dtype result
arrays) with host buffers.  ``--impl reference`` times the reference
algorithm on the host CPU (the C restatement in oracle/, all host threads).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "particle-steps/sec (1/2/4/8 B200) and fraction of FP32 roofline vs CPU ref"
UNIT = "psteps/s"


# ----------------------------------------------------------------------------
# workloads
class Workload:
    name = ""
    desc = ""
    unit = UNIT

    def __init__(self, rank=0, world=1):
        self.rank, self.world = rank, world


class Ensemble(Workload):
    def __init__(self, name, desc, build, n_per_gpu, n_steps, dt, initial, grid_fn, rank=0,
                 world=1, rng="native"):
        super().__init__(rank, world)
        import paper_2512_02175_b200 as gs

        self.name, self.desc = name, desc
        self.build = build
        self.g, self.f = build()
        self.n, self.n_steps, self.dt = n_per_gpu, n_steps, dt
        self.initial = initial(self.g)
        self.grid = grid_fn(self.g)
        self.rng = rng
        self.cfg = gs.SimulationConfig(dt=dt, n_steps=n_steps, n_particles=n_per_gpu * world,
                                       seed=20251202, initial=self.initial, rng=rng)
        self.units_per_step = n_per_gpu * n_steps  # per GPU

    def build_ref(self, R):
        """The same graph built through the reference package ``R``."""
        return self.build(api=R)

    def config(self):
        return {"workload": self.desc, "n_particles_per_gpu": self.n, "n_steps": self.n_steps,
                "dt": self.dt, "graph_edges": self.g.n_edges,
                "rng": ("native (FP32, Philox4x32-10)" if self.rng == "native" else
                        "reference (the reference's Philox4x32-10 + AS241 streams, FP64)")}

    def launch(self, stream):
        from paper_2512_02175_b200 import engine

        return engine.ensemble_device(self.g, self.f, self.cfg, pid_offset=self.rank * self.n,
                                      n_particles=self.n, outputs=("edge_counts",),
                                      grid=self.grid, stream=stream)

    def reduce_tensor(self, res):
        import torch

        return torch.cat([res["m_hist"], res["totals"], res["edge_counts"], res["hist"]])

    def crossings(self, res):
        return int(res["totals"][0])

    def e2e_call(self):
        """One public-API call with host buffers; returns D2H bytes.  N = 1:
        ``run_ensemble`` (the drop-in call).  N > 1: the sharded job,
        ``parallel.run_ensemble_distributed(particles=True)`` -- every rank
        simulates its global-id shard, copies its per-particle arrays to host
        memory, and the fused estimators are merged with one all-reduce."""
        import paper_2512_02175_b200 as gs
        from paper_2512_02175_b200 import parallel

        self.g._device.clear()  # inputs travel every step: graph + field upload
        if self.world == 1:
            r = gs.run_ensemble(self.g, self.f, self.cfg_single())
            d2h = sum(a.nbytes for a in (r.edges, r.positions, r.crossings, r.crossing_events))
            return d2h + r.stats.m_histogram.nbytes + 4 * 8
        r = parallel.run_ensemble_distributed(self.g, self.f, self.cfg, grid=self.grid,
                                              particles=True)
        d2h = sum(a.nbytes for a in r.particles.values())
        return d2h + r.m_histogram.nbytes + 4 * 8 + r.edge_counts.nbytes + r.histogram.nbytes

    def e2e_path(self):
        if self.world == 1:
            return ("paper_2512_02175_b200.run_ensemble (C-ABI gsde_ensemble): graph upload, "
                    "kernel, pinned D2H of the reference-dtype result arrays (5 particle-id "
                    "chunks: each chunk's D2H overlaps the next kernel)")
        return ("paper_2512_02175_b200.parallel.run_ensemble_distributed(particles=True): per "
                "rank graph upload, its global-id shard through the chunked run_ensemble "
                "pipeline (per-particle arrays to host), one all-reduce of the fused "
                "estimators, D2H of the merged estimators; time = max over ranks")

    def cfg_single(self):
        import dataclasses

        return dataclasses.replace(self.cfg, n_particles=self.n)

    def cpu_sample(self, scale):
        """(oracle callable, units) for a bounded CPU sample."""
        from oracle import oracle

        og = oracle.OracleGraph(self.g, self.f)
        from paper_2512_02175_b200.engine import _resolve_initial

        init = _resolve_initial(self.g, self.initial)
        n = max(4096, int(scale))

        def run(threads):
            oracle.ensemble(og, 20251202, n, self.n_steps, self.dt, init, 100, 0.0,
                            threads=threads)

        return run, n * self.n_steps, f"{n} particles x {self.n_steps} steps"


class Trials(Workload):
    """C3: the dt-convergence sweep of exit_probability_experiment (analysis.py:348-384):
    vertex trials at dt = 1e-2 .. 1e-5 (seed + i per dt, like the reference), fused exit
    counts + M histogram; one launch per dt."""

    unit = "trials/s"

    def __init__(self, rank=0, world=1, n_per_dt=1_000_000_000,
                 dts=(1e-2, 1e-3, 1e-4, 1e-5)):
        super().__init__(rank, world)
        from paper_2512_02175_b200 import workloads

        self.name = "star5_trials"
        self.desc = ("C3: paper §4.1 5-edge star, ConstantDrift(-10 i), dt sweep "
                     f"{', '.join(f'{d:g}' for d in dts)} x {n_per_dt:.0e} vertex trials per "
                     "GPU each (fused exit counts + M histogram)")
        self.g, self.f = workloads.star5("linear")
        self.n, self.dts = n_per_dt, tuple(dts)
        self.units_per_step = n_per_dt * len(dts)

    def build_ref(self, R):
        from paper_2512_02175_b200 import workloads

        return workloads.star5("linear", api=R)

    def config(self):
        return {"workload": self.desc, "n_trials_per_dt_per_gpu": self.n, "dts": list(self.dts)}

    def launch(self, stream):
        import torch
        from paper_2512_02175_b200 import engine

        parts = [engine.trials_device(self.g, self.f, dt, self.n, 11 + i, per_trial=False,
                                      trial_offset=self.rank * self.n, stream=stream)
                 for i, dt in enumerate(self.dts)]
        return {k: torch.cat([p[k] for p in parts]) for k in ("exit_counts", "m_hist", "totals")}

    def reduce_tensor(self, res):
        import torch

        return torch.cat([res["exit_counts"], res["m_hist"], res["totals"]])

    def e2e_call(self):
        """The public exit-probability API with host results: N = 1
        ``analysis.exit_probability_experiment`` over the dt sweep (fused exit
        counts, no per-trial arrays); N > 1 ``parallel.exit_counts_distributed``
        per dt (global trial-id shards, one all-reduce each)."""
        from paper_2512_02175_b200 import analysis, parallel

        self.g._device.clear()
        if self.world == 1:
            analysis.exit_probability_experiment(self.g, self.f, self.dts, self.n, 11)
        else:
            for i, dt in enumerate(self.dts):
                parallel.exit_counts_distributed(self.g, self.f, dt, self.n * self.world, 11 + i)
        return len(self.dts) * 8 * (self.g.n_edges + 101 + 4)

    def e2e_path(self):
        if self.world == 1:
            return ("paper_2512_02175_b200.analysis.exit_probability_experiment: graph upload, "
                    "one fused vertex-trials launch per dt, D2H of exit counts + M histogram")
        return ("paper_2512_02175_b200.parallel.exit_counts_distributed per dt: global "
                "trial-id shards, one all-reduce of the fused counts; time = max over ranks")

    def crossings(self, res):
        return int(res["totals"].view(-1, 4)[:, 0].sum())

    def cpu_run(self, n, threads):
        """The same dt sweep on the CPU port: n trials split evenly over the dts."""
        from oracle import oracle

        og = oracle.OracleGraph(self.g, self.f)
        per = max(1, n // len(self.dts))
        for i, dt in enumerate(self.dts):
            oracle.vertex_trials(og, 11 + i, per, dt, threads=threads)
        return per * len(self.dts)


class FvmWork(Workload):
    """Finite-volume baseline on the C4 network: 8 cells per edge,
    dt = 0.9 x the stability limit, 2000 explicit steps per bench step, one launch."""

    unit = "cell-steps/s"

    def __init__(self, rank=0, world=1, cells=8, n_steps=2000):
        super().__init__(rank, world)
        import paper_2512_02175_b200 as gs
        import torch
        from paper_2512_02175_b200 import fvm

        self.name = "fvm_vascular"
        self.g, self.f = _vascular_cached()
        self.grid = gs.EdgeGrid.uniform(self.g, cells)
        self.dt = 0.9 * fvm.stability_limit(self.g, self.f, self.grid)
        self.n_steps = n_steps
        self.fd = fvm.FvmDevice(self.g, self.f, self.grid, torch.cuda.current_device())
        self.rho0 = torch.tensor(fvm.FvmState.uniform(self.grid).rho, device="cuda")
        self.rho = self.rho0.clone()
        self.units_per_step = self.grid.n_cells * n_steps
        self.desc = (f"FVM baseline (fvm_run) on the C4 network: {self.g.n_edges} edges x "
                     f"{cells} cells, dt = 0.9 x stability limit, {n_steps} steps per launch")

    def config(self):
        return {"workload": self.desc, "n_cells": self.grid.n_cells, "n_steps": self.n_steps,
                "dt": self.dt}

    def launch(self, stream):
        self.rho.copy_(self.rho0)
        return {"neg": self.fd.run(self.rho, self.n_steps, self.dt, stream)}

    def reduce_tensor(self, res):
        return res["neg"]

    def crossings(self, res):
        return 0

    def e2e_call(self):
        """``fvm.fvm_run`` with a host initial state: the CFL check, the static
        packing (not reused across calls: inputs travel every call), the upload,
        every step on the GPU and the host copy of the final density."""
        from paper_2512_02175_b200 import fvm

        fvm._PACK_MEMO.clear()
        r = fvm.fvm_run(self.g, self.f, self.grid, self.dt, self.n_steps,
                        fvm.FvmState.uniform(self.grid))
        return r.state.rho.nbytes

    def e2e_h2d(self):
        return int(sum(getattr(self.fd.packed, k).nbytes for k in _FVM_DESC)) + \
            8 * self.grid.n_cells

    def e2e_path(self):
        return ("paper_2512_02175_b200.fvm.fvm_run (C-ABI gsde_fvm_run): CFL check, static "
                "packing, upload, all steps on the GPU, D2H of the final density")

    def cpu_baseline(self, steps=20):
        """The reference's own FVM stepper (``graphsde.fvm._fvm_step_loop``, numba,
        single-threaded by design, fvm.py:253-340) on the same C4 grid, fed the
        packed arrays of this package's vectorised ``_pack_static`` restatement
        (bit-identical inputs: tests/test_fvm.py; the reference's own Python
        packing takes ~110 s on this network); JIT excluded.  The C restatement
        in oracle/ stands in only if the reference cannot run."""
        rho = self.rho0.cpu().numpy().copy()
        packed = self.fd.packed.reference_tuple()
        R, why = reference_package()
        if R is not None:
            import importlib

            step_loop = importlib.import_module(R.__name__ + ".fvm")._fvm_step_loop
            step_loop(rho.copy(), 1, self.dt, *packed, -1e-10)  # JIT / cache load
            t0 = time.perf_counter()
            step_loop(rho, steps, self.dt, *packed, -1e-10)
            el = time.perf_counter() - t0
            return {"value": self.grid.n_cells * steps / el, "unit": self.unit, "cores": 1,
                    "kind": "reference",
                    "sample": f"{steps} steps of graphsde.fvm._fvm_step_loop on the C4 grid "
                              "(numba, single-threaded like the reference, baseline/_ref)"}
        from oracle import oracle

        t0 = time.perf_counter()
        oracle.fvm_steps(rho, 10, self.dt, packed)
        return {"value": self.grid.n_cells * 10 / (time.perf_counter() - t0), "unit": self.unit,
                "cores": 1, "kind": "port", "reference_unavailable": why,
                "sample": "10 steps, oracle/gsde_oracle.c orc_fvm_steps (single thread)"}


_FVM_DESC = ("cell_mu_l", "cell_mu_r", "cell_D", "cell_dx", "cell_flags", "v_off", "v_cells",
             "v_b", "v_dx", "v_speed_in", "v_D", "slot_vertex", "pslot", "vser", "tstart",
             "rstart", "rpos")


def make_workload(name, rank, world):
    import paper_2512_02175_b200 as gs
    from paper_2512_02175_b200 import workloads

    if name == "star3":
        return Ensemble(
            "star3", "C1-throughput: 3-edge star, Brownian (mu=0, sigma=1), AtVertex(0), "
            "dt=1e-3, 1000 steps, 1.6e7 particles/GPU; fused 3x16-cell snapshot histogram + "
            "final-edge counts",
            workloads.star3, 16_000_000, 1000, 1e-3, lambda g: gs.AtVertex(0),
            lambda g: gs.EdgeGrid.uniform(g, 16, lengths=[3.0] * 3), rank, world)
    if name == "hub64":
        return Ensemble(
            "hub64", "C2: 64-edge hub (lengths U[0.5,2]), LinearDrift(-k_i) quadratic potential, "
            "PerEdgeUniform(2.0), dt=1e-3, 1000 steps, 1e8 particles/GPU; fused 64x8 histogram",
            workloads.hub64, 100_000_000, 1000, 1e-3, lambda g: gs.PerEdgeUniform(2.0),
            lambda g: gs.EdgeGrid.uniform(g, 8), rank, world)
    if name == "vascular":
        return Ensemble(
            "vascular", "C4/C5: synthetic vascular network (~1.02e5 edges, kNN-MST + 2% loops), "
            "drift from_flux, PerEdgeUniform(max l), dt=1e-3, 100 steps, 1e8 particles/GPU; "
            "fused 8-cell/edge histogram",
            _vascular_cached, 100_000_000, 100, 1e-3,
            lambda g: gs.PerEdgeUniform(float(g.edge_length.max())),
            lambda g: gs.EdgeGrid.uniform(g, 8), rank, world)
    if name == "vascular_c5":  # C5: 1e8 particles x 100 steps in TOTAL, sharded over the ranks
        return Ensemble(
            "vascular_c5", "C5: the C4 network, 1e10 particle-steps per bench step in total "
            "(1e8 particles x 100 steps) sharded by particle id across the GPUs; per-step NCCL "
            "all-reduce of the fused estimators (8-cell/edge histogram, edge counts, M histogram)",
            _vascular_cached, 100_000_000 // world, 100, 1e-3,
            lambda g: gs.PerEdgeUniform(float(g.edge_length.max())),
            lambda g: gs.EdgeGrid.uniform(g, 8), rank, world)
    if name == "star3_ref":  # the bit-compatible FP64 reference stream on C1-throughput
        return Ensemble(
            "star3_ref", "C1-throughput in the reference's own streams (rng='reference': "
            "Philox4x32-10 + AS241 normals, FP64, inverse-CDF exits; edge ids / crossings "
            "bit-identical to graphsde): 3-edge Brownian star, 1.6e7 particles/GPU x 1000 steps",
            workloads.star3, 16_000_000, 1000, 1e-3, lambda g: gs.AtVertex(0),
            lambda g: gs.EdgeGrid.uniform(g, 16, lengths=[3.0] * 3), rank, world,
            rng="reference")
    if name == "star5_trials":
        return Trials(rank, world)
    if name == "fvm":
        return FvmWork(rank, world)
    raise SystemExit(f"unknown workload {name}")


_VASC = {}


def _vascular_cached(api=None):
    """The C4 network (this package's objects, or the reference's with ``api``)."""
    key = None if api is None else api.__name__
    if key not in _VASC:
        from paper_2512_02175_b200 import workloads

        _VASC[key] = workloads.vascular(api=api)
    return _VASC[key]


# ----------------------------------------------------------------------------
# measurement helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML in-process,
    initialised before the region and sampled every 10 ms -- C1's timed region is
    ~0.12 s; nvidia-smi subprocesses every 50 ms only if NVML is unavailable)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

            def sample():
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                return [str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)), str(mx)] + [
                    "Active" if r & b else "Not Active" for b in bits]
            sample()
            return sample
        except Exception:
            return None

    def _smi(self):
        out = subprocess.run(
            ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        return [p.strip() for p in out.stdout.strip().split(",")]

    def _run(self, sample, every):
        while not self._stop.is_set():
            try:
                parts = sample()
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(every)

    def __enter__(self):
        nv = self._nvml()
        sample, every = (nv, 0.01) if nv else (self._smi, 0.05)
        self._t = threading.Thread(target=self._run, args=(sample, every), daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def flush_l2(buf):
    buf.fill_(1)  # 256 MiB write > 126 MB L2


# FVM step, algorithmic bytes per cell: read rho[c] (8) + the per-cell record
# (left / right face drift, D, dx: 32; flags: 1), write new[c] (8); the
# neighbour densities are L1 hits.
FVM_BYTES_PER_CELL_STEP = 49


def lane_ops_per_pstep(crossings_per_pstep):
    """SURVEY.md §8(d) / BASELINE.md §3: W = 40 + 70 c lane-ops per pstep."""
    return 40.0 + 70.0 * crossings_per_pstep


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            entry = json.load(fh).get(workload)
        return None if entry is None else entry["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


# ----------------------------------------------------------------------------
# the reference's own CPU path (numba), installed unmodified under baseline/_ref
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_package():
    """``(graphsde, None)``: the UNMODIFIED reference package, installed with
    ``pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref <copy of /root/reference/pkg>`` (its numba / numpy / scipy
    dependencies are already in the image; pip's resolver only fails on the
    pins), running its own numba CPU kernels -- or ``(None, reason)``."""
    if not os.path.isdir(os.path.join(REF_DIR, "graphsde")):
        return None, "baseline/_ref/graphsde is not installed"
    # the reference's kernels are @njit(cache=True): keep the JIT cache off the repo copy
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "gsde_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(1, REF_DIR)
    try:
        import graphsde
        import graphsde.graphfile  # noqa: F401  (not re-exported by graphsde/__init__)
    except Exception as exc:  # numba missing, ...
        return None, f"import graphsde failed: {exc!r}"
    return graphsde, None


class RefRunner:
    """One bench workload on the reference's public API and stock code path
    (``graphsde.run_ensemble`` / ``graphsde.vertex_crossing_trials``, numba
    ``prange`` over all host threads): same graph (built through the
    reference's own ``build_graph`` / graph-file parser), seed, dt, steps and
    initial law; a bounded particle / trial sample."""

    def __init__(self, wl, R):
        import dataclasses

        self.R = R
        self.threads = int(R.engine.available_workers())
        self.unit = wl.unit
        self.trials = isinstance(wl, Trials)
        if self.trials:
            self.g, self.f = wl.build_ref(R)
            self.dts = wl.dts
            self.desc = "graphsde.vertex_crossing_trials"
        else:
            self.g, self.f = wl.build_ref(R)
            init = wl.initial
            self.initial = getattr(R, type(init).__name__)(*dataclasses.astuple(init))
            self.n_steps, self.dt = wl.n_steps, wl.dt
            self.desc = "graphsde.run_ensemble"

    def run(self, n):
        """n particles (ensembles) / n trials split over the dts; returns units done."""
        R = self.R
        if self.trials:
            per = max(1, int(n) // len(self.dts))
            for i, dt in enumerate(self.dts):
                R.vertex_crossing_trials(self.g, self.f, dt, per, 11 + i, workers=self.threads)
            return per * len(self.dts)
        n = max(1, int(n))
        cfg = R.SimulationConfig(dt=self.dt, n_steps=self.n_steps, n_particles=n,
                                 seed=20251202, initial=self.initial, workers=self.threads)
        R.run_ensemble(self.g, self.f, cfg)
        return n * self.n_steps

    def per_unit(self):
        return len(self.dts) if self.trials else self.n_steps

    def sized(self, seconds):
        """(n, rate): JIT warm-up (compile or cache load) excluded, then a
        ~1 s calibration, then n sized for ``seconds`` of CPU work."""
        t0 = time.perf_counter()
        self.run(4096 if self.trials else 256)
        self.jit_s = time.perf_counter() - t0
        n = 4096 * self.threads * (4 if self.trials else 1)
        while True:
            t0 = time.perf_counter()
            units = self.run(n)
            el = time.perf_counter() - t0
            if el > 0.5 or n > 1e9:
                break
            n *= 4
        rate = units / el
        per = self.per_unit()
        return max(n, int(rate * seconds / per)), rate

    def sample_desc(self, n):
        if self.trials:
            per = max(1, int(n) // len(self.dts))
            return (f"{per} trials per dt x {len(self.dts)} dts via {self.desc} (numba, "
                    f"{self.threads} threads, baseline/_ref)")
        return (f"{int(n)} particles x {self.n_steps} steps via {self.desc} (numba, "
                f"{self.threads} threads, baseline/_ref)")


def _port_baseline(wl, seconds, why):
    """Fallback when the reference package cannot run: the C restatement of its
    kernels in oracle/ (strict IEEE, OpenMP over the reference's chunks)."""
    threads = os.cpu_count() or 1
    if isinstance(wl, Trials):
        t0 = time.perf_counter()
        n_cal = wl.cpu_run(200_000, threads)
        rate = n_cal / max(time.perf_counter() - t0, 1e-6)
        t0 = time.perf_counter()
        n = wl.cpu_run(int(min(max(rate * seconds, n_cal), 2e9)), threads)
        return {"value": n / (time.perf_counter() - t0), "unit": wl.unit, "cores": threads,
                "kind": "port", "sample": f"{n} trials (oracle/gsde_oracle.c, {threads} threads)",
                "reference_unavailable": why}
    run, units, desc = wl.cpu_sample(20_000)
    t0 = time.perf_counter()
    run(threads)
    rate = units / max(time.perf_counter() - t0, 1e-6)
    run, units, desc = wl.cpu_sample(20_000 * max(1.0, rate * seconds / units))
    t0 = time.perf_counter()
    run(threads)
    return {"value": units / (time.perf_counter() - t0), "unit": UNIT, "cores": threads,
            "kind": "port", "sample": f"{desc} (oracle/gsde_oracle.c, {threads} threads)",
            "reference_unavailable": why}


def cpu_baseline(wl, seconds=12.0):
    """The reference's own CPU path (numba, all host threads) timed on a
    bounded sample of the same workload; the C port only if it cannot run."""
    R, why = reference_package()
    if R is None:
        return _port_baseline(wl, seconds, why)
    rr = RefRunner(wl, R)
    n, _ = rr.sized(seconds)
    t0 = time.perf_counter()
    units = rr.run(n)
    el = time.perf_counter() - t0
    return {"value": units / el, "unit": wl.unit, "cores": rr.threads, "kind": "reference",
            "sample": rr.sample_desc(n), "seconds": round(el, 2),
            "jit_s_excluded": round(rr.jit_s, 2)}


def run_reference_arm(args, rank, world):
    """``--impl reference``: the reference's own CPU implementation (numba, all
    host threads; rank 0 only), each step a ~2 s bounded sample of the same
    workload."""
    if rank != 0:
        return
    wl = make_workload(args.workload, 0, 1)
    R, why = reference_package()
    if R is None:  # the port stands in, and the line says so
        base = _port_baseline(wl, 2.0, why)
        threads = base["cores"]
        if isinstance(wl, Trials):
            n = max(len(wl.dts), int(base["value"] * 2.0))
            units = max(1, n // len(wl.dts)) * len(wl.dts)
            step = lambda: wl.cpu_run(n, threads)
            sample = f"{units} trials per step (oracle port)"
        else:
            run, units, sample = wl.cpu_sample(max(4096, base["value"] * 2.0 / wl.n_steps))
            step = lambda: run(threads)
        kind = "port"
    else:
        rr = RefRunner(wl, R)
        n, _ = rr.sized(2.0)
        threads = rr.threads
        units = max(1, n // len(rr.dts)) * len(rr.dts) if rr.trials else n * rr.n_steps
        step = lambda: rr.run(n)
        sample = rr.sample_desc(n)
        kind = "reference"
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = units * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(wl.config(), sample=sample, same_workload_bounded_sample=True,
                       rng="reference streams (Philox4x32-10 + AS241, FP64)"),
        "cpu_baseline": {"value": value, "unit": wl.unit, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": wl.unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if R is None:
        line["reference_unavailable"] = why
    print(json.dumps(line), flush=True)


STEP_MS = []  # per-step device times of the last time_workload call


def time_workload(wl, steps, warmup, dist, torch, dev, flush_buf, clocks_index=None):
    """Returns (elapsed_s max over ranks, kernel_s, res, launches)."""
    from paper_2512_02175_b200 import _native

    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        res = wl.launch(stream.cuda_stream)
        if dist is not None:
            dist.all_reduce(wl.reduce_tensor(res))
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = _native.launch_count()
    STEP_MS.clear()
    total = 0.0
    kern = 0.0
    sampler = ClockSampler(clocks_index) if clocks_index is not None else None
    if sampler:
        sampler.__enter__()
    try:
        # steps are enqueued back to back (no host sync inside the loop), so the
        # host-side launch work overlaps the previous step and never sits
        # between a start event and its kernel
        ev = []
        for _ in range(steps):
            flush_l2(flush_buf)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = wl.launch(stream.cuda_stream)
            e1.record(stream)
            if dist is not None:
                dist.all_reduce(wl.reduce_tensor(res))
            e2.record(stream)
            ev.append((e0, e1, e2, res))
        for e0, e1, e2, _ in ev:
            e2.synchronize()
            total += e0.elapsed_time(e2) / 1e3
            kern += e0.elapsed_time(e1) / 1e3
            STEP_MS.append(round(e0.elapsed_time(e2), 3))
    finally:
        if sampler:
            sampler.__exit__()
    torch.cuda.synchronize(dev)
    launches = _native.launch_count() - l0
    if dist is not None:
        dist.barrier()
        t = torch.tensor([total, kern], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, kern = float(t[0]), float(t[1])
    return total, kern, res, launches, (sampler.summary() if sampler else None)


def measure_e2e(wl, steps, warmup, dist, torch, dev, world):
    """``e2e``: the workload's public-API call with host buffers (graph
    upload, kernels, D2H of the result), every rank at once; each call's time
    is the max over ranks, the value the whole job's units over those times."""
    from paper_2512_02175_b200 import _native

    for _ in range(max(2, warmup)):  # first calls allocate pinned / device pools
        wl.e2e_call()
    torch.cuda.synchronize(dev)
    times, nbytes = [], 0
    for _ in range(steps):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        nbytes = wl.e2e_call()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t[0])
        times.append(el)
    h2d = wl.e2e_h2d() if hasattr(wl, "e2e_h2d") else \
        int(_native.device_graph(wl.g, wl.f, dev).device_bytes)
    return {"value": wl.units_per_step * world * len(times) / sum(times), "unit": wl.unit,
            "h2d_bytes_per_step": int(h2d) * world,
            "d2h_bytes_per_step": int(nbytes) * world,
            "ms_per_call": [round(t * 1e3, 2) for t in times], "path": wl.e2e_path()}


def extra_line(name, torch, dev, flush_buf, peaks, peak_ops, with_cpu):
    """One secondary workload at N = 1: device-timed value + roofline, e2e
    through its public API, and the reference CPU path beside it."""
    w2 = make_workload(name, 0, 1)
    t2, k2, r2, l2, _ = time_workload(w2, 3, 2, None, torch, dev, flush_buf)
    rate2 = w2.units_per_step * 3 / t2
    if name == "fvm":
        bpc = FVM_BYTES_PER_CELL_STEP
        return {
            "value": rate2, "unit": w2.unit, "config": w2.config(), "gpu_launches": int(l2),
            "bytes_per_cell_step": bpc, "achieved_gbs": rate2 * bpc / 1e9,
            "frac_of_hbm_peak": rate2 * bpc / 1e9 / float(peaks.get("hbm_gbs", 7700)),
            "note": "working set (~40 MB) is L2-resident across steps",
            "e2e": measure_e2e(w2, 3, 1, None, torch, dev, 1),
            "cpu_baseline": w2.cpu_baseline() if with_cpu else None}
    c2 = w2.crossings(r2) / w2.units_per_step
    out = {"value": rate2, "unit": w2.unit, "config": w2.config(), "step_ms": list(STEP_MS),
           "gpu_launches": int(l2), "crossings_per_unit": c2,
           "roofline_frac": w2.units_per_step * 3 / k2 * lane_ops_per_pstep(c2) / peak_ops}
    if getattr(w2, "rng", "native") != "native":
        out["roofline_frac"] = None
        out["roofline_note"] = ("FP64 reference stream (AS241 normals, strict IEEE): the FP32 "
                                "lane-op work model does not apply")
    if hasattr(w2, "e2e_call"):
        out["e2e"] = measure_e2e(w2, 3, 2, None, torch, dev, 1)
    if with_cpu:
        out["cpu_baseline"] = cpu_baseline(w2, seconds=8.0)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="star3",
                    choices=["star3", "hub64", "star5_trials", "vascular", "fvm", "star3_ref"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" not in os.environ:
        world = 1
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    # GSDE_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0, gloo collectives --
    # exercises the multi-rank sharding / reduction / max-over-ranks logic on a 1-GPU box
    shared = os.environ.get("GSDE_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = local
    dist = None
    if world > 1:
        import torch.distributed as tdist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator setup (nranks, NVLS / NVLink transport) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        # (NCCL logs to stdout by default: keep stdout for the one JSON line)
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = tdist
    import paper_2512_02175_b200 as gs  # noqa: F401
    from paper_2512_02175_b200 import _native

    _native.lib()
    flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    wl = make_workload(args.workload, rank, world)
    total, kern, res, launches, clocks = time_workload(
        wl, args.steps, args.warmup, dist, torch, dev, flush_buf,
        clocks_index=torch.cuda.current_device() if rank == 0 else None)
    units = wl.units_per_step * world * args.steps
    value = units / total
    crossings = wl.crossings(res)
    c_per = crossings / wl.units_per_step

    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_ops = sm_count * 128 * f_max * 1e6
    w_ops = lane_ops_per_pstep(c_per)
    kern_rate = wl.units_per_step * args.steps / kern  # per GPU, kernel only
    achieved = kern_rate * w_ops

    e2e = measure_e2e(wl, args.steps, args.warmup, dist, torch, dev, world) \
        if hasattr(wl, "e2e_call") else None
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "step_ms": list(STEP_MS),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if getattr(wl, "rng", "native") == "native" else "f64",
            "data": "synthetic (seeded graph generators, random streams; no external data)",
            "config": dict(wl.config(), parallelism=f"particle-sharded x{world}",
                           l2="flushed between steps (256 MiB write)"),
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": {
                "bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12,
                "unit": "Tlane-op/s", "frac": achieved / peak_ops,
                "traffic": load_traffic(wl.name),
                "work_model": f"W = 40 + 70 c lane-ops/pstep, c = {c_per:.4f} crossings/pstep "
                              f"(BASELINE.md §3); peak = {sm_count} SM x 128 lanes x "
                              f"{f_max:.0f} MHz ({'MEASURED_PEAKS.json' if peaks else 'nominal'})",
                "kernel_ms_per_step": kern / args.steps * 1e3,
            },
            "crossings_per_pstep": c_per,
        }
        if not args.no_cpu and world == 1:  # (the contract's CPU leg: rank 0 at N=1 only)
            line["cpu_baseline"] = cpu_baseline(wl)
        if not args.no_extras and world == 1:
            line["workloads"] = {
                name: extra_line(name, torch, dev, flush_buf, peaks, peak_ops, not args.no_cpu)
                for name in ("hub64", "star5_trials", "vascular", "star3_ref", "fvm")
                if name != args.workload}
    if not args.no_extras:
        # C5 strong scaling on every rank (a collective run): fixed 1e10 psteps per step
        w5 = make_workload("vascular_c5", rank, world)
        t5, _, r5, _, _ = time_workload(w5, 3, 2, dist, torch, dev, flush_buf)
        e5 = measure_e2e(w5, 3, 2, dist, torch, dev, world) if world > 1 else None
        if rank == 0:
            rate5 = w5.units_per_step * world * 3 / t5
            c5 = w5.crossings(r5) / w5.units_per_step
            line.setdefault("workloads", {})["vascular_c5"] = {
                "value": rate5, "unit": w5.unit, "scaling": "strong", "n_gpus": world,
                "config": dict(w5.config(), parallelism=f"particle-sharded x{world}"),
                "step_ms": list(STEP_MS), "crossings_per_unit": c5,
                "roofline_frac": rate5 / world * lane_ops_per_pstep(c5) / peak_ops,
                "e2e": e5 if e5 is not None else line.get("workloads", {}).get(
                    "vascular", {}).get("e2e")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
