"""star3 (C1) e2e timeline: per-chunk kernel and copy start / end (CUDA events,
ms from the call's first event), the pipeline of engine._ensemble_to_host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_02175_b200 import engine

wl = bench.make_workload("star3", 0, 1)
cfg = wl.cfg_single()
g, f = wl.g, wl.f
names = ("edge", "x", "crossings", "events")
n = cfg.n_particles
dev = 0
compute = torch.cuda.current_stream()
copier, side = torch.cuda.Stream(), torch.cuda.Stream()


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


def run(sched):
    engine._CHUNKS = sched
    t0 = ev(compute)
    side.wait_stream(compute)
    hosts = [torch.empty(n, dtype=torch.float64 if k == "x" else torch.int64, pin_memory=True)
             for k in names]
    bounds = engine._chunk_bounds(n, cfg.n_steps)
    rec, parts = [], []
    for c, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:])):
        st = compute if c % 2 == 0 else side
        k0 = ev(st)
        with torch.cuda.stream(st):
            res = engine.ensemble_device(g, f, cfg, pid_offset=int(lo), n_particles=int(hi - lo),
                                         outputs=names, stream=st.cuda_stream)
        k1 = ev(st)
        copier.wait_event(k1)
        c0 = ev(copier)
        with torch.cuda.stream(copier):
            for h, k in zip(hosts, names):
                h[lo:hi].copy_(res[k], non_blocking=True)
        c1 = ev(copier)
        rec.append((k0, k1, c0, c1)); parts.append(res)
    copier.synchronize()
    compute.wait_stream(side)
    torch.cuda.synchronize()
    return [(t0.elapsed_time(a), t0.elapsed_time(b), t0.elapsed_time(c), t0.elapsed_time(d))
            for a, b, c, d in rec]


for sched in (engine._CHUNKS, (0.6, 0.25, 0.1, 0.04, 0.01)):
    for _ in range(3):
        torch.cuda.synchronize(); w0 = time.perf_counter(); r = run(sched); w = time.perf_counter() - w0
    print("schedule", sched, "wall %.3f ms" % (1e3 * w))
    for i, (a, b, c, d) in enumerate(r):
        print("  chunk %d kernel %.3f-%.3f (%.3f)  copy %.3f-%.3f (%.3f)" % (i, a, b, b - a, c, d, d - c))
