"""star3 (C1) e2e: where the ~1 ms between the per-particle kernel and the
run_ensemble call goes -- graph upload, host-side launch prep, chunk schedule."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_02175_b200 import engine, _native

wl = bench.make_workload("star3", 0, 1)
cfg = wl.cfg_single()


def best(fn, k=5):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts[1:])


def upload():
    wl.g._device.clear()
    _native.device_graph(wl.g, wl.f, 0)


print("graph clear+upload %.3f ms" % best(upload))
outs = ("edge", "x", "crossings", "events")
t = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = engine.ensemble_device(wl.g, wl.f, cfg, outputs=outs)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    t.append((t1 - t0, t2 - t0)); del r
print("ensemble_device host-side %.3f ms, total %.3f ms" % (1e3 * min(a for a, _ in t[1:]), 1e3 * min(b for _, b in t[1:])))
for sched in ((1.0,), engine._CHUNKS, (0.7, 0.2, 0.07, 0.025, 0.005), (0.8, 0.15, 0.04, 0.01),
              (0.6, 0.25, 0.1, 0.04, 0.01), (0.45, 0.3, 0.15, 0.07, 0.025, 0.005)):
    engine._CHUNKS = sched
    print("chunks", sched, "e2e %.3f ms" % best(wl.e2e_call, 6), flush=True)
