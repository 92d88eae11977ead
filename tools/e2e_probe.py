"""Where the e2e time of a large run_ensemble goes: PCIe D2H / H2D bandwidth into
pinned memory, and the phases of one run_ensemble call (vascular, 1e8 particles)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

dev = torch.device("cuda:0")
for nbytes in (256 << 20, 1 << 30):
    d = torch.empty(nbytes // 8, dtype=torch.int64, device=dev)
    h = torch.empty(nbytes // 8, dtype=torch.int64, pin_memory=True)
    for direction in ("d2h", "h2d"):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
        print(f"{direction} {nbytes >> 20} MiB: {nbytes / el / 1e9:.1f} GB/s")
    # two halves on two streams at once
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    half = nbytes // 16
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): h[:half].copy_(d[:half], non_blocking=True)
    with torch.cuda.stream(s2): h[half:].copy_(d[half:], non_blocking=True)
    torch.cuda.synchronize(); el = time.perf_counter() - t0
    print(f"d2h 2 streams {nbytes >> 20} MiB: {nbytes / el / 1e9:.1f} GB/s")
    del d, h

import bench
wl = bench.make_workload("vascular", 0, 1)
for _ in range(2):
    wl.e2e_call()
torch.cuda.synchronize()
t0 = time.perf_counter(); nb = wl.e2e_call(); el = time.perf_counter() - t0
print(f"vascular e2e call {el*1e3:.1f} ms, D2H {nb/1e9:.2f} GB -> {nb/el/1e9:.1f} GB/s effective")

# phases
from paper_2512_02175_b200 import _native, engine
g, f = wl.g, wl.f
for _ in range(2):
    g._device.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.device_graph(g, f, 0); torch.cuda.synchronize()
print(f"graph upload (gsde_graph_create) {1e3*(time.perf_counter()-t0):.1f} ms")
cfg = wl.cfg_single()
for outs in (("edge_counts",), ("edge", "x", "crossings", "events")):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = engine.ensemble_device(g, f, cfg, outputs=outs); torch.cuda.synchronize()
        el = time.perf_counter() - t0
    print(f"ensemble_device {outs}: {el*1e3:.1f} ms")
    del r
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hosts = engine._ensemble_to_host(g, f, cfg); torch.cuda.synchronize()
    el = time.perf_counter() - t0
print(f"_ensemble_to_host (chunked pipeline): {el*1e3:.1f} ms")
import paper_2512_02175_b200 as gs
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rr = gs.run_ensemble(g, f, cfg); torch.cuda.synchronize()
    el = time.perf_counter() - t0
print(f"run_ensemble (graph cached): {el*1e3:.1f} ms")
