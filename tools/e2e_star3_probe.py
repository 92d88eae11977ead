"""star3 (C1): lean kernel vs per-particle kernel vs the run_ensemble e2e call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_02175_b200 import engine

wl = bench.make_workload("star3", 0, 1)
cfg = wl.cfg_single()
s = torch.cuda.current_stream()
for outs, name in ((("edge_counts",), "lean"), (("edge", "x", "crossings", "events"), "per-particle")):
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); r = engine.ensemble_device(wl.g, wl.f, cfg, outputs=outs); b.record(s)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b)); del r
    print(name, "kernel %.2f ms" % min(ts[1:]), flush=True)
for _ in range(2): wl.e2e_call()
ts = []
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter(); wl.e2e_call(); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("e2e %.2f ms" % (1e3 * min(ts)))
