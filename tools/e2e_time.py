"""Per-call wall time of each bench workload's public-API e2e call (host buffers)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

for w in (sys.argv[1:] or ["star3", "hub64", "vascular"]):
    wl = bench.make_workload(w, 0, 1)
    for _ in range(2):
        wl.e2e_call()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); wl.e2e_call(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(w, "e2e %.2f ms -> %.4g %s" % (1e3 * min(ts), wl.units_per_step / min(ts), wl.unit), flush=True)
