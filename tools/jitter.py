"""Per-launch device times of one bench workload, back to back (no sampler, no flush)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

w = sys.argv[1] if len(sys.argv) > 1 else "star3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = bench.make_workload(w, 0, 1)
s = torch.cuda.current_stream()
for _ in range(2):
    wl.launch(s.cuda_stream)
torch.cuda.synchronize()
ev = []
for _ in range(n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); r = wl.launch(s.cuda_stream); b.record(s); ev.append((a, b, r))
torch.cuda.synchronize()
ms = [round(a.elapsed_time(b), 2) for a, b, _ in ev]
print(w, "min %.2f ms" % min(ms), "-> %.4g %s" % (wl.units_per_step / min(ms) * 1e3, wl.unit), ms)
