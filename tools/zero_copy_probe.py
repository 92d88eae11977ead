"""Probe: the per-particle kernel writing run_ensemble's arrays straight into
mapped pinned host memory (zero-copy over PCIe) vs device arrays + D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2512_02175_b200 import engine

names = ("edge", "x", "crossings", "events")
for wname in (sys.argv[1:] or ["star3", "vascular"]):
    wl = bench.make_workload(wname, 0, 1)
    cfg = wl.cfg_single()
    n = cfg.n_particles
    s = torch.cuda.current_stream()
    real_empty = torch.empty

    def host_empty(*a, **k):
        if str(k.get("device", "")).startswith("cuda") and a and a[0] == n:
            k = dict(k)
            k.pop("device")
            return real_empty(*a, pin_memory=True, **k)
        return real_empty(*a, **k)

    for mode in ("device", "zerocopy", "device", "zerocopy"):
        torch.empty = host_empty if mode == "zerocopy" else real_empty
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); w0 = time.perf_counter()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            r = engine.ensemble_device(wl.g, wl.f, cfg, outputs=names)
            b.record(s)
            if mode == "device":
                hosts = [real_empty(n, dtype=r[k].dtype, pin_memory=True) for k in names]
                for h, k in zip(hosts, names):
                    h.copy_(r[k], non_blocking=True)
            torch.cuda.synchronize()
            ts.append((a.elapsed_time(b), 1e3 * (time.perf_counter() - w0)))
            last = {k: (r[k] if mode == "zerocopy" else hosts[names.index(k)]).numpy().copy() for k in names}
        torch.empty = real_empty
        print(wname, mode, "kernel %.2f ms, kernel + copies (wall) %.2f ms" % (min(t[0] for t in ts), min(t[1] for t in ts)), flush=True)
        if mode == "device":
            ref = last
        else:
            for k in names:
                assert np.array_equal(ref[k], last[k]), k
