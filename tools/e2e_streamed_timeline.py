"""Streamed results timeline: device time of the per-particle launch with /
without progress counters, and when each progress range completes (a copy
stream waits on every range in turn and records an event) relative to the
launch's end."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2512_02175_b200 import engine, _native

names = ("edge", "x", "crossings", "events")
L = _native.lib()
for wname in (sys.argv[1:] or ["star3"]):
    wl = bench.make_workload(wname, 0, 1)
    cfg = wl.cfg_single()
    n = cfg.n_particles
    g, f = wl.g, wl.f
    s = torch.cuda.current_stream()
    shift = max(0, (n - 1).bit_length() - 8)
    nr = ((n - 1) >> shift) + 1
    for use in (False, True, False, True):
        prog = torch.zeros(nr, dtype=torch.int32, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        r = engine.ensemble_device(g, f, cfg, outputs=names, progress=(prog, shift) if use else None)
        b.record(s); torch.cuda.synchronize()
        print(wname, "kernel progress=%s %.3f ms" % (use, a.elapsed_time(b)), flush=True)
        del r
    copier = torch.cuda.Stream()
    prog = torch.zeros(nr, dtype=torch.int32, device="cuda")
    z = torch.cuda.Event(); z.record(s); copier.wait_event(z)
    t0 = torch.cuda.Event(enable_timing=True); t0.record(s)
    r = engine.ensemble_device(g, f, cfg, outputs=names, progress=(prog, shift))
    k1 = torch.cuda.Event(enable_timing=True); k1.record(s)
    evs = []
    for rr in range(nr):
        cnt = min(n, (rr + 1) << shift) - (rr << shift)
        _native.check(L.gsde_stream_wait_geq32(copier.cuda_stream, prog.data_ptr() + 4 * rr, cnt))
        e = torch.cuda.Event(enable_timing=True); e.record(copier); evs.append(e)
    torch.cuda.synchronize()
    kend = t0.elapsed_time(k1)
    done = np.array([t0.elapsed_time(e) for e in evs])
    print(wname, "kernel end %.3f ms; ranges done by kernel end - 1 / 0.5 / 0.2 / 0.1 ms: %d / %d / %d / %d of %d"
          % (kend, (done <= kend - 1).sum(), (done <= kend - 0.5).sum(), (done <= kend - 0.2).sum(),
             (done <= kend - 0.1).sum(), nr))
    print("   last 12 ranges complete at (ms before the end):", np.round(kend - done[-12:], 3).tolist())
    print("   range completion is monotone except", int((np.diff(done) < -0.05).sum()), "inversions > 50 us")
    if os.environ.get("TL_ALL"):
        print("   completion times (ms):", np.round(done, 3).tolist())
        # the same run's counters read back by the host while the launch runs
    if os.environ.get("TL_POLL"):
        torch.cuda.synchronize()
        prog.zero_()
        hp = torch.empty(nr, dtype=torch.int32, pin_memory=True)
        pol = torch.cuda.Stream()
        t0 = time.perf_counter()
        r = engine.ensemble_device(g, f, cfg, outputs=names, progress=(prog, shift))
        k1 = torch.cuda.Event(); k1.record(s)
        samples = []
        while not k1.query():
            with torch.cuda.stream(pol):
                hp.copy_(prog, non_blocking=True)
            pol.synchronize()
            want = np.minimum(n, (np.arange(nr) + 1) << shift) - (np.arange(nr) << shift)
            samples.append((time.perf_counter() - t0, int((hp.numpy() >= want).sum()),
                            int(hp.numpy().sum())))
        tend = time.perf_counter() - t0
        print("   host polling of the counters (t ms, ranges complete, particles published):")
        for t, c, p_ in samples[:: max(1, len(samples) // 40)]:
            print("     %.3f %d %d" % (1e3 * t, c, p_))
        print("   launch ended by %.3f ms (host)" % (1e3 * tend))
