"""Streamed run_ensemble timeline: device time of the launch with / without
progress counters, and when each copy group is waited for / copied relative
to the launch's end -- copies as one 2-D copy per group (rows of one block)
or four 1-D copies."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    dblk = torch.empty((4, n), dtype=torch.int64, device="cuda")
    hblk = torch.empty((4, n), dtype=torch.int64, pin_memory=True)
    rows = {k: (dblk[j].view(torch.float64) if k == "x" else dblk[j]) for j, k in enumerate(names)}
    for mode in ("2d", "1d", "2d", "1d"):
        prog = torch.zeros(nr, dtype=torch.int32, device="cuda")
        z = torch.cuda.Event(); z.record(s); copier.wait_event(z)
        t0 = torch.cuda.Event(enable_timing=True); t0.record(s)
        h0 = time.perf_counter()
        engine.ensemble_device(g, f, cfg, outputs=names, progress=(prog, shift), buffers=rows)
        k1 = torch.cuda.Event(enable_timing=True); k1.record(s)
        evs = []
        st = copier.cuda_stream
        for ga, gb in engine._copy_groups(nr):
            for rr in range(ga, gb):
                cnt = min(n, (rr + 1) << shift) - (rr << shift)
                _native.check(L.gsde_stream_wait_geq32(st, prog.data_ptr() + 4 * rr, cnt))
            w = torch.cuda.Event(enable_timing=True); w.record(copier)
            lo, hi = ga << shift, min(n, gb << shift)
            if mode == "2d":
                _native.check(L.gsde_memcpy2d_async(hblk.data_ptr() + 8 * lo, 8 * n, dblk.data_ptr() + 8 * lo,
                                                    8 * n, 8 * (hi - lo), 4, st))
            else:
                for j in range(4):
                    _native.check(L.gsde_memcpy2d_async(hblk.data_ptr() + 8 * (j * n + lo), 8 * (hi - lo),
                                                        dblk.data_ptr() + 8 * (j * n + lo), 8 * (hi - lo),
                                                        8 * (hi - lo), 1, st))
            e = torch.cuda.Event(enable_timing=True); e.record(copier)
            evs.append((ga, gb, w, e))
        h1 = time.perf_counter()
        copier.synchronize(); torch.cuda.synchronize()
        h2 = time.perf_counter()
        kend = t0.elapsed_time(k1)
        last = t0.elapsed_time(evs[-1][3])
        busy = sum(e.elapsed_time and w.elapsed_time(e) for _, _, w, e in evs)
        print(wname, mode, "kernel end %.3f, last copy %.3f, copy busy %.3f ms, host issue %.3f, wall %.3f" %
              (kend, last, busy, 1e3 * (h1 - h0), 1e3 * (h2 - h0)), flush=True)
        if mode == "1d" or mode == "2d":
            for ga, gb, w, e in evs[::6] + evs[-9:]:
                print("   ranges %3d-%3d waited %.3f copied %.3f" % (ga, gb, t0.elapsed_time(w), t0.elapsed_time(e)))
