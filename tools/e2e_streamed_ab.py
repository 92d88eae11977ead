"""run_ensemble e2e (bench's e2e_call: graph upload, kernel, D2H of the
reference-dtype arrays): one streamed launch vs chunked launches
(GSDE_NO_STREAMING=1), per workload; best of 4 after 2 warm-up calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

for name in (sys.argv[1:] or ["star3", "hub64", "vascular"]):
    wl = bench.make_workload(name, 0, 1)
    for mode in ("streamed", "chunked", "streamed"):
        if mode == "chunked":
            os.environ["GSDE_NO_STREAMING"] = "1"
        else:
            os.environ.pop("GSDE_NO_STREAMING", None)
        for _ in range(2):
            wl.e2e_call()
        ts = []
        for _ in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter(); wl.e2e_call(); torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        units = wl.cfg_single().n_particles * wl.cfg_single().n_steps
        print(f"{name} {mode}: {1e3 * min(ts):.2f} ms  {units / min(ts):.4g} psteps/s", flush=True)
