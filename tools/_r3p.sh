mkdir -p gpurun_out/r3p
timeout 900 python - > gpurun_out/r3p/chunks.txt 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2512_02175_b200 import engine
scheds = {"A": (0.5, 0.28, 0.14, 0.06, 0.02), "F": (0.5, 0.28, 0.14, 0.06, 0.015, 0.005),
          "G": (0.45, 0.3, 0.15, 0.07, 0.025, 0.005), "H": (0.55, 0.25, 0.12, 0.055, 0.02, 0.005)}
for w in ("star3", "hub64"):
    wl = bench.make_workload(w, 0, 1)
    for rep in range(2):
        for k, sc in scheds.items():
            engine._CHUNKS = sc
            for _ in range(2): wl.e2e_call()
            ts = []
            for _ in range(4):
                torch.cuda.synchronize(); t0 = time.perf_counter(); wl.e2e_call(); torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            print(w, k, "%.2f ms" % (1e3 * min(ts)), flush=True)
PY
echo done
