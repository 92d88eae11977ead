mkdir -p gpurun_out/r2o
GSDE_TIMING=1 timeout 600 python - > gpurun_out/r2o/probe.txt 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2512_02175_b200 import _native
wl = bench.make_workload("vascular", 0, 1)
for i in range(4):
    wl.g._device.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.device_graph(wl.g, wl.f, 0); torch.cuda.synchronize()
    print(f"device_graph {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); wl.e2e_call(); torch.cuda.synchronize()
    print(f"e2e_call {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
PY
echo done
