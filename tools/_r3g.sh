mkdir -p gpurun_out/r3g
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3g/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3g/pytest_gpu.txt
nproc > gpurun_out/r3g/probe.txt
GSDE_TIMING=1 timeout 600 python - >> gpurun_out/r3g/probe.txt 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2512_02175_b200 import _native
wl = bench.make_workload("vascular", 0, 1)
for i in range(3):
    wl.g._device.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.device_graph(wl.g, wl.f, 0); torch.cuda.synchronize()
    print(f"device_graph {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
PY
timeout 600 python tools/e2e_time.py star3 hub64 vascular >> gpurun_out/r3g/probe.txt 2>&1
echo done
