"""Probe (GPU box): pinned D2H bandwidth and host-side widening throughput
(int32 -> int64, float32 -> float64) -- does a compact transfer + host widen
beat moving the reference dtypes over PCIe?"""
import os, time, torch
n = 100_000_000
print("cpu_count", os.cpu_count(), "sched", len(os.sched_getaffinity(0)), "torch threads", torch.get_num_threads())
d32 = torch.randint(0, 1 << 20, (n,), dtype=torch.int32, device="cuda")
d64 = d32.to(torch.int64)
h32 = torch.empty(n, dtype=torch.int32, pin_memory=True)
h64 = torch.empty(n, dtype=torch.int64, pin_memory=True)
for name, d, h in (("d2h int32 400MB", d32, h32), ("d2h int64 800MB", d64, h64)):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        h.copy_(d, non_blocking=True); torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(name, "%.1f GB/s" % (h.numel() * h.element_size() / dt / 1e9))
h64b = torch.empty(n, dtype=torch.int64, pin_memory=True)
f32 = torch.rand(n, dtype=torch.float32, pin_memory=True)
f64 = torch.empty(n, dtype=torch.float64, pin_memory=True)
for th in (1, 4, 8, 16, os.cpu_count()):
    torch.set_num_threads(th)
    for _ in range(2):
        t = time.perf_counter(); h64b.copy_(h32); dt1 = time.perf_counter() - t
        t = time.perf_counter(); f64.copy_(f32); dt2 = time.perf_counter() - t
    print("threads %d  i32->i64 %.1f ms (%.1f GB/s written)  f32->f64 %.1f ms" %
          (th, dt1 * 1e3, n * 8 / dt1 / 1e9, dt2 * 1e3))
# fresh (unfaulted) destination
t = time.perf_counter(); z = h32.to(torch.int64); dt = time.perf_counter() - t
print("i32->i64 into fresh pageable array %.1f ms" % (dt * 1e3))
