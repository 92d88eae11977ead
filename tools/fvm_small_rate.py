"""FVM on the paper's small star grids: time per explicit step (single-block path)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import analysis, fvm, workloads

for kind in ("quadratic", "linear"):
    g, f = workloads.star5(kind)
    orc = analysis.SteadyStateOracle.from_field(g, f)
    for cells in (50, 200):
        grid = gs.EdgeGrid.uniform(g, cells, lengths=orc.truncation_lengths(1e-8))
        dt = 0.9 * fvm.stability_limit(g, f, grid)
        fd = fvm.FvmDevice(g, f, grid)
        rho = torch.tensor(fvm.FvmState.uniform(grid).rho, device="cuda")
        fd.run(rho, 1000, dt)
        torch.cuda.synchronize()
        n = 200_000
        t0 = time.perf_counter()
        fd.run(rho, n, dt)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        print(f"{kind} {cells} cells/edge ({grid.n_cells} cells): {el / n * 1e6:.2f} us/step, "
              f"{grid.n_cells * n / el:.3e} cell-steps/s")
