// gsde_fvm.cu -- finite-volume Fokker-Planck baseline (reference fvm.py) on the GPU.
//
// One persistent cooperative kernel runs all explicit Euler steps: per step
// every work item writes a disjoint set of cells of the next density, then
// one grid barrier.  Work items:
//   * a cell not adjacent to a degree >= 2 vertex: rho +- its two interior
//     face fluxes;
//   * a vertex whose adjacent cells no other vertex touches: its cells'
//     face terms, then the vertex exchange in the reference's loop order;
//   * one item for the remaining vertices (cells shared through single-cell
//     edges): the same, one vertex after another in ascending order.
// Every cell therefore sees the same sequence of IEEE additions as in
// _fvm_step_loop (fvm.py:254-340): the file is compiled without FMA
// contraction and results are bit-identical to the reference.  The density
// (8 B/cell, e.g. 6.5 MB for a 1e5-edge network at 8 cells per edge) stays in
// L2 across steps; the step is bound by L2 bandwidth and the barrier.
// The negativity check (fvm.py:330-337) is a per-step max-reduction through
// 64-bit atomics on the bit patterns of non-negative doubles.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "gsde_internal.h"

namespace cg = cooperative_groups;

namespace gsde {
namespace {

constexpr int kFvmThreads = 256;

struct Fvm {
  const gsde_fvm_desc &d;
  double dt;
  const double *rho;
  double *out;

  // interior face flux at face j of edge e (between cells j-1 and j), exactly
  // fvm.py:287-292
  __device__ __forceinline__ double face(int64_t e, int64_t lo, int64_t j) const {
    const double mu = d.face_mu[d.face_off[e] + (j - lo - 1)];
    double F;
    if (mu > 0.0)
      F = mu * rho[j - 1];
    else
      F = mu * rho[j];
    F -= d.D_edge[e] * (rho[j] - rho[j - 1]) / d.dx_edge[e];
    return F;
  }

  // rho[c] plus its interior-face terms in the reference's order:
  // new[c] += scale F(left face), then new[c] -= scale F(right face)
  __device__ __forceinline__ double base(int64_t c) const {
    const int64_t e = d.cell_edge[c];
    const int64_t lo = d.offs[e], hi = d.offs[e + 1];
    const double scale = dt / d.dx_edge[e];
    double v = rho[c];
    if (c > lo) v += scale * face(e, lo, c);
    if (c + 1 < hi) v -= scale * face(e, lo, c + 1);
    return v;
  }

  // vertex exchange at v (fvm.py:305-328) applied to out[] (cells owned here),
  // through accessors so the same loop runs on registers/local memory (small
  // degree) or directly on global memory (hubs, shared cells)
  template <class Nw, class Rho, class B, class Dx, class Sp, class Dv>
  __device__ __forceinline__ void exchange(int n, Nw &&nw, Rho &&r, B &&b, Dx &&dx, Sp &&sp,
                                           Dv &&Dd) const {
    for (int i = 0; i < n; ++i) {
      const double bi = b(i);
      const double rho_i = r(i);
      if (sp(i) > 0.0) {
        const double others = 1.0 - bi;
        if (others > 0.0) {
          const double total = sp(i) * rho_i;
          for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double f = total * b(j) / others;
            nw(j) += dt * f / dx(j);
            nw(i) -= dt * f / dx(i);
          }
        }
      }
      const double conc_i = rho_i / bi;
      for (int j = i + 1; j < n; ++j) {
        const double dpair = 0.5 * (Dd(i) + Dd(j));
        const double dxh = 2.0 * dx(i) * dx(j) / (dx(i) + dx(j));
        const double g = dpair * (conc_i - r(j) / b(j)) / dxh;
        if (g >= 0.0) {
          const double f = g * b(j);
          nw(j) += dt * f / dx(j);
          nw(i) -= dt * f / dx(i);
        } else {
          const double f = -g * b(i);
          nw(i) += dt * f / dx(i);
          nw(j) -= dt * f / dx(j);
        }
      }
    }
  }

  // whole update of a vertex whose cells no other vertex touches: face terms
  // then exchange, slot values staged in local arrays (L1) for degree <= 8
  __device__ void vertex_private(int64_t v, double &amax, double &nmin) const;

  // exchange on global memory, in place on out[] (cells already initialised)
  __device__ void vertex(int64_t v) const {
    const int64_t lo = d.v_off[v], hi = d.v_off[v + 1];
    if (hi - lo < 2) return;
    const int64_t *cell = d.v_cells + lo;
    exchange((int)(hi - lo), [&](int k) -> double & { return out[cell[k]]; },
             [&](int k) { return rho[cell[k]]; }, [&](int k) { return d.v_b[lo + k]; },
             [&](int k) { return d.v_dx[lo + k]; }, [&](int k) { return d.v_speed_in[lo + k]; },
             [&](int k) { return d.v_D[lo + k]; });
  }

  __device__ __forceinline__ void init_cells(int64_t v) const {
    for (int64_t i = d.v_off[v]; i < d.v_off[v + 1]; ++i) out[d.v_cells[i]] = base(d.v_cells[i]);
  }
};

__device__ __forceinline__ void track(double v, double &amax, double &nmin) {
  amax = fmax(amax, fabs(v));
  nmin = fmax(nmin, -v);
}

constexpr int kLocalDeg = 8;

__device__ void Fvm::vertex_private(int64_t v, double &amax, double &nmin) const {
  const int64_t lo = d.v_off[v], hi = d.v_off[v + 1];
  const int n = (int)(hi - lo);
  if (n > kLocalDeg) {
    init_cells(v);
    vertex(v);
    for (int64_t i = lo; i < hi; ++i) track(out[d.v_cells[i]], amax, nmin);
    return;
  }
  double nw[kLocalDeg], r[kLocalDeg], b[kLocalDeg], dx[kLocalDeg], sp[kLocalDeg], Dd[kLocalDeg];
  int64_t cell[kLocalDeg];
  for (int k = 0; k < n; ++k) {
    cell[k] = d.v_cells[lo + k];
    nw[k] = base(cell[k]);
    r[k] = rho[cell[k]];
    b[k] = d.v_b[lo + k];
    dx[k] = d.v_dx[lo + k];
    sp[k] = d.v_speed_in[lo + k];
    Dd[k] = d.v_D[lo + k];
  }
  exchange(n, [&](int k) -> double & { return nw[k]; }, [&](int k) { return r[k]; },
           [&](int k) { return b[k]; }, [&](int k) { return dx[k]; },
           [&](int k) { return sp[k]; }, [&](int k) { return Dd[k]; });
  for (int k = 0; k < n; ++k) {
    out[cell[k]] = nw[k];
    track(nw[k], amax, nmin);
  }
}

__global__ void __launch_bounds__(kFvmThreads)
    fvm_kernel(const __grid_constant__ gsde_fvm_desc d, double *rho, double *scratch, int64_t n_steps, double dt,
               double neg_floor, int64_t *neg_step, unsigned long long *red) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_amax[kFvmThreads / 32], s_nmin[kFvmThreads / 32];
  const int64_t n_items = d.n_cells + d.n_vpar + (d.n_vser > 0 ? 1 : 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool leader = tid == 0;
  if (leader) *neg_step = 0;
  int64_t done = 0;
  for (int64_t step = 0; step < n_steps; ++step) {
    Fvm f{d, dt, (step & 1) ? scratch : rho, (step & 1) ? rho : scratch};
    double amax = 0.0, nmin = 0.0;  // max |rho|, max(-rho) over the cells written here
    for (int64_t it = tid; it < n_items; it += stride) {
      if (it < d.n_cells) {
        if (d.owned[it]) continue;
        const double v = f.base(it);
        f.out[it] = v;
        track(v, amax, nmin);
      } else if (it < d.n_cells + d.n_vpar) {
        f.vertex_private(d.vpar[it - d.n_cells], amax, nmin);
      } else {
        for (int64_t k = 0; k < d.n_vser; ++k) f.init_cells(d.vser[k]);
        for (int64_t k = 0; k < d.n_vser; ++k) f.vertex(d.vser[k]);
        for (int64_t k = 0; k < d.n_vser; ++k)
          for (int64_t i = d.v_off[d.vser[k]]; i < d.v_off[d.vser[k] + 1]; ++i)
            track(f.out[d.v_cells[i]], amax, nmin);
      }
    }
    // block max, then one atomic per block into this step's slot (ring of 3:
    // the slot reset here was last read before the previous barrier)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      nmin = fmax(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
    }
    if ((threadIdx.x & 31) == 0) {
      s_amax[threadIdx.x >> 5] = amax;
      s_nmin[threadIdx.x >> 5] = nmin;
    }
    __syncthreads();
    unsigned long long *slot = red + 2 * (step % 3);
    if (threadIdx.x == 0) {
      for (int w = 1; w < kFvmThreads / 32; ++w) {
        amax = fmax(amax, s_amax[w]);
        nmin = fmax(nmin, s_nmin[w]);
      }
      // canonical +0: the bit-pattern max below orders non-negative doubles only
      amax = amax > 0.0 ? amax : 0.0;
      nmin = nmin > 0.0 ? nmin : 0.0;
      atomicMax(&slot[0], (unsigned long long)__double_as_longlong(amax));
      atomicMax(&slot[1], (unsigned long long)__double_as_longlong(nmin));
      if (leader) {
        unsigned long long *next = red + 2 * ((step + 1) % 3);
        next[0] = 0ull;
        next[1] = 0ull;
      }
    }
    grid.sync();
    done = step + 1;
    const double mx = fmax(1.0, __longlong_as_double((long long)*(volatile unsigned long long *)&slot[0]));
    const double mn = -__longlong_as_double((long long)*(volatile unsigned long long *)&slot[1]);
    if (mn < neg_floor * mx) {
      if (leader) *neg_step = step + 1;
      break;
    }
  }
  // after an odd number of steps the newest density is in scratch: move it
  if (done & 1)
    for (int64_t c = tid; c < d.n_cells; c += stride) rho[c] = scratch[c];
}

}  // namespace

cudaError_t launch_fvm(const gsde_fvm_desc &d, double *rho, double *scratch, int64_t n_steps,
                       double dt, double neg_floor, int64_t *neg_step, uint64_t *red,
                       cudaStream_t s) {
  int device = 0;
  cudaError_t err = cudaGetDevice(&device);
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fvm_kernel, kFvmThreads, 0);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  const int64_t items = d.n_cells + d.n_vpar + 1;
  int64_t grid = (int64_t)dev_info(device).sm_count * per_sm;
  const int64_t need = (items + kFvmThreads - 1) / kFvmThreads;
  if (need < grid) grid = need < 1 ? 1 : need;
  err = cudaMemsetAsync(red, 0, 6 * sizeof(uint64_t), s);
  if (err != cudaSuccess) return err;
  unsigned long long *r = reinterpret_cast<unsigned long long *>(red);
  void *args[] = {(void *)&d, &rho, &scratch, &n_steps, &dt, &neg_floor, &neg_step, &r};
  err = cudaLaunchCooperativeKernel((const void *)fvm_kernel, dim3((unsigned)grid),
                                    dim3(kFvmThreads), args, 0, s);
  count_launch();
  return err;
}

}  // namespace gsde
