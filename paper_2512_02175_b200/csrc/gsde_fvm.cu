// gsde_fvm.cu -- finite-volume Fokker-Planck baseline (reference fvm.py) on the GPU.
//
// One kernel per explicit Euler step, one thread per work item, every item
// writing a disjoint set of cells of the next density:
//   * a cell not adjacent to a degree >= 2 vertex: rho +- its two interior
//     face fluxes (per-cell SoA records: face drifts, D, dx -- one level of
//     independent, coalesced loads);
//   * a slot of a vertex whose adjacent cells no other vertex touches: the
//     slot cell's face terms, then the contributions of the vertex exchange
//     to that cell in the reference's loop order (O(degree) per thread);
//   * one item for the remaining vertices (cells shared through single-cell
//     edges): the same, one vertex after another in ascending order.
// Every cell therefore sees the same sequence of IEEE operations as in
// _fvm_step_loop (fvm.py:254-340): the file is compiled without FMA
// contraction and results are bit-identical to the reference.  The state
// (8 B/cell: 6.5 MB for the 1e5-edge network at 8 cells per edge) stays in L2
// across steps.  The negativity check (fvm.py:330-337) is a per-step max
// reduction through 64-bit atomics on the bit patterns of non-negative
// doubles, evaluated by the step's last block; later step kernels see the
// stop flag and return at once, so the whole run is enqueued without a host
// round trip.
#include <cuda_runtime.h>

#include "gsde_internal.h"

namespace gsde {
namespace {

constexpr int kFvmThreads = 256;
enum : uint8_t { kLeft = 1, kRight = 2, kOwned = 4 };

// red[] layout: [0] max |rho|, [1] max(-rho) of the running step (double bit
// patterns), [2] blocks finished, [3] steps done
struct Fvm {
  const gsde_fvm_desc &d;
  double dt;
  const double *rho;
  double *out;

  // interior face flux with drift mu between cells l and r (fvm.py:287-292)
  __device__ __forceinline__ double face(double mu, double D, double dx, double rl,
                                         double rr) const {
    double F;
    if (mu > 0.0)
      F = mu * rl;
    else
      F = mu * rr;
    F -= D * (rr - rl) / dx;
    return F;
  }

  // rho[c] plus its interior-face terms in the reference's order:
  // new[c] += scale F(left face), then new[c] -= scale F(right face)
  __device__ __forceinline__ double base(int64_t c) const {
    const uint8_t fl = d.cell_flags[c];
    const double D = d.cell_D[c], dx = d.cell_dx[c];
    const double rc = rho[c];
    const double rl = (fl & kLeft) ? rho[c - 1] : 0.0;
    const double rr = (fl & kRight) ? rho[c + 1] : 0.0;
    const double scale = dt / dx;
    double v = rc;
    if (fl & kLeft) v += scale * face(d.cell_mu_l[c], D, dx, rl, rc);
    if (fl & kRight) v -= scale * face(d.cell_mu_r[c], D, dx, rc, rr);
    return v;
  }

  // vertex exchange (fvm.py:305-328) through accessors, so the same loop runs
  // on local arrays (small degree) or on global memory (hubs, shared cells)
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

  // exchange in place on out[] (cells already initialised)
  __device__ void vertex_global(int64_t v) const {
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

// New density of the cell of slot k of vertex v (cells of v touched by no
// other vertex): its face terms, then exactly the contributions the
// reference's exchange loop (fvm.py:305-328) adds to THIS cell, in loop order.
// Terms are recomputed per slot (the same IEEE operations as the serial loop),
// so one vertex's slots update in parallel: O(deg) per thread, not O(deg^2).
__device__ double slot_update(const Fvm &f, int64_t v, int k) {
  const gsde_fvm_desc &d = f.d;
  const int64_t lo = d.v_off[v];
  const int n = (int)(d.v_off[v + 1] - lo);
  const double *b = d.v_b + lo, *dx = d.v_dx + lo, *sp = d.v_speed_in + lo, *Dd = d.v_D + lo;
  const int64_t *cell = d.v_cells + lo;
  const double dt = f.dt;
  double acc = f.base(cell[k]);
  const double bk = b[k], dxk = dx[k], rk = f.rho[cell[k]];
  for (int i = 0; i < n; ++i) {
    const double bi = b[i];
    const double rho_i = i == k ? rk : f.rho[cell[i]];
    if (sp[i] > 0.0) {
      const double others = 1.0 - bi;
      if (others > 0.0) {
        const double total = sp[i] * rho_i;
        if (i == k) {  // cell i exports to every other slot, in j order
          for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double fl = total * b[j] / others;
            acc -= dt * fl / dxk;
          }
        } else {  // cell k receives its share once
          const double fl = total * bk / others;
          acc += dt * fl / dxk;
        }
      }
    }
    if (i > k) continue;  // pairs (i, j > i) touching k need i <= k
    const double conc_i = rho_i / bi;
    for (int j = (i == k ? i + 1 : k); j < (i == k ? n : k + 1); ++j) {
      const double dpair = 0.5 * (Dd[i] + Dd[j]);
      const double dxh = 2.0 * dx[i] * dx[j] / (dx[i] + dx[j]);
      const double rj = j == k ? rk : f.rho[cell[j]];
      const double g = dpair * (conc_i - rj / b[j]) / dxh;
      if (g >= 0.0) {
        const double fl = g * b[j];
        if (j == k)
          acc += dt * fl / dx[j];
        else
          acc -= dt * fl / dx[i];
      } else {
        const double fl = -g * b[i];
        if (i == k)
          acc += dt * fl / dx[i];
        else
          acc -= dt * fl / dx[j];
      }
    }
  }
  return acc;
}

// 6 blocks / SM (40 registers): the step is latency-bound, resident warps
// beat the few spills of the vertex-slot path (+8% over 64 registers)
__global__ void __launch_bounds__(kFvmThreads, 6)
    fvm_step_kernel(const __grid_constant__ gsde_fvm_desc d, double *rho, double *scratch,
                    double dt, double neg_floor, int64_t *neg_step,
                    unsigned long long *red) {
  if (*(volatile int64_t *)neg_step) return;  // an earlier step went negative
  const int64_t step = (int64_t)red[3];
  const Fvm f{d, dt, (step & 1) ? scratch : rho, (step & 1) ? rho : scratch};
  // item order: the serial vertices, then vertex slots (the long items start
  // first), then cells
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_ser = d.n_vser > 0 ? 1 : 0;
  double amax = 0.0, nmin = 0.0;  // max |rho|, max(-rho) over the cells written here
  if (it < n_ser) {
    for (int64_t k = 0; k < d.n_vser; ++k) f.init_cells(d.vser[k]);
    for (int64_t k = 0; k < d.n_vser; ++k) f.vertex_global(d.vser[k]);
    for (int64_t k = 0; k < d.n_vser; ++k)
      for (int64_t i = d.v_off[d.vser[k]]; i < d.v_off[d.vser[k] + 1]; ++i)
        track(f.out[d.v_cells[i]], amax, nmin);
  } else if (it < n_ser + d.n_pslot) {
    const int64_t sl = d.pslot[it - n_ser];
    const int64_t v = d.slot_vertex[sl];
    const double val = slot_update(f, v, (int)(sl - d.v_off[v]));
    f.out[d.v_cells[sl]] = val;
    track(val, amax, nmin);
  } else if (it < n_ser + d.n_pslot + d.n_cells) {
    const int64_t c = it - n_ser - d.n_pslot;
    if (!(d.cell_flags[c] & kOwned)) {
      const double v = f.base(c);
      f.out[c] = v;
      track(v, amax, nmin);
    }
  }
  __shared__ double s_amax[kFvmThreads / 32], s_nmin[kFvmThreads / 32];
  __shared__ bool s_last;
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
  if (threadIdx.x == 0) {
    for (int w = 1; w < kFvmThreads / 32; ++w) {
      amax = fmax(amax, s_amax[w]);
      nmin = fmax(nmin, s_nmin[w]);
    }
    // canonical +0: the bit-pattern max below orders non-negative doubles only
    amax = amax > 0.0 ? amax : 0.0;
    nmin = nmin > 0.0 ? nmin : 0.0;
    atomicMax(&red[0], (unsigned long long)__double_as_longlong(amax));
    atomicMax(&red[1], (unsigned long long)__double_as_longlong(nmin));
    __threadfence();
    s_last = atomicAdd(&red[2], 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {  // every block's maxima are in: the stop test
    __threadfence();
    const volatile unsigned long long *vr = red;
    const double mx = fmax(1.0, __longlong_as_double((long long)vr[0]));
    const double mn = -__longlong_as_double((long long)vr[1]);
    if (mn < neg_floor * mx) *neg_step = step + 1;
    red[0] = 0ull;
    red[1] = 0ull;
    red[2] = 0ull;
    red[3] = (unsigned long long)(step + 1);
  }
}

// after an odd number of completed steps the newest density is in scratch
__global__ void fvm_finish_kernel(double *rho, const double *scratch, int64_t n_cells,
                                  const unsigned long long *red) {
  if (!(red[3] & 1ull)) return;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x)
    rho[c] = scratch[c];
}

}  // namespace

cudaError_t launch_fvm(const gsde_fvm_desc &d, double *rho, double *scratch, int64_t n_steps,
                       double dt, double neg_floor, int64_t *neg_step, uint64_t *red,
                       cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(red, 0, 4 * sizeof(uint64_t), s);
  if (err == cudaSuccess) err = cudaMemsetAsync(neg_step, 0, sizeof(int64_t), s);
  if (err != cudaSuccess) return err;
  unsigned long long *r = reinterpret_cast<unsigned long long *>(red);
  const int64_t items = d.n_cells + d.n_pslot + (d.n_vser > 0 ? 1 : 0);
  const unsigned grid = (unsigned)((items + kFvmThreads - 1) / kFvmThreads);
  // the step kernels are identical (the step index lives in red[3]), so runs of
  // kGraphSteps launches are captured once into a CUDA graph and replayed;
  // the remainder (or a stream the caller is already capturing) launches directly
  constexpr int64_t kGraphSteps = 64;
  int64_t left = n_steps;
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  err = cudaStreamIsCapturing(s, &cap_status);
  if (err != cudaSuccess) return err;
  if (n_steps >= 2 * kGraphSteps && cap_status == cudaStreamCaptureStatusNone) {
    // capture on a private stream (the caller's may be the legacy default stream,
    // which cannot capture), replay on the caller's
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
    err = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (err != cudaSuccess) return err;
    err = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (err == cudaSuccess) {
      for (int64_t k = 0; k < kGraphSteps; ++k)
        fvm_step_kernel<<<grid, kFvmThreads, 0, cs>>>(d, rho, scratch, dt, neg_floor, neg_step,
                                                      r);
      err = cudaStreamEndCapture(cs, &graph);
    }
    cudaStreamDestroy(cs);
    if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
    for (; err == cudaSuccess && left >= kGraphSteps; left -= kGraphSteps)
      err = cudaGraphLaunch(exec, s);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (err != cudaSuccess) return err;
  }
  for (; left > 0; --left) {
    fvm_step_kernel<<<grid, kFvmThreads, 0, s>>>(d, rho, scratch, dt, neg_floor, neg_step, r);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  count_launch((int)(n_steps < (1 << 30) ? n_steps : (1 << 30)));
  int device = 0;
  cudaGetDevice(&device);
  const int64_t blocks = (d.n_cells + kFvmThreads - 1) / kFvmThreads;
  const int64_t cap = (int64_t)dev_info(device).sm_count * 8;
  fvm_finish_kernel<<<(unsigned)(blocks < cap ? blocks : cap), kFvmThreads, 0, s>>>(
      rho, scratch, d.n_cells, r);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gsde
