// gsde_fvm.cu -- finite-volume Fokker-Planck baseline (reference fvm.py) on the GPU.
//
// Two kernels per explicit Euler step (exchange terms, then the update), one
// thread per work item, every update item writing a disjoint set of cells of
// the next density:
//   * a cell not adjacent to a degree >= 2 vertex: rho +- its two interior
//     face fluxes (per-cell SoA records: face drifts, D, dx -- one level of
//     independent, coalesced loads);
//   * a slot of a vertex whose adjacent cells no other vertex touches: the
//     slot cell's face terms, then the exchange terms of that cell in the
//     reference's loop order -- computed by the step's first kernel, one
//     thread per exchange row (fvm_terms_kernel), so no thread carries a
//     vertex's O(degree^2) chain of divisions;
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
// NC: the density read by a step is read-only for the whole kernel (the
// one-step phase kernels), so it may take the non-coherent path (__ldg).  The
// single-block kernel runs many steps in one launch and rewrites both buffers:
// it reads the density with plain loads.
template <bool NC>
struct FvmT {
  const gsde_fvm_desc &d;
  double dt;
  const double *rho;
  double *out;

  __device__ __forceinline__ double rd(int64_t c) const { return NC ? __ldg(rho + c) : rho[c]; }

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
    const uint8_t fl = __ldg(d.cell_flags + c);
    const double D = __ldg(d.cell_D + c), dx = __ldg(d.cell_dx + c);
    const double rc = rd(c);
    const double rl = (fl & kLeft) ? rd(c - 1) : 0.0;
    const double rr = (fl & kRight) ? rd(c + 1) : 0.0;
    const double scale = dt / dx;
    double v = rc;
    if (fl & kLeft) v += scale * face(__ldg(d.cell_mu_l + c), D, dx, rl, rc);
    if (fl & kRight) v -= scale * face(__ldg(d.cell_mu_r + c), D, dx, rc, rr);
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

// Phase A of the vertex exchange: row i of vertex v (fvm.py:305-328) -- drift
// exports i -> j and the diffusion pairs (i, j > i) -- written as signed terms
// to the positions the destinations read them from (fvm._term_layout).  Every
// term is the reference's own expression; a subtraction is stored negated.
template <class Fvm>
__device__ void exchange_row(const Fvm &f, int64_t t) {
  // every input is read-only during the step: __ldg lets the loads of later
  // iterations run ahead of this row's term stores
  const gsde_fvm_desc &d = f.d;
  const int64_t sl = __ldg(d.pslot + t);
  const int64_t v = __ldg(d.slot_vertex + sl);
  const int64_t lo = __ldg(d.v_off + v);
  const int n = (int)(__ldg(d.v_off + v + 1) - lo), i = (int)(sl - lo);
  const double *b = d.v_b + lo, *dx = d.v_dx + lo, *Dd = d.v_D + lo;
  const int64_t *cell = d.v_cells + lo;
  const int64_t *pos = d.rpos + __ldg(d.rstart + t);
  const double dt = f.dt, bi = __ldg(b + i), dxi = __ldg(dx + i), Di = __ldg(Dd + i);
  const double rho_i = f.rd(__ldg(cell + i));
  const double sp = __ldg(d.v_speed_in + sl), others = 1.0 - bi;
  if (sp > 0.0 && others > 0.0) {
    const double total = sp * rho_i;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double fl = total * __ldg(b + j) / others;
      const int64_t p0 = __ldg(pos), p1 = __ldg(pos + 1);
      d.terms[p0] = dt * fl / __ldg(dx + j);
      d.terms[p1] = -(dt * fl / dxi);
      pos += 2;
    }
  }
  const double conc_i = rho_i / bi;
#pragma unroll 2
  for (int j = i + 1; j < n; ++j) {
    const double bj = __ldg(b + j), dxj = __ldg(dx + j);
    const double rj = f.rd(__ldg(cell + j));
    const int64_t p0 = __ldg(pos), p1 = __ldg(pos + 1);
    const double dpair = 0.5 * (Di + __ldg(Dd + j));
    const double dxh = 2.0 * dxi * dxj / (dxi + dxj);
    const double g = dpair * (conc_i - rj / bj) / dxh;
    if (g >= 0.0) {
      const double fl = g * bj;
      d.terms[p0] = dt * fl / dxj;
      d.terms[p1] = -(dt * fl / dxi);
    } else {
      const double fl = -g * bi;
      d.terms[p1] = dt * fl / dxi;
      d.terms[p0] = -(dt * fl / dxj);
    }
    pos += 2;
  }
}

// Block max of (|rho|, -rho) over the cells a block wrote, folded into red[0..1]
// with one pair of 64-bit atomics per block (bit patterns of non-negative doubles
// order like the doubles).  Returns true in the block that finished last when
// `count` is set (red[2] counts those blocks).
__device__ __forceinline__ bool block_fold(double amax, double nmin, unsigned long long *red,
                                           bool count) {
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
    // canonical +0: the bit-pattern max orders non-negative doubles only
    amax = amax > 0.0 ? amax : 0.0;
    nmin = nmin > 0.0 ? nmin : 0.0;
    if (amax > 0.0) atomicMax(&red[0], (unsigned long long)__double_as_longlong(amax));
    if (nmin > 0.0) atomicMax(&red[1], (unsigned long long)__double_as_longlong(nmin));
    s_last = false;
    if (count) {
      __threadfence();
      s_last = atomicAdd(&red[2], 1ull) == gridDim.x - 1;
    }
  }
  __syncthreads();
  return s_last;
}

// Phase 1 of a step: exchange rows (terms for phase 2) and every cell no vertex
// owns (its final value).  One resident wave of blocks strides over
// [rows | cells]; both kinds are independent, latency-bound work.
// phase kernels at 64 registers (4 blocks / SM): measured 4/4 72 ms, 4/6 74 ms,
// 6/6 75 ms, 8/8 80 ms per 2000 C4 steps
__global__ void __launch_bounds__(kFvmThreads, 4)
    fvm_phase1_kernel(const __grid_constant__ gsde_fvm_desc d, double *rho, double *scratch,
                      double dt, const int64_t *neg_step, unsigned long long *red) {
  if (*(volatile const int64_t *)neg_step) return;  // an earlier step went negative
  const int64_t step = (int64_t)red[3];
  const FvmT<true> f{d, dt, (step & 1) ? scratch : rho, (step & 1) ? rho : scratch};
  const int64_t n_items = d.n_pslot + d.n_cells;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double amax = 0.0, nmin = 0.0;  // max |rho|, max(-rho) over the cells written here
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += stride) {
    if (it < d.n_pslot) {
      exchange_row(f, it);
    } else {
      const int64_t c = it - d.n_pslot;
      if (!(d.cell_flags[c] & kOwned)) {
        const double v = f.base(c);
        f.out[c] = v;
        track(v, amax, nmin);
      }
    }
  }
  block_fold(amax, nmin, red, false);
}

// Phase 2: vertex-adjacent cells (face terms + their exchange terms in the
// reference's order), the serial vertices, and the stop test in the last block.
__global__ void __launch_bounds__(kFvmThreads, 4)
    fvm_phase2_kernel(const __grid_constant__ gsde_fvm_desc d, double *rho, double *scratch,
                      double dt, double neg_floor, int64_t *neg_step,
                      unsigned long long *red) {
  if (*(volatile int64_t *)neg_step) return;
  const int64_t step = (int64_t)red[3];
  const FvmT<true> f{d, dt, (step & 1) ? scratch : rho, (step & 1) ? rho : scratch};
  const int64_t n_ser = d.n_vser > 0 ? 1 : 0;
  const int64_t n_items = n_ser + d.n_pslot;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double amax = 0.0, nmin = 0.0;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += stride) {
    if (it < n_ser) {
      for (int64_t k = 0; k < d.n_vser; ++k) f.init_cells(d.vser[k]);
      for (int64_t k = 0; k < d.n_vser; ++k) f.vertex_global(d.vser[k]);
      for (int64_t k = 0; k < d.n_vser; ++k)
        for (int64_t i = d.v_off[d.vser[k]]; i < d.v_off[d.vser[k] + 1]; ++i)
          track(f.out[d.v_cells[i]], amax, nmin);
    } else {
      const int64_t t = it - n_ser;
      const int64_t c = d.v_cells[d.pslot[t]];
      double val = f.base(c);
      for (int64_t m = d.tstart[t]; m < d.tstart[t + 1]; ++m) val += d.terms[m];
      f.out[c] = val;
      track(val, amax, nmin);
    }
  }
  if (block_fold(amax, nmin, red, true) && threadIdx.x == 0) {  // all maxima are in
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

// Small grids (the paper's star experiments: 10^2..10^4 cells) are bound by
// kernel launches, not work: one 1024-thread block runs every step, the two
// phases separated by __syncthreads(), the stop test on a block reduction.
// Same items, same per-cell operation sequence as the two-kernel path.
constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallItems = 16384;  // rows + cells up to which one block runs the run

__global__ void __launch_bounds__(kSmallThreads, 1)
    fvm_small_kernel(const __grid_constant__ gsde_fvm_desc d, double *rho, double *scratch,
                     int64_t n_steps, double dt, double neg_floor, int64_t *neg_step,
                     unsigned long long *red) {
  __shared__ double s_amax[kSmallThreads / 32], s_nmin[kSmallThreads / 32];
  const int64_t n_ser = d.n_vser > 0 ? 1 : 0;
  const int tid = threadIdx.x;
  int64_t done = 0;
  for (int64_t step = 0; step < n_steps; ++step) {
    const FvmT<false> f{d, dt, (step & 1) ? scratch : rho, (step & 1) ? rho : scratch};
    double amax = 0.0, nmin = 0.0;
    for (int64_t it = tid; it < d.n_pslot + d.n_cells; it += kSmallThreads) {
      if (it < d.n_pslot) {
        exchange_row(f, it);
      } else {
        const int64_t c = it - d.n_pslot;
        if (!(d.cell_flags[c] & kOwned)) {
          const double v = f.base(c);
          f.out[c] = v;
          track(v, amax, nmin);
        }
      }
    }
    __syncthreads();  // terms written
    for (int64_t it = tid; it < n_ser + d.n_pslot; it += kSmallThreads) {
      if (it < n_ser) {
        for (int64_t k = 0; k < d.n_vser; ++k) f.init_cells(d.vser[k]);
        for (int64_t k = 0; k < d.n_vser; ++k) f.vertex_global(d.vser[k]);
        for (int64_t k = 0; k < d.n_vser; ++k)
          for (int64_t i = d.v_off[d.vser[k]]; i < d.v_off[d.vser[k] + 1]; ++i)
            track(f.out[d.v_cells[i]], amax, nmin);
      } else {
        const int64_t t = it - n_ser;
        const int64_t c = d.v_cells[d.pslot[t]];
        double val = f.base(c);
        for (int64_t m = d.tstart[t]; m < d.tstart[t + 1]; ++m) val += d.terms[m];
        f.out[c] = val;
        track(val, amax, nmin);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      nmin = fmax(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
    }
    if ((tid & 31) == 0) {
      s_amax[tid >> 5] = amax;
      s_nmin[tid >> 5] = nmin;
    }
    __syncthreads();  // new densities and the warp maxima are in
    amax = s_amax[0];
    nmin = s_nmin[0];
    for (int w = 1; w < kSmallThreads / 32; ++w) {
      amax = fmax(amax, s_amax[w]);
      nmin = fmax(nmin, s_nmin[w]);
    }
    __syncthreads();  // everyone read the maxima before the next step rewrites them
    done = step + 1;
    if (-nmin < neg_floor * fmax(1.0, amax)) {  // fvm.py:329-337
      if (tid == 0) *neg_step = step + 1;
      break;
    }
  }
  if (done & 1)
    for (int64_t c = tid; c < d.n_cells; c += kSmallThreads) rho[c] = scratch[c];
  if (tid == 0) red[3] = (unsigned long long)done;
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
  if (d.n_pslot + d.n_cells <= kSmallItems) {
    fvm_small_kernel<<<1, kSmallThreads, 0, s>>>(d, rho, scratch, n_steps, dt, neg_floor,
                                                  neg_step, r);
    count_launch();
    return cudaGetLastError();
  }
  int device = 0;
  cudaGetDevice(&device);
  int per1 = 0, per2 = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, fvm_phase1_kernel, kFvmThreads, 0);
  if (err == cudaSuccess)
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, fvm_phase2_kernel, kFvmThreads, 0);
  if (err != cudaSuccess) return err;
  const int64_t sms = dev_info(device).sm_count;
  auto wave = [&](int64_t items, int per) {
    const int64_t need = (items + kFvmThreads - 1) / kFvmThreads;
    const int64_t w = sms * (per > 0 ? per : 1);
    return (unsigned)(need < 1 ? 1 : (need < w ? need : w));
  };
  const unsigned g1 = wave(d.n_pslot + d.n_cells, per1);
  const unsigned g2 = wave((d.n_vser > 0 ? 1 : 0) + d.n_pslot, per2);
  auto step = [&](cudaStream_t st) {
    fvm_phase1_kernel<<<g1, kFvmThreads, 0, st>>>(d, rho, scratch, dt, neg_step, r);
    fvm_phase2_kernel<<<g2, kFvmThreads, 0, st>>>(d, rho, scratch, dt, neg_floor, neg_step, r);
  };
  // the step kernels are identical (the step index lives in red[3]), so runs of
  // kGraphSteps steps are captured once into a CUDA graph and replayed; the
  // remainder (or a stream the caller is already capturing) launches directly
  constexpr int64_t kGraphSteps = 64;
  int64_t left = n_steps;
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  err = cudaStreamIsCapturing(s, &cap_status);
  if (err != cudaSuccess) return err;
  if (n_steps >= 2 * kGraphSteps && cap_status == cudaStreamCaptureStatusNone) {
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot capture), replay on the caller's
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
    err = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (err != cudaSuccess) return err;
    err = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (err == cudaSuccess) {
      for (int64_t k = 0; k < kGraphSteps; ++k) step(cs);
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
    step(s);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  count_launch((int)(n_steps < (1 << 29) ? 2 * n_steps : (1 << 30)));
  const int64_t blocks = (d.n_cells + kFvmThreads - 1) / kFvmThreads;
  const int64_t cap = (int64_t)dev_info(device).sm_count * 8;
  fvm_finish_kernel<<<(unsigned)(blocks < cap ? blocks : cap), kFvmThreads, 0, s>>>(
      rho, scratch, d.n_cells, r);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gsde
