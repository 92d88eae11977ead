// gsde_ref.cu -- reference-stream and injected-draw kernels.
//
// Bit-compatible mode of the simulator: the per-particle macro step follows
// the reference's control flow and draw order exactly (kernels.py:146-288)
// with draws from the reference stream (Philox4x32-10 keyed by
// (seed, particle, draw index), AS241 normals) or from caller-injected
// arrays.  Compiled with --fmad=false so every FP operation rounds like the
// strict-IEEE oracle; edge ids, crossing counts and truncations then match
// the reference exactly and positions to ~1e-11.
//
// One thread per particle, grid-stride; M histogram in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gsde_epilogue.cuh"

namespace gsde {
namespace {

// Draws from the reference stream; caches the current Philox block so the
// two draws of a block cost one evaluation (value-neutral, like the
// reference's lookahead buffer, kernels.py:55-64).
struct PhiloxDraws {
  uint64_t seed, pid, k, blk;
  Block b;
  __device__ PhiloxDraws(uint64_t s, uint64_t p, uint64_t k0)
      : seed(s), pid(p), k(k0), blk(~0ull), b{0, 0, 0, 0} {}
  __device__ __forceinline__ uint64_t raw() {
    const uint64_t bi = k >> 1;
    if (bi != blk) {
      b = ref_block(seed, pid, bi);
      blk = bi;
    }
    const uint64_t r = ref_half(b, k);
    ++k;
    return r;
  }
  __device__ __forceinline__ uint64_t u53() { return raw() >> 11; }
  __device__ __forceinline__ double normal() { return u64_to_normal(raw()); }
  __device__ __forceinline__ bool overrun() const { return false; }
};

// Draws injected by the caller: row i holds draw indices k0, k0+1, ...
struct InjectDraws {
  const uint64_t *raw_row;
  const double *nrm_row;
  int64_t stride;
  uint64_t k0, k;
  bool over;
  __device__ InjectDraws(const uint64_t *r, const double *n, int64_t st, uint64_t kk)
      : raw_row(r), nrm_row(n), stride(st), k0(kk), k(kk), over(false) {}
  __device__ __forceinline__ int64_t slot() {
    const int64_t j = (int64_t)(k - k0);
    ++k;
    if (j >= stride) {
      over = true;
      return -1;
    }
    return j;
  }
  __device__ __forceinline__ uint64_t u53() {
    const int64_t j = slot();
    return j < 0 ? 0 : (raw_row[j] >> 11);
  }
  __device__ __forceinline__ double normal() {
    const int64_t j = slot();
    return j < 0 ? 0.0 : nrm_row[j];
  }
  __device__ __forceinline__ bool overrun() const { return over; }
};

template <class R>
__device__ __forceinline__ R drift_at(const RefGraph<R> &g, int e, R x) {
  const int kd = g.dkind[e];
  if (kd == 0) return g.dcoef[e];
  if (kd == 1) return g.dcoef[e] * x;
  const int lo = g.tab_off[e], hi = g.tab_off[e + 1];
  if (x <= g.tab_x[lo]) return g.tab_mu[lo];
  if (x >= g.tab_x[hi - 1]) return g.tab_mu[hi - 1];
  int j = lo + 1;
  while (g.tab_x[j] < x) ++j;
  const R x0 = g.tab_x[j - 1];
  const R t = (x - x0) / (g.tab_x[j] - x0);
  return g.tab_mu[j - 1] + t * (g.tab_mu[j] - g.tab_mu[j - 1]);
}

// kernels.py:134-143 with u <= cumw[j]  <=>  (r >> 11) <= thresh[j].
template <class R>
__device__ __forceinline__ int pick_slot(const RefGraph<R> &g, int v, uint64_t u53) {
  const int lo = g.v_off[v], hi = g.v_off[v + 1];
  for (int j = lo; j < hi; ++j)
    if (u53 <= g.v_thresh[j]) return j;
  return hi - 1;
}

struct StepOut {
  int M;
  bool trunc;
};

// kernels.py:146-220 (Alg. 1): free proposal, split at the vertex, one-sided
// |W| excursions until accepted / time exhausted / cap.
template <class R, class D>
__device__ StepOut step_star(const RefGraph<R> &g, int &edge, R &x, R dt, D &d, int cap,
                             R reflect_len) {
  int M = 0;
  if (x > R(0)) {
    const R w = (R)d.normal();
    const R mu = drift_at(g, edge, x);
    const R a = mu * dt;
    const R b = g.sigma[edge] * sqrt(dt) * w;
    R xn = x + a + b;
    if (xn > R(0)) {
      if (reflect_len > R(0) && xn > reflect_len) {
        xn = R(2) * reflect_len - xn;
        if (xn < R(0)) xn = R(0);
      }
      x = xn;
      return {0, false};
    }
    R s = solve_first_passage_s<R>(a, b, x);
    if (s < R(0)) s = R(1);
    dt = (R(1) - s * s) * dt;
    if (dt < R(0)) dt = R(0);
  }
  for (;;) {
    ++M;
    edge = g.v_edges[pick_slot(g, 0, d.u53())];
    const R w = (R)d.normal();
    const R mu0 = drift_at(g, edge, R(0));
    const R sig0 = g.sigma[edge];
    R xn = mu0 * dt + sig0 * sqrt(dt) * fabs(w);
    if (xn >= R(0)) {
      if (reflect_len > R(0) && xn > reflect_len) {
        xn = R(2) * reflect_len - xn;
        if (xn < R(0)) xn = R(0);
      }
      x = xn;
      return {M, false};
    }
    const R alpha = (w * w * sig0 * sig0) / (mu0 * mu0 * dt);
    dt = (R(1) - alpha) * dt;
    if (dt <= R(0)) {
      x = R(0);
      return {M, false};
    }
    if (M >= cap) {
      x = R(0);
      return {M, true};
    }
  }
}

// kernels.py:223-288 (Alg. 2): per iteration [U if at a vertex], N; accept
// strictly inside (0, l); otherwise split at the hit end.
template <class R, class D>
__device__ StepOut step_general(const RefGraph<R> &g, int &edge, R &x, R dt, D &d, int cap) {
  int M = 0;
  for (;;) {
    R l = g.edge_len[edge];
    if (x <= R(0) || x >= l) {
      const int v = x <= R(0) ? g.edge_init[edge] : g.edge_term[edge];
      const int slot = pick_slot(g, v, d.u53());
      edge = g.v_edges[slot];
      l = g.edge_len[edge];
      x = g.v_orient[slot] == 0 ? R(0) : l;
    }
    const R w = (R)d.normal();
    const R mu = drift_at(g, edge, x);
    const R a = mu * dt;
    const R b = g.sigma[edge] * sqrt(dt) * w;
    const R xn = x + a + b;
    if (R(0) < xn && xn < l) {
      x = xn;
      return {M, false};
    }
    ++M;
    R s;
    if (xn <= R(0)) {
      s = solve_first_passage_s<R>(a, b, x);
      x = R(0);
    } else {
      s = solve_first_passage_s<R>(-a, -b, l - x);
      x = l;
    }
    if (s < R(0)) s = R(1);
    dt = (R(1) - s * s) * dt;
    if (dt <= R(0)) return {M, false};
    if (M >= cap) return {M, true};
  }
}

template <class D>
__device__ __forceinline__ D make_draws(uint64_t seed, uint64_t pid, uint64_t k,
                                        const uint64_t *inj_raw, const double *inj_nrm,
                                        int64_t stride, int64_t row);

template <>
__device__ __forceinline__ PhiloxDraws make_draws<PhiloxDraws>(uint64_t seed, uint64_t pid,
                                                               uint64_t k, const uint64_t *,
                                                               const double *, int64_t,
                                                               int64_t) {
  return PhiloxDraws(seed, pid, k);
}

template <>
__device__ __forceinline__ InjectDraws make_draws<InjectDraws>(uint64_t, uint64_t, uint64_t k,
                                                               const uint64_t *inj_raw,
                                                               const double *inj_nrm,
                                                               int64_t stride, int64_t row) {
  return InjectDraws(inj_raw + row * stride, inj_nrm + row * stride, stride, k);
}

// kernels.py:291-307 (draws k = 0, 1 for PerEdgeUniform).
template <class R, class D>
__device__ __forceinline__ void place(const RefGraph<R> &g, const gsde_run &a, D &d, int &edge,
                                      R &x) {
  if (a.init_kind == GSDE_INIT_POINT) {
    edge = (int)a.init_edge;
    x = (R)a.init_x;
    return;
  }
  const double u = u53_to_uniform(d.u53());
  const int m = g.n_edges;
  int e = (int)(u * (double)m);
  if (e >= m) e = m - 1;
  const double u2 = u53_to_uniform(d.u53());
  double span = a.init_xmax;
  const double le = (double)g.edge_len[e];
  if (le < span) span = le;
  edge = e;
  x = (R)(u2 * span);
}

template <class R, class D, bool STAR>
__global__ void __launch_bounds__(256) ref_ensemble_kernel(RefGraph<R> g, gsde_run a,
                                                           KOut o, int mh_smem) {
  extern __shared__ int s_mh[];
  const int nb = a.cap + 1;
  if (mh_smem)
    for (int j = threadIdx.x; j < nb; j += blockDim.x) s_mh[j] = 0;
  __syncthreads();
  int64_t t_cross = 0, t_events = 0, t_trunc = 0, t_over = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_particles;
       i += stride) {
    const uint64_t pid = (uint64_t)(a.pid_offset + i);
    D d = make_draws<D>(a.seed, pid, 0, a.inj_raw, a.inj_normal, a.inj_stride, i);
    int edge;
    R x;
    place<R, D>(g, a, d, edge, x);
    int64_t cross = 0, events = 0, truncs = 0;
    for (int64_t s = 0; s < a.n_steps; ++s) {
      const StepOut so = STAR ? step_star<R, D>(g, edge, x, (R)a.dt, d, a.cap, (R)a.reflect_len)
                              : step_general<R, D>(g, edge, x, (R)a.dt, d, a.cap);
      if (so.M > 0) {
        cross += so.M;
        events += 1;
        const int mm = so.M > a.cap ? a.cap : so.M;
        if (mh_smem)
          atomicAdd(&s_mh[mm], 1);
        else if (o.m_hist)
          add_i64(&o.m_hist[mm], 1);
        if (so.trunc) truncs += 1;
      }
      if (o.occ) {  // time-integrated occupation: sample after selected steps
        const int64_t k = s + 1 - o.occ_start;
        if (k > 0 && k % o.occ_every == 0)
          add_i64(&o.occ[hist_cell(o.hist_offsets, o.hist_counts, o.hist_dx, edge, (double)x)], 1);
      }
    }
    t_over += d.overrun() ? 1 : 0;
    t_cross += cross;
    t_events += events;
    t_trunc += truncs;
    ensemble_epilogue(o, (int64_t)i, edge, (double)x, cross, events, truncs);
  }
  if (o.totals) {
    warp_add_i64(&o.totals[0], t_cross);
    warp_add_i64(&o.totals[1], t_events);
    warp_add_i64(&o.totals[2], t_trunc);
    warp_add_i64(&o.totals[3], t_over);
  }
  __syncthreads();
  if (mh_smem && o.m_hist)
    for (int j = threadIdx.x; j < nb; j += blockDim.x)
      if (s_mh[j]) add_i64(&o.m_hist[j], s_mh[j]);
}

template <class R, class D, bool STAR>
__global__ void __launch_bounds__(256) ref_trials_kernel(RefGraph<R> g, gsde_trials a,
                                                         gsde_trials_out o, int mh_smem) {
  extern __shared__ int s_mh[];
  const int nb = a.cap + 1;
  if (mh_smem)
    for (int j = threadIdx.x; j < nb; j += blockDim.x) s_mh[j] = 0;
  __syncthreads();
  int64_t t_M = 0, t_ev = 0, t_tr = 0, t_over = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_trials; i += stride) {
    const uint64_t pid = (uint64_t)(a.trial_offset + i);
    D d = make_draws<D>(a.seed, pid, 0, a.inj_raw, a.inj_normal, a.inj_stride, i);
    int edge = STAR ? 0 : (int)a.start_edge;
    R x = STAR ? R(0) : (R)a.start_x;
    const StepOut so = STAR ? step_star<R, D>(g, edge, x, (R)a.dt, d, a.cap, R(0))
                            : step_general<R, D>(g, edge, x, (R)a.dt, d, a.cap);
    if (o.M) o.M[i] = so.M;
    if (o.edge) o.edge[i] = edge;
    if (o.x) o.x[i] = (double)x;
    if (o.trunc) o.trunc[i] = so.trunc ? 1 : 0;
    if (o.exit_counts) add_i64(&o.exit_counts[edge], 1);
    const int mm = so.M > a.cap ? a.cap : so.M;
    if (mh_smem)
      atomicAdd(&s_mh[mm], 1);
    else if (o.m_hist)
      add_i64(&o.m_hist[mm], 1);
    t_M += so.M;
    t_ev += so.M > 0;
    t_tr += so.trunc;
    t_over += d.overrun() ? 1 : 0;
  }
  if (o.totals) {
    warp_add_i64(&o.totals[0], t_M);
    warp_add_i64(&o.totals[1], t_ev);
    warp_add_i64(&o.totals[2], t_tr);
    warp_add_i64(&o.totals[3], t_over);
  }
  __syncthreads();
  if (mh_smem && o.m_hist)
    for (int j = threadIdx.x; j < nb; j += blockDim.x)
      if (s_mh[j]) add_i64(&o.m_hist[j], s_mh[j]);
}

template <class R, class D, bool STAR>
__global__ void __launch_bounds__(256) step_batch_kernel(RefGraph<R> g, gsde_step_args a,
                                                         int64_t *edge_io, double *x_io,
                                                         uint64_t *k_io, int64_t *M_out,
                                                         int64_t *trunc_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  D d = make_draws<D>(a.seed ? a.seed[i] : 0, a.pid ? a.pid[i] : 0, k_io[i], a.inj_raw,
                      a.inj_normal, a.inj_stride, i);
  int edge = (int)edge_io[i];
  R x = (R)x_io[i];
  const StepOut so = STAR ? step_star<R, D>(g, edge, x, (R)a.dt, d, a.cap, (R)a.reflect_len)
                          : step_general<R, D>(g, edge, x, (R)a.dt, d, a.cap);
  edge_io[i] = edge;
  x_io[i] = (double)x;
  k_io[i] = d.overrun() ? ~0ull : d.k;
  if (M_out) M_out[i] = so.M;
  if (trunc_out) trunc_out[i] = so.trunc ? 1 : 0;
}

int grid_for(int64_t n, int device) {
  const int sms = dev_info(device).sm_count;
  int64_t blocks = (n + 255) / 256;
  // several waves of blocks (grid-stride, static shares): later blocks refill
  // the slots of warps the schedulers favoured (8 -> 32 blocks per SM: C1
  // 4.91e10 -> 5.13e10, hub64 1.18e10 -> 1.29e10 psteps/s, tools/ref_rate.py)
  const int64_t cap = (int64_t)sms * 32;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

template <class R, class D>
cudaError_t ensemble_one(const RefGraph<R> &g, bool star, const gsde_run &a, const gsde_out &o,
                         int device, cudaStream_t s) {
  const size_t mh = (size_t)(a.cap + 1) * sizeof(int);
  const int grid = grid_for(a.n_particles, device);
  // shared int M bins while a block's count cannot reach 2^31 (grid-stride:
  // exact per-block particle counts); ensemble_impl chunks calls to keep this
  const double per_block = std::ceil((double)a.n_particles / ((double)grid * 256.0)) * 256.0 *
                           (double)(a.n_steps > 0 ? a.n_steps : 1);
  const int use_smem = (mh <= 32 * 1024 && per_block < 2147483647.0) ? 1 : 0;
  if (star)
    ref_ensemble_kernel<R, D, true><<<grid, 256, use_smem ? mh : 0, s>>>(g, a, kernel_out(o), use_smem);
  else
    ref_ensemble_kernel<R, D, false><<<grid, 256, use_smem ? mh : 0, s>>>(g, a, kernel_out(o), use_smem);
  count_launch();
  return cudaGetLastError();
}

// Calls whose blocks could count 2^31 steps into a shared bin run as
// consecutive launches over particle-id chunks (streams are keyed by global
// id, estimators accumulate: bit-identical to one launch).
template <class R, class D>
cudaError_t ensemble_impl(const RefGraph<R> &g, bool star, const gsde_run &a, const gsde_out &o,
                          int device, cudaStream_t s) {
  const double wave = (double)dev_info(device).sm_count * 32.0 * 256.0;  // grid_for's cap x 256
  const double k = std::floor(2147483647.0 / (256.0 * (double)(a.n_steps > 0 ? a.n_steps : 1)));
  int64_t chunk = k >= 1.0 ? (int64_t)std::min(k * wave, 9.0e18) : 0;
  static const char *forced = std::getenv("GSDE_CHUNK_PARTICLES");  // (testing)
  if (forced && std::atoll(forced) > 0) chunk = std::atoll(forced);
  if (chunk <= 0 || a.n_particles <= chunk) return ensemble_one<R, D>(g, star, a, o, device, s);
  for (int64_t off = 0; off < a.n_particles; off += chunk) {
    gsde_run ac = a;
    ac.n_particles = std::min(chunk, a.n_particles - off);
    ac.pid_offset = a.pid_offset + off;
    if (ac.inj_raw) ac.inj_raw += off * a.inj_stride;
    if (ac.inj_normal) ac.inj_normal += off * a.inj_stride;
    gsde_out oc = o;
    if (oc.edge) oc.edge += off;
    if (oc.x) oc.x += off;
    if (oc.crossings) oc.crossings += off;
    if (oc.events) oc.events += off;
    if (oc.truncs) oc.truncs += off;
    const cudaError_t err = ensemble_one<R, D>(g, star, ac, oc, device, s);
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

template <class R, class D>
cudaError_t trials_impl(const RefGraph<R> &g, bool star, const gsde_trials &a,
                        const gsde_trials_out &o, int device, cudaStream_t s) {
  const size_t mh = (size_t)(a.cap + 1) * sizeof(int);
  const int grid = grid_for(a.n_trials, device);
  const double per_block = std::ceil((double)a.n_trials / ((double)grid * 256.0)) * 256.0;
  const int use_smem = (mh <= 32 * 1024 && per_block < 2147483647.0) ? 1 : 0;
  if (star)
    ref_trials_kernel<R, D, true><<<grid, 256, use_smem ? mh : 0, s>>>(g, a, o, use_smem);
  else
    ref_trials_kernel<R, D, false><<<grid, 256, use_smem ? mh : 0, s>>>(g, a, o, use_smem);
  count_launch();
  return cudaGetLastError();
}

template <class R, class D>
cudaError_t step_impl(const RefGraph<R> &g, bool star, const gsde_step_args &a, int64_t *edge,
                      double *x, uint64_t *k, int64_t *M, int64_t *trunc, cudaStream_t s) {
  const int grid = (int)((a.n + 255) / 256);
  if (star)
    step_batch_kernel<R, D, true><<<grid, 256, 0, s>>>(g, a, edge, x, k, M, trunc);
  else
    step_batch_kernel<R, D, false><<<grid, 256, 0, s>>>(g, a, edge, x, k, M, trunc);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ref_ensemble(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                cudaStream_t s) {
  if (a.stream == GSDE_STREAM_REFERENCE)
    return ensemble_impl<double, PhiloxDraws>(g->ref64, g->is_star, a, o, g->device, s);
  if (a.precision == GSDE_PREC_F64)
    return ensemble_impl<double, InjectDraws>(g->ref64, g->is_star, a, o, g->device, s);
  return ensemble_impl<float, InjectDraws>(g->ref32, g->is_star, a, o, g->device, s);
}

cudaError_t launch_ref_trials(const gsde_graph *g, const gsde_trials &a,
                              const gsde_trials_out &o, cudaStream_t s) {
  if (a.stream == GSDE_STREAM_REFERENCE)
    return trials_impl<double, PhiloxDraws>(g->ref64, g->is_star, a, o, g->device, s);
  if (a.precision == GSDE_PREC_F64)
    return trials_impl<double, InjectDraws>(g->ref64, g->is_star, a, o, g->device, s);
  return trials_impl<float, InjectDraws>(g->ref32, g->is_star, a, o, g->device, s);
}

cudaError_t launch_step_batch(const gsde_graph *g, const gsde_step_args &a, int64_t *edge,
                              double *x, uint64_t *k, int64_t *M, int64_t *trunc,
                              cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  if (a.stream == GSDE_STREAM_REFERENCE)
    return step_impl<double, PhiloxDraws>(g->ref64, g->is_star, a, edge, x, k, M, trunc, s);
  if (a.precision == GSDE_PREC_F64)
    return step_impl<double, InjectDraws>(g->ref64, g->is_star, a, edge, x, k, M, trunc, s);
  return step_impl<float, InjectDraws>(g->ref32, g->is_star, a, edge, x, k, M, trunc, s);
}

}  // namespace gsde
