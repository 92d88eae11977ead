// gsde_native.cu -- the B200 production stepper (FP32, native stream).
//
// Design:
//  * one particle per lane, persistent grid (SMs x resident CTAs), particles
//    assigned by grid stride; all per-particle state lives in registers for
//    the whole run;
//  * flattened state machine: every loop trip performs exactly one proposal
//    per lane -- either a free Euler-Maruyama step or one vertex iteration --
//    so split/excursion loops never serialise a warp (kernels.py:198-220 and
//    :257-288 become extra trips of the same loop body);
//  * RNG: one Philox4x32-10 block per TWO trips, counter (trip pair, domain,
//    particle id) under the seed: words 0,1 -> Box-Muller -> the trips'
//    Gaussians, words 2,3 -> the trips' 32-bit exit-slot uniforms.  Every
//    trip consumes the same amount, so lanes stay phase-aligned and the block
//    is generated warp-convergently;
//  * exit slot: per-vertex alias table, one column record (16 B) per pick;
//  * star graphs / small graphs: edge records + alias columns staged in
//    shared memory; large networks read them through L2 (__ldg);
//  * estimators fused: M histogram in lane-private shared counters
//    (M < kPriv) + shared atomics, final-edge occupancy and snapshot histogram
//    in the epilogue, totals warp-reduced.
#include <cuda_runtime.h>

#include "gsde_epilogue.cuh"

namespace gsde {
namespace {

constexpr int kThreads = 256;
constexpr int kPriv = 8;  // lane-private M-histogram bins
constexpr uint32_t kDomainEnsemble = 0u;
constexpr uint32_t kDomainTrials = 1u;
constexpr uint32_t kDomainPlace = 0xFFFFFFFFu;

struct NatParams {
  uint64_t seed;
  int64_t n;          // particles / trials in this call
  int64_t id_offset;  // global id of item 0
  int32_t n_steps;
  int32_t cap;
  float dt, sqdt;
  float reflect;      // star mirror wall (0 = off)
  int32_t init_kind;
  int32_t init_edge;
  float init_x;
  double init_xmax;
  int32_t start_edge; // trials (general)
  float start_x;
  int32_t smem_graph;
};

// Box-Muller on two 32-bit words: u1 in (0, 1] with 2^-33 resolution near 0
// (|z| <= 6.8), angle uniform on [-pi, pi).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float &z0, float &z1) {
  const float u1 = fmaf((float)a, 0x1p-32f, 0x1p-33f);
  const float r = sqrtf(fmaxf(-2.0f * __logf(u1), 0.0f));
  float s, c;
  __sincosf((float)(int32_t)b * 0x1p-31f * 3.14159265358979f, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

__device__ __forceinline__ float drift_tab(const NativeGraph &G, int e, float x) {
  const int lo = G.tab_off[e], hi = G.tab_off[e + 1];
  if (x <= G.tab_x[lo]) return G.tab_mu[lo];
  if (x >= G.tab_x[hi - 1]) return G.tab_mu[hi - 1];
  int j = lo + 1;
  while (G.tab_x[j] < x) ++j;
  const float x0 = G.tab_x[j - 1];
  const float t = (x - x0) / (G.tab_x[j] - x0);
  return G.tab_mu[j - 1] + t * (G.tab_mu[j] - G.tab_mu[j - 1]);
}

__device__ __forceinline__ float drift(const NativeGraph &G, const float4 &ep, int e, float x) {
  if (G.has_tab && isnan(ep.z)) return drift_tab(G, e, x);
  return fmaf(ep.z, x, ep.y);
}

// Alias pick with a 32-bit uniform: column = floor(u * deg), then the
// column's threshold on the low word.  Returns edge | orient << 31.
__device__ __forceinline__ int alias_pick(const int4 *cols, int off, int deg, uint32_t u) {
  const uint64_t t = (uint64_t)u * (uint32_t)deg;
  const int4 c = cols[off + (int)(t >> 32)];
  return (uint32_t)t < (uint32_t)c.x ? c.y : c.z;
}

// Shared-memory layout: [priv: kPriv * kThreads ints][mh: cap+1 ints][pad]
// [edges E float4][edgev E int4][cols S int4]  (graph part optional).
struct Smem {
  int *priv;
  int *mh;
  const float4 *edge;
  const int4 *edgev;
  const int4 *col;
};

__device__ __forceinline__ size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

__device__ Smem smem_setup(const NativeGraph &G, int nb, int stage_graph, bool star) {
  extern __shared__ __align__(16) unsigned char smem[];
  Smem S;
  S.priv = reinterpret_cast<int *>(smem);
  S.mh = S.priv + kPriv * kThreads;
  size_t off = align16((size_t)(kPriv * kThreads + nb) * sizeof(int));
  for (int j = threadIdx.x; j < kPriv * kThreads + nb; j += blockDim.x) S.priv[j] = 0;
  S.edge = G.edge;
  S.edgev = G.edgev;
  S.col = G.col;
  if (stage_graph) {
    float4 *se = reinterpret_cast<float4 *>(smem + off);
    off += (size_t)G.n_edges * sizeof(float4);
    int4 *sv = reinterpret_cast<int4 *>(smem + off);
    if (!star) off += (size_t)G.n_edges * sizeof(int4);
    int4 *sc = reinterpret_cast<int4 *>(smem + off);
    for (int j = threadIdx.x; j < G.n_edges; j += blockDim.x) {
      se[j] = G.edge[j];
      if (!star) sv[j] = G.edgev[j];
    }
    for (int j = threadIdx.x; j < G.n_slots; j += blockDim.x) sc[j] = G.col[j];
    S.edge = se;
    S.edgev = sv;
    S.col = sc;
  }
  __syncthreads();
  return S;
}

__device__ __forceinline__ void mh_add(const Smem &S, int bin) {
  if (bin < kPriv)
    S.priv[bin * kThreads + threadIdx.x] += 1;
  else
    atomicAdd(&S.mh[bin], 1);
}

__device__ void mh_flush(const Smem &S, int nb, int64_t *dst) {
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    int64_t v = S.mh[b];
    if (b < kPriv)
      for (int t = 0; t < kThreads; ++t) v += S.priv[b * kThreads + t];
    if (v && dst) add_i64(&dst[b], v);
  }
}

// Per-lane simulation state.
struct Lane {
  int e;        // current edge
  float x;      // position on e
  float dtr;    // time left in the current macro step
  float sq;     // sqrt(dtr)
  int M;        // vertex resolutions in the current macro step
  bool trunc;
  float4 ep;    // cached edge record of e
  int4 ev;      // cached endpoint alias info of e (general graphs)
};

// One trip of the star-graph state machine (kernels.py:146-220 semantics).
// Returns true when the macro step completed.
__device__ __forceinline__ bool star_trip(Lane &L, const NativeGraph &G, const Smem &S,
                                          const NatParams &p, float z, uint32_t u) {
  const bool at_v = !(L.x > 0.0f);
  float4 ep = L.ep;
  int e = L.e;
  float xb = L.x, w = z;
  if (at_v) {  // sample the exit edge, one-sided excursion
    e = alias_pick(S.col, 0, G.n_edges, u) & 0x7fffffff;
    ep = S.edge[e];
    xb = 0.0f;
    w = fabsf(z);
    L.M += 1;
  }
  const float mu = drift(G, ep, e, xb);
  const float a = mu * L.dtr;
  const float b = ep.w * L.sq * w;
  float xn = xb + a + b;
  const bool acc = at_v ? (xn >= 0.0f) : (xn > 0.0f);
  L.e = e;
  L.ep = ep;
  if (acc) {
    if (p.reflect > 0.0f && xn > p.reflect) xn = fmaxf(2.0f * p.reflect - xn, 0.0f);
    L.x = xn;
    return true;
  }
  L.x = 0.0f;
  if (at_v) {  // failed excursion: consume its return time (Alg. 1)
    const float alpha = (w * w * ep.w * ep.w) / (mu * mu * L.dtr);
    L.dtr = (1.0f - alpha) * L.dtr;
    if (L.dtr <= 0.0f) return true;
    if (L.M >= p.cap) {
      L.trunc = true;
      return true;
    }
  } else {  // free step overshot: split at the vertex
    float s = solve_first_passage_s<float>(a, b, xb);
    if (s < 0.0f) s = 1.0f;
    L.dtr = fmaxf((1.0f - s * s) * L.dtr, 0.0f);
  }
  L.sq = sqrtf(L.dtr);
  return false;
}

// One trip of the general-graph state machine (kernels.py:223-288 semantics).
__device__ __forceinline__ bool general_trip(Lane &L, const NativeGraph &G, const Smem &S,
                                             const NatParams &p, float z, uint32_t u) {
  const bool at_init = !(L.x > 0.0f);
  const bool at_term = !(L.x < L.ep.x);
  if (at_init || at_term) {  // resample the exit slot at the hit vertex
    const int off = at_init ? L.ev.x : L.ev.z;
    const int deg = at_init ? L.ev.y : L.ev.w;
    const int s = alias_pick(S.col, off, deg, u);
    L.e = s & 0x7fffffff;
    L.ep = S.edge[L.e];
    L.ev = S.edgev[L.e];
    L.x = s < 0 ? L.ep.x : 0.0f;
  }
  const float l = L.ep.x;
  const float mu = drift(G, L.ep, L.e, L.x);
  const float a = mu * L.dtr;
  const float b = L.ep.w * L.sq * z;
  const float xn = L.x + a + b;
  if (xn > 0.0f && xn < l) {
    L.x = xn;
    return true;
  }
  L.M += 1;
  float s;
  if (xn <= 0.0f) {
    s = solve_first_passage_s<float>(a, b, L.x);
    L.x = 0.0f;
  } else {
    s = solve_first_passage_s<float>(-a, -b, l - L.x);
    L.x = l;
  }
  if (s < 0.0f) s = 1.0f;
  L.dtr = (1.0f - s * s) * L.dtr;
  if (L.dtr <= 0.0f) return true;
  if (L.M >= p.cap) {
    L.trunc = true;
    return true;
  }
  L.sq = sqrtf(L.dtr);
  return false;
}

__device__ __forceinline__ Block native_block(uint64_t seed, uint32_t pair, uint32_t domain,
                                              uint64_t id) {
  return philox4x32_10(Block{pair, domain, (uint32_t)id, (uint32_t)(id >> 32)}, (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

template <bool STAR>
__device__ __forceinline__ void place_native(Lane &L, const NativeGraph &G, const Smem &S,
                                             const NatParams &p, uint64_t id) {
  if (p.init_kind == GSDE_INIT_POINT) {
    L.e = p.init_edge;
    L.x = p.init_x;
  } else {
    const Block r = native_block(p.seed, 0u, kDomainPlace, id);
    const double u = (double)((((uint64_t)r.x << 32) | r.y) >> 11) * kInv2p53;
    const double u2 = (double)((((uint64_t)r.z << 32) | r.w) >> 11) * kInv2p53;
    int e = (int)(u * (double)G.n_edges);
    if (e >= G.n_edges) e = G.n_edges - 1;
    const double le = (double)S.edge[e].x;
    L.e = e;
    L.x = (float)(u2 * (le < p.init_xmax ? le : p.init_xmax));
  }
  L.ep = S.edge[L.e];
  if (!STAR) L.ev = S.edgev[L.e];
}

template <bool STAR>
__global__ void __launch_bounds__(kThreads) native_ensemble_kernel(NativeGraph G, NatParams p,
                                                                  gsde_out o) {
  const int nb = p.cap + 1;
  const Smem S = smem_setup(G, nb, p.smem_graph, STAR);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < p.n;
  Lane L{};
  int steps_left = p.n_steps;
  int64_t cross = 0, events = 0, truncs = 0;
  int64_t t_cross = 0, t_events = 0, t_trunc = 0;
  uint32_t pair = 0;
  uint64_t id = (uint64_t)(p.id_offset + i);
  auto start = [&]() {
    id = (uint64_t)(p.id_offset + i);
    place_native<STAR>(L, G, S, p, id);
    L.dtr = p.dt;
    L.sq = p.sqdt;
    L.M = 0;
    L.trunc = false;
    steps_left = p.n_steps;
    cross = events = truncs = 0;
    pair = 0;
  };
  auto finish = [&]() {
    t_cross += cross;
    t_events += events;
    t_trunc += truncs;
    ensemble_epilogue(o, i, L.e, (double)L.x, cross, events, truncs);
    i += stride;
    active = i < p.n;
    if (active) start();
  };
  // one trip; returns true when the particle finished its last step
  auto trip = [&](float z, uint32_t u) -> bool {
    const bool done = STAR ? star_trip(L, G, S, p, z, u) : general_trip(L, G, S, p, z, u);
    if (!done) return false;
    if (L.M > 0) {
      cross += L.M;
      events += 1;
      truncs += L.trunc ? 1 : 0;
      mh_add(S, L.M > p.cap ? p.cap : L.M);
    }
    L.M = 0;
    L.trunc = false;
    L.dtr = p.dt;
    L.sq = p.sqdt;
    return --steps_left == 0;
  };
  if (active) {
    start();
    if (p.n_steps == 0) {  // placement only (engine.py:329-336)
      while (active) finish();
    }
  }
  while (__any_sync(0xffffffffu, active)) {
    if (active) {
      const Block r = native_block(p.seed, pair++, kDomainEnsemble, id);
      float z0, z1;
      box_muller(r.x, r.y, z0, z1);
      // a lane whose particle finishes on the first trip idles on the second
      // so that the next particle starts on a fresh block (pair 0)
      if (trip(z0, r.z) || trip(z1, r.w)) finish();
    }
  }
  if (o.totals) {
    warp_add_i64(&o.totals[0], t_cross);
    warp_add_i64(&o.totals[1], t_events);
    warp_add_i64(&o.totals[2], t_trunc);
  }
  mh_flush(S, nb, o.m_hist);
}

// Vertex trials: one macro step per trial, started at the vertex
// (kernels.py:447-521); fused exit counts and M histogram (incl. M = 0).
template <bool STAR>
__global__ void __launch_bounds__(kThreads) native_trials_kernel(NativeGraph G, NatParams p,
                                                                gsde_trials_out o, int priv_exit) {
  const int nb = p.cap + 1;
  const Smem S = smem_setup(G, nb, p.smem_graph, STAR);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // lane-private exit counters live after the staged graph (host sized it)
  int *s_exit = nullptr;
  if (priv_exit) {
    size_t off = align16((size_t)(kPriv * kThreads + nb) * sizeof(int));
    if (p.smem_graph)
      off += (size_t)G.n_edges * (STAR ? 16 : 32) + (size_t)G.n_slots * 16;
    s_exit = reinterpret_cast<int *>(smem_raw + off);
    for (int j = threadIdx.x; j < G.n_edges * kThreads; j += blockDim.x) s_exit[j] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < p.n;
  Lane L{};
  uint32_t pair = 0;
  uint64_t id = 0;
  int64_t t_M = 0, t_ev = 0, t_tr = 0;
  auto start = [&]() {
    id = (uint64_t)(p.id_offset + i);
    L.e = STAR ? 0 : p.start_edge;
    L.x = STAR ? 0.0f : p.start_x;
    L.ep = S.edge[L.e];
    if (!STAR) L.ev = S.edgev[L.e];
    L.dtr = p.dt;
    L.sq = p.sqdt;
    L.M = 0;
    L.trunc = false;
    pair = 0;
  };
  auto finish = [&]() {
    if (o.M) o.M[i] = L.M;
    if (o.edge) o.edge[i] = L.e;
    if (o.x) o.x[i] = (double)L.x;
    if (o.trunc) o.trunc[i] = L.trunc ? 1 : 0;
    if (s_exit)
      s_exit[L.e * kThreads + threadIdx.x] += 1;
    else if (o.exit_counts)
      add_i64(&o.exit_counts[L.e], 1);
    mh_add(S, L.M > p.cap ? p.cap : L.M);
    t_M += L.M;
    t_ev += L.M > 0;
    t_tr += L.trunc;
    i += stride;
    active = i < p.n;
    if (active) start();
  };
  if (active) start();
  while (__any_sync(0xffffffffu, active)) {
    if (active) {
      const Block r = native_block(p.seed, pair++, kDomainTrials, id);
      float z0, z1;
      box_muller(r.x, r.y, z0, z1);
      const bool d0 = STAR ? star_trip(L, G, S, p, z0, r.z) : general_trip(L, G, S, p, z0, r.z);
      if (d0 || (STAR ? star_trip(L, G, S, p, z1, r.w) : general_trip(L, G, S, p, z1, r.w)))
        finish();
    }
  }
  if (o.totals) {
    warp_add_i64(&o.totals[0], t_M);
    warp_add_i64(&o.totals[1], t_ev);
    warp_add_i64(&o.totals[2], t_tr);
  }
  mh_flush(S, nb, o.m_hist);
  if (s_exit && o.exit_counts) {
    for (int e = threadIdx.x; e < G.n_edges; e += blockDim.x) {
      int64_t v = 0;
      for (int t = 0; t < kThreads; ++t) v += s_exit[e * kThreads + t];
      if (v) add_i64(&o.exit_counts[e], v);
    }
  }
}

// Standalone snapshot histogram (histogram_accumulate): block-private shared
// counters when the grid fits, global red.add otherwise.
__global__ void __launch_bounds__(256) histogram_kernel(int64_t n, const int64_t *edge,
                                                        const double *x,
                                                        const int64_t *offsets,
                                                        const int64_t *counts,
                                                        const double *dx, int64_t n_cells,
                                                        int64_t *hist, int use_smem) {
  extern __shared__ unsigned long long s_h[];
  if (use_smem) {
    for (int64_t j = threadIdx.x; j < n_cells; j += blockDim.x) s_h[j] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t c = hist_cell(offsets, counts, dx, (int)edge[i], x[i]);
    if (use_smem)
      atomicAdd(&s_h[c], 1ull);
    else
      add_i64(&hist[c], 1);
  }
  if (use_smem) {
    __syncthreads();
    for (int64_t j = threadIdx.x; j < n_cells; j += blockDim.x)
      if (s_h[j]) add_i64(&hist[j], (int64_t)s_h[j]);
  }
}

size_t smem_bytes(const gsde_graph *g, int nb, int stage, bool priv_exit) {
  size_t b = ((size_t)(kPriv * kThreads + nb) * sizeof(int) + 15) & ~size_t(15);
  if (stage) b += (size_t)g->E * (g->is_star ? 16 : 32) + (size_t)g->S * 16;
  if (priv_exit) b += (size_t)g->E * kThreads * sizeof(int);
  return b;
}

template <class K>
int occupancy_grid(K kernel, size_t smem, int device, int64_t n_items) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t full = (int64_t)dev_info(device).sm_count * per_sm;
  const int64_t need = (n_items + kThreads - 1) / kThreads;
  return (int)(need < full ? (need < 1 ? 1 : need) : full);
}

NatParams make_params(const gsde_graph *g, uint64_t seed, int64_t n, int64_t off, double dt,
                      int32_t cap) {
  NatParams p{};
  p.seed = seed;
  p.n = n;
  p.id_offset = off;
  p.cap = cap;
  p.dt = (float)dt;
  p.sqdt = sqrtf((float)dt);
  p.smem_graph = g->nat_graph_smem > 0 ? 1 : 0;
  return p;
}

cudaError_t set_smem_attr(const void *fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

cudaError_t launch_native_ensemble(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                   cudaStream_t s) {
  NatParams p = make_params(g, a.seed, a.n_particles, a.pid_offset, a.dt, a.cap);
  p.n_steps = (int32_t)a.n_steps;
  p.reflect = (float)a.reflect_len;
  p.init_kind = a.init_kind;
  p.init_edge = (int32_t)a.init_edge;
  p.init_x = (float)a.init_x;
  p.init_xmax = a.init_xmax;
  const size_t smem = smem_bytes(g, a.cap + 1, p.smem_graph, false);
  cudaError_t err;
  if (g->is_star) {
    auto k = native_ensemble_kernel<true>;
    if ((err = set_smem_attr((const void *)k, smem)) != cudaSuccess) return err;
    k<<<occupancy_grid(k, smem, g->device, a.n_particles), kThreads, smem, s>>>(g->nat, p, o);
  } else {
    auto k = native_ensemble_kernel<false>;
    if ((err = set_smem_attr((const void *)k, smem)) != cudaSuccess) return err;
    k<<<occupancy_grid(k, smem, g->device, a.n_particles), kThreads, smem, s>>>(g->nat, p, o);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_native_trials(const gsde_graph *g, const gsde_trials &a,
                                 const gsde_trials_out &o, cudaStream_t s) {
  NatParams p = make_params(g, a.seed, a.n_trials, a.trial_offset, a.dt, a.cap);
  p.start_edge = (int32_t)a.start_edge;
  p.start_x = (float)a.start_x;
  const int priv_exit = (o.exit_counts && g->E <= 32) ? 1 : 0;
  const size_t smem = smem_bytes(g, a.cap + 1, p.smem_graph, priv_exit);
  cudaError_t err;
  if (g->is_star) {
    auto k = native_trials_kernel<true>;
    if ((err = set_smem_attr((const void *)k, smem)) != cudaSuccess) return err;
    k<<<occupancy_grid(k, smem, g->device, a.n_trials), kThreads, smem, s>>>(g->nat, p, o,
                                                                              priv_exit);
  } else {
    auto k = native_trials_kernel<false>;
    if ((err = set_smem_attr((const void *)k, smem)) != cudaSuccess) return err;
    k<<<occupancy_grid(k, smem, g->device, a.n_trials), kThreads, smem, s>>>(g->nat, p, o,
                                                                              priv_exit);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_histogram(int64_t n, const int64_t *edge, const double *x,
                             const int64_t *offsets, const int64_t *counts, const double *dx,
                             int64_t n_cells, int64_t *hist, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int device = 0;
  cudaGetDevice(&device);
  const size_t bytes = (size_t)n_cells * sizeof(unsigned long long);
  const int use_smem = bytes <= 32 * 1024 ? 1 : 0;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)dev_info(device).sm_count * 4;
  if (blocks > cap) blocks = cap;
  histogram_kernel<<<(int)blocks, 256, use_smem ? bytes : 0, s>>>(n, edge, x, offsets, counts,
                                                                  dx, n_cells, hist, use_smem);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gsde
