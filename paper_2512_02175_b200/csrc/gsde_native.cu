// gsde_native.cu -- the B200 production stepper (FP32, native stream).
//
// Design:
//  * one particle per lane, persistent grid (SMs x resident CTAs), particles
//    handed out dynamically (warp-aggregated atomic on a grid-wide counter);
//    all per-particle state lives in registers for the whole run;
//  * flattened state machine: every loop trip performs exactly one proposal
//    per lane -- a free Euler-Maruyama step or one vertex iteration -- so the
//    split / excursion loops of kernels.py:198-220 and :257-288 become extra
//    trips of the same loop body and never serialise a warp;
//  * common path is branch-free: a lane strictly inside an edge always starts
//    a fresh macro step (dtr == dt), so its proposal is 3 FFMAs with cached
//    per-edge constants and the accept test is 2-4 compares.  Everything else
//    (vertex iterations, splits, reflections, statistics) is one divergent
//    "rare" region per trip, followed by an explicit warp reconvergence;
//  * iterations of Q = 14 trips; the vertex slots (trip 0, and trip 7 on
//    general graphs) are the only trips that carry the divergent vertex
//    region; lanes at a vertex wait for a slot, particles start on iteration
//    boundaries, so the warp resolves its vertices together;
//  * RNG: 4 Philox4x32-10 blocks per iteration, counter (per-particle block
//    index, domain, particle id) under the seed: 14 words -> Box-Muller ->
//    the trips' Gaussians, one 32-bit exit uniform per slot.  Every iteration
//    consumes the same amount, so all lanes generate blocks in lockstep;
//  * exit slot: per-vertex alias table, one 16 B column record per pick;
//  * star / small graphs: edge records and alias columns staged in shared
//    memory; large networks read them through L2 (__ldg);
//  * estimators fused: M histogram in shared counters (one shared atomic
//    per step with M > 0); totals in shared memory; occupancy and snapshot
//    histogram in the particle epilogue.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "gsde_epilogue.cuh"

namespace gsde {
namespace {

constexpr int kThreads = 256;
#ifndef GSDE_MIN_BLOCKS
#define GSDE_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = GSDE_MIN_BLOCKS;  // 4: caps registers at 64 -> 32 warps / SM
constexpr int kMinBlocksStar = 3;            // star-graph ensembles: <= 85 registers
// trials: the compiler settles at 40 registers (48 warps / SM) under a 64-register
// bound; the same kernel scheduled under a 51-register bound (5 blocks) ran 3% slower
constexpr int kMinBlocksTrials = 4;
constexpr int kTrialWaves = 4;  // trials grid: resident blocks x 4
constexpr int kTrips = 14;     // ensemble: trips per iteration
#ifndef GSDE_EXIT_PRIV
#define GSDE_EXIT_PRIV 1  // trials: lane-private exit counters (+0.6% over shared atomics)
#endif
constexpr uint32_t kDomainEnsemble = 0u;
constexpr uint32_t kDomainTrials = 1u;
constexpr uint32_t kDomainPlace = 0xFFFFFFFFu;

struct NatParams {
  uint32_t rk[20];    // Philox round keys of the seed (constant-bank operands)
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
  // shared 32-bit counters stay exact: each warp of an ensemble block takes
  // particles only while it has taken fewer than warp_budget (0 = no limit),
  // and FULL kernels keep only the first mh_smem M bins in shared memory (0
  // when a block could count 2^32)
  uint32_t warp_budget;
  int32_t mh_smem;
};

// Injected reference draws (Cfg::INJ ensembles): per particle [stride] raw
// words and their normals, consumed in the reference's order (kernels.py:55-64)
struct InjParams {
  const uint64_t *raw;
  const double *normal;
  int64_t stride;
  // the reference's slot tables in CSR order (exit slots by inverse CDF)
  const uint64_t *thresh;
  const int32_t *vedges;
  const uint8_t *vorient;
  // FULL / INJ kernels (the last kernel parameter, so it may grow without
  // moving the others -- see KOut): GSDE_INIT_STATE's per-particle SoA state,
  // the NATIVE stream's next Philox block per particle, and the per-particle
  // counter output
  const int32_t *st_e;
  const float *st_x;
  const uint64_t *st_k;
  uint64_t *counter;
  // fused final-state estimators in shared memory (0 = global atomics): byte
  // offset of the block's uint32 counters -- edge_counts [E] then the
  // snapshot histogram [n_cells] -- flushed to the call's int64 arrays once
  unsigned bin_off;
  int bin_edges, bin_cells;
  // streamed results (gsde_out.progress): particle i's range counter,
  // progress[(progress_base + i) >> progress_shift]
  unsigned *progress;
  int64_t progress_base;
  int progress_shift;
};

// Publish particle i's stored per-particle outputs: a GPU-scope release add on
// its range counter (a copy stream waits on the counter, then reads the range)
__device__ __forceinline__ void publish_particle(const InjParams &q, int64_t i) {
  unsigned *c = q.progress + ((q.progress_base + i) >> q.progress_shift);
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}

__device__ __forceinline__ float fast_sqrt(float v) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ float fast_lg2(float v) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Box-Muller on two 32-bit words: u1 in (0, 1] with 2^-33 resolution near 0
// (|z| <= sqrt(2 * 33 ln 2) = 6.77), angle uniform on [-pi, pi).  The tail cut
// drops P(|z| > 6.77) = 1.3e-11 of the Gaussian mass per draw, so any
// estimator moves by O(1e-11) -- far below the Monte-Carlo resolution of the
// largest runs here (1e13 psteps: relative SE ~3e-7).  Returns z / sqrt(2 ln 2): the
// native edge records carry sigma * sqrt(2 ln 2) (gsde_abi.cu), so every
// sigma * z product is unchanged and the scale costs no instruction here.
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float &z0, float &z1) {
  const float u1 = fmaf((float)a, 0x1p-32f, 0x1p-33f);
  // u1 <= 1 so -log2 u1 >= 0 (lg2.approx(1) == 0)
  const float r = fast_sqrt(-fast_lg2(u1));
  float s, c;
  __sincosf((float)(int32_t)b * 1.4629180792671596e-9f, &s, &c);  // pi * 2^-31
  z0 = r * c;
  z1 = r * s;
}

__device__ __forceinline__ float fast_rcp(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Split time of an overshooting proposal, FP32, branch-free.  Callers ask
// only when the proposal x' = c + a + b reached the vertex at distance c >= 0
// (a + b + c <= 0).  For c > 0, a s^2 + b s + c then has exactly one root in
// (0, 1] and it is the reference's answer -- the smallest non-negative root
// clamped to 1, -1 (-> 1) if none (kernels.py:88-131, :191-192).  Both cases
// of that root without cancellation, D = b^2 - 4ac:
//   b <  0:  s = 2c / (|b| + sqrt(D))
//   b >= 0:  s = (|b| + sqrt(D)) / (-2a)      (overshoot forces a < 0)
// c = 0 (a zero-time re-hit from the vertex): b <= 0 -> 0 (kernels.py:99-107);
// b > 0 falls out of the second form as -b/a.  Rounding that leaves [0, 1]
// (or NaN) falls back to 1.
__device__ __forceinline__ float split_root(float a, float b, float c) {
  const float t = fabsf(b) + fast_sqrt(fmaxf(fmaf(b, b, -4.0f * a * c), 0.0f));
  const bool neg = b < 0.0f;
  const float s = (neg ? 2.0f * c : t) * fast_rcp(neg ? t : -2.0f * a);
  if (c == 0.0f && b <= 0.0f) return 0.0f;
  return (s >= 0.0f && s <= 1.0f) ? s : 1.0f;
}

// Philox4x32-10 with the key schedule precomputed in the kernel parameters:
// per round 2 IMAD.WIDE + 2 LOP3 (the round key is a constant-bank operand).
__device__ __forceinline__ Block native_block(const NatParams &p, uint32_t pair, uint32_t domain,
                                              uint64_t id) {
  Block c{pair, domain, (uint32_t)id, (uint32_t)(id >> 32)};
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_hilo(c.x, kPhiloxM0, hi0, lo0);
    mul_hilo(c.z, kPhiloxM1, hi1, lo1);
    c = Block{hi1 ^ c.y ^ p.rk[2 * r], lo1, hi0 ^ c.w ^ p.rk[2 * r + 1], lo0};
  }
  return c;
}

__host__ __device__ __forceinline__ size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// Graph tables: shared-memory copies (SMEM) or global/L2 (read-only path).
template <bool SMEM>
struct Tables {
  const float4 *edge;
  const int4 *edgev;
  const int4 *col;
  const int4 *fat;  // L2 path: fat alias columns
  const int4 *ufat; // L2 path, uniform exits: {slot, edge record, endpoint record}
  __device__ __forceinline__ float4 E(int e) const { return SMEM ? edge[e] : __ldg(edge + e); }
  __device__ __forceinline__ int4 V(int e) const { return SMEM ? edgev[e] : __ldg(edgev + e); }
  __device__ __forceinline__ int4 C(int j) const { return SMEM ? col[j] : __ldg(col + j); }
};

// Alias pick with a 32-bit uniform: column = floor(u * deg), then the
// column's threshold on the low word.  Returns edge | orient << 31.
template <bool SMEM>
__device__ __forceinline__ int alias_pick(const Tables<SMEM> &T, int off, int deg, uint32_t u) {
  uint32_t hi, lo;
  mul_hilo(u, (uint32_t)deg, hi, lo);
  const int4 c = T.C(off + (int)hi);
  return lo < (uint32_t)c.x ? c.y : c.z;
}

// Injected-draw parity mode: the reference's exit slot for a raw draw -- the
// first slot j of [off, off + deg) with (r >> 11) <= thresh[j], else the last
// (kernels.py:134-143) -- as edge | orient << 31 like an alias pick.
template <class L_>
__device__ __forceinline__ int ref_pick(const L_ &L, int off, int deg, uint64_t raw) {
  const uint64_t u53 = raw >> 11;
  int j = off;
  while (j < off + deg - 1 && u53 > __ldg(L.thr + j)) ++j;
  return __ldg(L.ved + j) | ((int)__ldg(L.vor + j) << 31);
}

__device__ float drift_tab(const NativeGraph &G, int e, float x) {
  const int lo = G.tab_off[e], hi = G.tab_off[e + 1];
  if (x <= G.tab_x[lo]) return G.tab_mu[lo];
  if (x >= G.tab_x[hi - 1]) return G.tab_mu[hi - 1];
  int j = lo + 1;
  while (G.tab_x[j] < x) ++j;
  const float x0 = G.tab_x[j - 1];
  const float t = (x - x0) / (G.tab_x[j] - x0);
  return G.tab_mu[j - 1] + t * (G.tab_mu[j] - G.tab_mu[j - 1]);
}

// Compile-time kernel variant.
template <bool STAR_, bool SMEM_, bool TAB_, bool REFLECT_, bool OCC_, bool ZD_ = false,
          bool INJ_ = false, bool FULL_ = false, bool PP_ = true, bool CD_ = false,
          bool UNI_ = false>
struct Cfg {
  static constexpr bool STAR = STAR_;        // star graph (one vertex, semi-infinite edges)
  static constexpr bool SMEM = SMEM_;        // graph tables staged in shared memory
  static constexpr bool TAB = TAB_;          // some edge has a tabulated drift
  static constexpr bool REFLECT = REFLECT_;  // star mirror wall enabled
  static constexpr bool OCC = OCC_;          // time-integrated occupation histogram
  static constexpr bool ZD = ZD_;            // Brownian: every drift is zero
  // parity mode: the production kernel fed the reference's injected draws
  // (one per use, in the reference's order) and its inverse-CDF exit slots
  static constexpr bool INJ = INJ_;
  // The full-featured kernel, chosen by the host only when a run needs it:
  // int64 per-particle counts, M bins beyond kMaxSmemBins in global memory and
  // a 64-bit Philox block index (runs where a 32-bit one could overflow),
  // per-particle state-in (GSDE_INIT_STATE) and the per-particle counter
  // output (resume).  The common configuration keeps the lean kernel, whose
  // register allocation the extra code would otherwise perturb.
  static constexpr bool FULL = FULL_;
  static constexpr bool STATE = FULL_ || INJ_;  // state-in / counter out compiled in
  // Per-particle counters (crossings, events, truncations per particle) and
  // the per-particle result arrays.  Off (the "lean" ensemble kernel) when a
  // call asks only for fused estimators: the run totals then follow from the
  // M histogram (M <= cap, so crossings = sum b h[b], events = sum_{b>=1} h[b])
  // plus one shared truncation counter, and the lane carries three
  // registers and a per-step update less.
  static constexpr bool PP = PP_;
  // run totals from the block's M histogram + the shared truncation counter
  // (every kernel but FULL -- global M bins -- and INJ -- overrun counts)
  static constexpr bool HT = !FULL_ && !INJ_;
  // every drift constant in x (general graphs; advection fields such as C4's
  // drift from_flux): mu(x) = mu_a, the proposal one FFMA shorter and the
  // lane one register lighter -- bit-identical to the generic kernel, whose
  // fmaf(mu_b = 0, x, mu_a) is exactly mu_a
  static constexpr bool CD = CD_;
  static_assert(!(CD_ && (TAB_ || ZD_)), "constant drift excludes tabulated / zero drift");
  // every exit column keeps its own slot (equal jump weights at every vertex,
  // as on C2 and C4): the exit pick is the column -- no threshold compare, no
  // candidate selects, and on L2-resident graphs a 48 B record (the slot and
  // its edge's records) instead of 80 B; the same slot as the alias pick
  static constexpr bool UNI = UNI_;
  static_assert(!(UNI_ && INJ_), "uniform exits: native-stream kernels");
  static_assert(PP_ || !(INJ_ || FULL_), "INJ / FULL kernels keep per-particle counters");
  using Cnt = std::conditional_t<FULL_, long long, int>;
  static_assert(!(TAB_ && ZD_), "a tabulated drift is not zero");
};

// Occupation histogram: grid arrays + counters (shared uint32 or global int64).
struct Occ {
  const int64_t *off, *cnt;
  const double *dx;
  int64_t *out;
  unsigned *s_cnt;   // shared counters, or null -> global atomics
  int32_t every, start;
  const float4 *tab;  // shared per-edge {first cell, cells - 1, 1/dx, -} or null -> global
  // grid cell of position x on edge e (floor(x/dx) clipped to the edge's cells)
  __device__ __forceinline__ int cell(int e, float x) const {
    int o, top;
    float inv;
    if (tab) {
      const float4 r = tab[e];
      o = __float_as_int(r.x);
      top = __float_as_int(r.y);
      inv = r.z;
    } else {
      o = (int)__ldg(off + e);
      top = (int)__ldg(cnt + e) - 1;
      inv = (float)(1.0 / __ldg(dx + e));
    }
    const int local = __float2int_rz(fminf(x * inv, (float)top));
    return o + (local < 0 ? 0 : local);
  }
};
constexpr int kOccTabEdges = 1024;  // per-edge occupation records staged in shared memory

// Shared block state: M histogram, totals, staged
// graph, occupation counters.
struct Shared {
  unsigned *mh;              // [min(cap+1, kMaxSmemBins)]
  int nbs;                   // M bins in shared memory (FULL kernels: the rest in mh_g)
  int64_t *mh_g;             // the call's M histogram (global: FULL bins, carries)
  unsigned long long *tot;   // [4]
  unsigned *exit_cnt;        // trials: exit counts [E] (shared atomics) or null
  unsigned *occ;             // [n_cells] or null
};

// M-histogram bins kept in shared memory: caps up to 8191 (32 KB); a larger
// cap (the reference accepts any) selects a FULL kernel, which counts the
// bins beyond in global memory
constexpr int kMaxSmemBins = 8192;
__host__ __device__ __forceinline__ int smem_bins(int nb) {
  return nb < kMaxSmemBins ? nb : kMaxSmemBins;
}

__device__ __forceinline__ size_t shared_head_bytes(int nbs) {
  return align16((size_t)nbs * sizeof(int)) + 4 * sizeof(unsigned long long);
}

// (FULL: the shared M bins are capped at kMaxSmemBins; otherwise the host
// guarantees cap + 1 <= kMaxSmemBins)
template <bool STAR, bool SMEM, bool FULL = false>
__device__ __forceinline__ void shared_setup(const NativeGraph &G, int nb, int64_t *m_hist,
                                             Shared &S, Tables<SMEM> &T, bool exit_cnt,
                                             int occ_cells, int mh_smem = kMaxSmemBins) {
  extern __shared__ __align__(16) unsigned char smem[];
  // (FULL: the first mh_smem bins -- 0 when a block could count 2^32 -- in
  // shared memory, the rest in the call's int64 histogram)
  const int nbs = FULL ? min(smem_bins(nb), mh_smem) : nb;
  S.mh = reinterpret_cast<unsigned *>(smem);
  S.mh_g = m_hist;
  if (FULL) S.nbs = nbs;
  S.tot = reinterpret_cast<unsigned long long *>(
      smem + align16((size_t)nbs * sizeof(int)));
  for (int j = threadIdx.x; j < nbs; j += blockDim.x) S.mh[j] = 0u;
  if (threadIdx.x < 4) S.tot[threadIdx.x] = 0ull;
  size_t off = shared_head_bytes(nbs);
  T.edge = G.edge;
  T.edgev = G.edgev;
  T.col = G.col;
  T.fat = G.fat;
  T.ufat = G.ufat;
  if (SMEM) {
    float4 *se = reinterpret_cast<float4 *>(smem + off);
    off += (size_t)G.n_edges * sizeof(float4);
    int4 *sv = reinterpret_cast<int4 *>(smem + off);
    if (!STAR) off += (size_t)G.n_edges * sizeof(int4);
    int4 *sc = reinterpret_cast<int4 *>(smem + off);
    off += (size_t)G.n_slots * sizeof(int4);
    for (int j = threadIdx.x; j < G.n_edges; j += blockDim.x) {
      se[j] = G.edge[j];
      if (!STAR) sv[j] = G.edgev[j];
    }
    for (int j = threadIdx.x; j < G.n_slots; j += blockDim.x) sc[j] = G.col[j];
    T.edge = se;
    T.edgev = sv;
    T.col = sc;
  }
  S.exit_cnt = nullptr;
  if (exit_cnt) {
    S.exit_cnt = reinterpret_cast<unsigned *>(smem + off);
    off += align16((size_t)G.n_edges * (GSDE_EXIT_PRIV ? kThreads : 1) * sizeof(unsigned));
    for (int j = threadIdx.x; j < G.n_edges * (GSDE_EXIT_PRIV ? kThreads : 1); j += blockDim.x)
      S.exit_cnt[j] = 0u;
  }
  S.occ = nullptr;
  if (occ_cells > 0) {
    S.occ = reinterpret_cast<unsigned *>(smem + off);
    for (int j = threadIdx.x; j < occ_cells; j += blockDim.x) S.occ[j] = 0u;
  }
  __syncthreads();
}

// One shared atomic per macro step with M > 0 (ATOMS.POPC.INC, no return
// value).  Measured against lane-private counters for the small bins (the
// former layout, 8 KB per block, load-add-store with per-lane addressing):
// +0.4% star3, +1% hub64, +0.8% vascular, +4% C3 trials.  Shared counters are
// 32-bit: the host bounds what one block can count (per-block particle budget,
// launch_native_ensemble) and otherwise keeps the bins in global memory
// (S.nbs = 0); a checked add that carries 2^31 into the int64 arrays cost
// 2-9% (measured) and was not kept.
template <bool FULL>
__device__ __forceinline__ void mh_add(const Shared &S, int bin) {
  if (!FULL || bin < S.nbs)
    atomicAdd(&S.mh[bin], 1u);
  else if (S.mh_g)
    add_i64(&S.mh_g[bin], 1);
}

template <bool FULL = false, bool TOTALS = false>
__device__ void shared_flush(const Shared &S, int nb, int64_t *m_hist, int occ_cells,
                             int64_t *occ_out, int64_t *totals = nullptr) {
  __syncthreads();
  const int nbs = FULL ? S.nbs : nb;
  int64_t t_cross = 0, t_events = 0;
  for (int b = threadIdx.x; b < nbs; b += blockDim.x) {
    const int64_t v = S.mh[b];
    if (v && m_hist) add_i64(&m_hist[b], v);
    if (TOTALS && b > 0) {
      t_cross += (int64_t)b * v;
      t_events += v;
    }
  }
  if (TOTALS && totals) {
    warp_add_i64(&totals[0], t_cross);
    warp_add_i64(&totals[1], t_events);
    if (threadIdx.x == 0 && S.tot[2]) add_i64(&totals[2], (int64_t)S.tot[2]);
  }
  if (S.occ)
    for (int j = threadIdx.x; j < occ_cells; j += blockDim.x)
      if (S.occ[j]) add_i64(&occ_out[j], (int64_t)S.occ[j]);
}

// Per-lane simulation state.
template <class C>
struct Lane {
  int e;           // current edge
  float x;         // position on e
  float dtr, sq;   // time left in the current macro step and its sqrt
  int M;           // vertex resolutions in the current macro step
  bool trunc;
  // a hit whose split time is not yet resolved (pending): star x = -start,
  // general steps_left < 0 with x = start; its Gaussian pz (a, b re-derived).
  // General ensembles: steps_left < 0 with pz = NaN = at the vertex x, no hit
  // to resolve (a step that ended there, or a start there)
  float px, pz;
  float mu_a, mu_b, sig, sig_sqdt;  // cached drift / diffusion of e
  float len;       // edge length (star: mirror wall or +inf)
  float kex;       // star: sig^2 / mu(0)^2 of e (the failed-excursion time, per w^2)
  int4 ev;         // endpoint alias info of e (general graphs)
  int steps_left;
  typename C::Cnt cross, events, truncs;
  int occ_left;    // steps to the next occupation sample
  // Cfg::INJ only: the reference's slot tables, this particle's injected
  // draws and the next draw index
  const uint64_t *thr;
  const int32_t *ved;
  const uint8_t *vor;
  const uint64_t *ir;
  const double *inn;
  int k, kmax;
  bool over;       // ran past the injected draws

  // next injected normal, scaled like box_muller's output (z / sqrt(2 ln 2))
  __device__ __forceinline__ float inj_gauss() {
    if (k < kmax) return (float)(__ldg(inn + k++) * 0.84932180028801907);
    over = true;
    return 0.0f;
  }
  __device__ __forceinline__ uint64_t inj_raw() {
    if (k < kmax) return __ldg(ir + k++);
    over = true;
    return 0ull;
  }

  __device__ __forceinline__ void load_edge(const Tables<C::SMEM> &T, const Occ &O, int e2,
                                            float sqdt, float star_len) {
    const float4 r = T.E(e2);
    e = e2;
    mu_a = r.y;
    mu_b = r.z;
    sig = r.w;
    sig_sqdt = r.w * sqdt;
    if (C::STAR) {
      len = star_len;
      kex = r.x;  // star records: sig^2 / mu(0)^2 (gsde_abi.cu), read by rare_star
    } else {
      len = r.x;
      ev = T.V(e2);
    }
  }

  // general graphs: install already-loaded records of edge e2
  __device__ __forceinline__ void load_edge_rec(const Occ &O, int e2, float4 r, int4 v,
                                                float sqdt) {
    e = e2;
    mu_a = r.y;
    mu_b = r.z;
    sig = r.w;
    sig_sqdt = r.w * sqdt;
    len = r.x;
    ev = v;
  }

  __device__ __forceinline__ float drift(const NativeGraph &G, float at) const {
    if (C::ZD) return 0.0f;
    if (C::CD) return mu_a;
    if (C::TAB && isnan(mu_b)) return drift_tab(G, e, at);
    return fmaf(mu_b, at, mu_a);
  }

  // split time of the pending hit: the proposal x' = px + mu(px) dtr + sig sq pz
  // left the edge through the vertex the lane now sits at (kernels.py:190-195,
  // :276-283); residual time (1 - s^2) dtr
  __device__ __forceinline__ float split_factor(const NativeGraph &G) const {
    const float b = (sig * sq) * pz;
    const bool lo = C::STAR || !(x > 0.0f);
    if (C::ZD) {  // split_root(0, bb, c): the linear root s = -c / bb, same fallbacks
      const float c = lo ? px : len - px, bb = lo ? b : -b;
      if (c == 0.0f) return bb <= 0.0f ? 1.0f : 0.0f;
      const float s = c * fast_rcp(-bb);
      return (s >= 0.0f && s <= 1.0f) ? 1.0f - s * s : 0.0f;
    }
    const float a = drift(G, px) * dtr;
    // one root evaluation for either end (selected operands): a divergent
    // warp would otherwise run both inlined copies
    const float s = split_root(lo ? a : -a, lo ? b : -b, lo ? px : len - px);
    return 1.0f - s * s;
  }

  // macro step finished: statistics, reset for the next step
  __device__ __forceinline__ void step_done(const Shared &S, int cap, float dt, float sqdt) {
    if (M > 0) {
      if constexpr (C::PP) {
        cross += M;
        events += 1;
        truncs += trunc ? 1 : 0;
      }
      // rare: a step cut at the cap -- a 32-bit shared add on the counter's low
      // word (a block counts < 2^32 steps; a 64-bit shared atomic is a CAS loop)
      if (C::HT && trunc) atomicAdd(reinterpret_cast<unsigned *>(&S.tot[2]), 1u);
      mh_add<C::FULL>(S, M > cap ? cap : M);
    }
    M = 0;
    trunc = false;
    dtr = dt;
    sq = sqdt;
  }

  // occupation sample of the state after a completed step (every `every`
  // steps); predicated, so the trips of an iteration stay one straight-line
  // block the compiler can interleave
  __device__ __forceinline__ void occ_tick(const Occ &O, bool done) {
    occ_left -= done ? 1 : 0;
    const bool smp = done && occ_left == 0;
    occ_left = smp ? O.every : occ_left;
    const int cell = O.cell(e, x);
    if (smp) {
      if (O.s_cnt)
        atomicAdd(&O.s_cnt[cell], 1u);
      else
        add_i64(&O.out[cell], 1);
    }
  }
};

// Rare trip of a star graph (kernels.py:146-220).  Lanes arrive here at the
// vertex (x == 0, possibly with an unresolved overshoot from an earlier trip)
// or beyond the optional mirror wall.  Returns true when the macro step
// completed.
#ifndef GSDE_EARLY_PICK
#define GSDE_EARLY_PICK 1  // measured: vascular +1.1% (30.03 -> 29.72 ms)
#endif
#ifndef GSDE_EARLY_SMEM
#define GSDE_EARLY_SMEM 0  // shared-memory tables (hub64): +0.06%, spills the tabulated-drift variants
#endif
#ifndef GSDE_STAR_UNI
#define GSDE_STAR_UNI 0  // uniform-exit pick in star ensembles: measured -0.7% on C1
#endif
#ifndef GSDE_STAR_NEG
#define GSDE_STAR_NEG 0  // measured: star3 -4.7% (the at-vertex flagging costs the region more than the trips save)
#endif
// Star ensembles (PEND): like general graphs, a lane at the vertex carries a
// negative step count -- a pending hit (x its start point, pz its Gaussian) or,
// with pz = NaN, a lane waiting there (a failed excursion, or a step that
// ended at the vertex) -- so the common trip tests one integer.
template <class C>
__device__ __forceinline__ void flag_at_vertex(Lane<C> &L, bool step_done) {
  // (step_done: trip()'s decrement then leaves -(steps_left - 1))
  L.steps_left = step_done ? 2 - L.steps_left : -L.steps_left;
  L.pz = __int_as_float(0x7fffffff);
}

template <class C, bool PEND>
__device__ __forceinline__ bool rare_star(Lane<C> &L, const NativeGraph &G,
                                          const Tables<C::SMEM> &T, const Occ &O,
                                          const NatParams &p, float z, uint32_t u) {
  constexpr bool NEG = PEND && GSDE_STAR_NEG;
  if constexpr (NEG) {
    const bool pend = L.steps_left < 0 && !isnan(L.pz);
    L.steps_left = abs(L.steps_left);
    if (pend) {  // pending hit: x is its start point
      L.px = L.x;
      L.dtr = fmaxf(L.split_factor(G) * L.dtr, 0.0f);
      L.sq = fast_sqrt(L.dtr);
    }
  } else if (PEND && L.x < 0.0f) {  // pending hit: the trip stored -px in x (x > 0 before a hit)
    L.px = -L.x;
    L.dtr = fmaxf(L.split_factor(G) * L.dtr, 0.0f);
    L.sq = fast_sqrt(L.dtr);
  }
  // sample the exit edge, one-sided |W| excursion (kernels.py:198-220)
  L.M += 1;
  if constexpr (C::INJ) {  // the reference's order: the uniform, then the normal
    L.load_edge(T, O, ref_pick(L, 0, G.n_edges, L.inj_raw()) & 0x7fffffff, p.sqdt, L.len);
    z = L.inj_gauss();
  } else {
    const int s = C::UNI ? T.C((int)__umulhi(u, (uint32_t)G.n_edges)).y
                         : alias_pick(T, 0, G.n_edges, u);
    L.load_edge(T, O, s & 0x7fffffff, p.sqdt, L.len);
  }
  const float w = fabsf(z);
  const float mu0 = C::TAB ? L.drift(G, 0.0f) : L.mu_a;  // mu(0) = mu_a (+ mu_b * 0)
  const float xn = C::ZD ? (L.sig * L.sq) * w : fmaf(L.sig * L.sq, w, mu0 * L.dtr);
  if (C::ZD || xn >= 0.0f) {
    L.x = (C::REFLECT && xn > p.reflect) ? fmaxf(2.0f * p.reflect - xn, 0.0f) : xn;
    if (NEG && !(L.x > 0.0f)) flag_at_vertex(L, true);  // (no residual time left: x == 0)
    return true;
  }
  // failed excursion: dt' = (1 - alpha) dt with alpha = w^2 sig^2 / (mu0^2 dt)
  // (kernels.py:210-212), i.e. dt' = dt - w^2 sig^2 / mu0^2 -- one FFMA with the
  // edge's sig^2 / mu0^2 from its record (tabulated drifts: mu0 from the table)
  if constexpr (C::TAB) {
    const float alpha = (w * w * L.sig * L.sig) * fast_rcp(mu0 * mu0 * L.dtr);
    L.dtr = (1.0f - alpha) * L.dtr;
  } else {
    L.dtr = fmaf(-(w * w), L.kex, L.dtr);
  }
  L.x = 0.0f;
  const bool ends = L.dtr <= 0.0f || L.M >= p.cap;
  if (ends) {
    L.trunc = L.dtr > 0.0f;
    if (NEG) flag_at_vertex(L, true);
    return true;
  }
  L.sq = fast_sqrt(L.dtr);
  if (NEG) flag_at_vertex(L, false);
  return false;
}

// Rare trip of a general graph (kernels.py:223-288).  Lanes arrive here at a
// vertex: first resolve a pending hit (residual time, stop / cap checks),
// then resample the exit slot and propose from the new edge's endpoint.
// VTX: an ensemble lane (a step ending at the vertex flags it at-vertex);
// vertex trials end there
template <class C, bool VTX>
__device__ __forceinline__ bool rare_general(Lane<C> &L, const NativeGraph &G,
                                             const Tables<C::SMEM> &T, const Occ &O,
                                             const NatParams &p, float z, uint32_t u) {
  // at a vertex (flag: the step count's sign): a pending hit -- x its start,
  // pz its Gaussian -- or, with pz = NaN (ensembles), a step that ended at
  // the vertex, x the vertex
  const bool pend = L.steps_left < 0 && !isnan(L.pz);
  L.steps_left = abs(L.steps_left);
  // uniform exits on L2-resident graphs (GSDE_EARLY_PICK): the vertex is known
  // once the overshoot's end is, so the exit record's L2 round trip is issued
  // before the split-time math and overlaps it (a step that then ends at the
  // vertex discards it)
  constexpr bool EARLY = (C::SMEM ? GSDE_EARLY_SMEM : GSDE_EARLY_PICK) && C::UNI && !C::INJ;
  int4 ec{}, eer{}, eev{};
  auto early_pick = [&]() {
    const bool at_v0 = !(L.x > 0.0f);
    const int off0 = at_v0 ? L.ev.x : L.ev.z, deg0 = at_v0 ? L.ev.y : L.ev.w;
    if constexpr (C::SMEM) {
      ec.x = T.C(off0 + (int)__umulhi(u, (uint32_t)deg0)).y;
      const float4 r = T.E(ec.x & 0x7fffffff);
      eer = *reinterpret_cast<const int4 *>(&r);
      eev = T.V(ec.x & 0x7fffffff);
    } else {
      const int4 *f = T.ufat + 3 * (off0 + (int)__umulhi(u, (uint32_t)deg0));
      ec = __ldg(f);
      eer = __ldg(f + 1);
      eev = __ldg(f + 2);
    }
  };
  if (EARLY && !pend) early_pick();
  if (pend) {
    L.px = L.x;
    // the proposal that overshot, recomputed bit for bit (a hit on the common
    // path had dtr == dt and sq == sqrt(dt)), tells which end it reached
    const float xn =
        fmaf(L.sig * L.sq, L.pz, C::ZD ? L.px : fmaf(L.drift(G, L.px), L.dtr, L.px));
    L.x = xn <= 0.0f ? 0.0f : L.len;
    if (EARLY) early_pick();
    // (an L1 prefetch of the exit column issued here, ahead of the split
    // math, measured -2.6% on vascular: its address math costs more than the
    // latency it hides at 32 warps / SM)
    L.M += 1;
    L.dtr = L.split_factor(G) * L.dtr;
    // the step ends at the vertex, on the old edge (residual time used up, or
    // the cap): ensembles start the next step there -- flagged at-vertex, no
    // hit to resolve: trip()'s decrement leaves -(steps_left - 1)
    const bool ends = L.dtr <= 0.0f || L.M >= p.cap;
    if (ends) {
      L.trunc = L.dtr > 0.0f;
      if (VTX) {
        L.steps_left = 2 - L.steps_left;
        L.pz = __int_as_float(0x7fffffff);
      }
      return true;
    }
    L.sq = fast_sqrt(L.dtr);
  }
  const bool at_init = !(L.x > 0.0f);
  const int off = at_init ? L.ev.x : L.ev.z, deg = at_init ? L.ev.y : L.ev.w;
  int s;
  if constexpr (C::INJ) {  // the reference's order: the uniform, then the normal
    s = ref_pick(L, off, deg, L.inj_raw());
    L.load_edge(T, O, s & 0x7fffffff, p.sqdt, 0.0f);
    z = L.inj_gauss();
  } else if constexpr (EARLY) {  // records loaded above
    s = ec.x;
    L.load_edge_rec(O, s & 0x7fffffff, *reinterpret_cast<const float4 *>(&eer), eev, p.sqdt);
  } else if constexpr (C::SMEM && C::UNI) {
    s = T.C(off + (int)__umulhi(u, (uint32_t)deg)).y;
    L.load_edge(T, O, s & 0x7fffffff, p.sqdt, 0.0f);
  } else if constexpr (C::SMEM) {
    s = alias_pick(T, off, deg, u);
    L.load_edge(T, O, s & 0x7fffffff, p.sqdt, 0.0f);
  } else if constexpr (C::UNI) {  // one round trip: the slot + its edge's records
    const int4 *f = T.ufat + 3 * (off + (int)__umulhi(u, (uint32_t)deg));
    const int4 c = __ldg(f), er = __ldg(f + 1), ev = __ldg(f + 2);
    s = c.x;
    L.load_edge_rec(O, s & 0x7fffffff, *reinterpret_cast<const float4 *>(&er), ev, p.sqdt);
  } else {  // one round trip: column + both candidates' records in flight together
    uint32_t hi, lo;
    mul_hilo(u, (uint32_t)deg, hi, lo);
    const int4 *f = T.fat + 5 * (off + (int)hi);
    const int4 c = __ldg(f), pe = __ldg(f + 1), pv = __ldg(f + 2), ae = __ldg(f + 3),
               av = __ldg(f + 4);
    const bool prim = lo < (uint32_t)c.x;
    s = prim ? c.y : c.z;
    const int4 er = prim ? pe : ae;
    L.load_edge_rec(O, s & 0x7fffffff, *reinterpret_cast<const float4 *>(&er), prim ? pv : av,
                    p.sqdt);
  }
  L.x = s < 0 ? L.len : 0.0f;
  const float mu = L.drift(G, L.x);
  const float xn = fmaf(L.sig * L.sq, z, C::ZD ? L.x : fmaf(mu, L.dtr, L.x));
  if (xn > 0.0f && xn < L.len) {
    L.x = xn;
    return true;
  }
  L.pz = z;  // zero-time re-hit: pending from the vertex x
  L.steps_left = -L.steps_left;
  return false;
}

// PEND: the lane may carry an unresolved hit (ensembles; trials never do)
template <class C, bool PEND = true>
__device__ __forceinline__ bool rare_trip(Lane<C> &L, const NativeGraph &G,
                                          const Tables<C::SMEM> &T, const Occ &O,
                                          const NatParams &p, float z, uint32_t u) {
  if constexpr (C::STAR)
    return rare_star<C, PEND>(L, G, T, O, p, z, u);
  else
    return rare_general<C, PEND>(L, G, T, O, p, z, u);
}

// One trip for every lane of the warp: lanes with steps left advance; returns
// true for lanes whose macro step completed.
//
// Common path: a lane strictly inside its edge always begins a fresh macro
// step (dtr == dt), so the proposal uses cached constants.  Accepted: done
// (the star mirror wall reflects in place, kernels.py:185-188).  Overshoot
// at an end: the hit is recorded with predicated moves (general: x = the
// vertex, start point and Gaussian saved; star: x = -start point, Gaussian
// saved) and its split time is solved by the lane's next
// vertex trip, so all vertex work is one divergent region.  That region is
// compiled only into the vertex-slot trip (SLOT), the first trip of every
// Q-trip iteration; lanes at a vertex wait for it, so the warp resolves its
// vertices together.
template <class C, bool SLOT>
__device__ __forceinline__ bool trip(Lane<C> &L, const NativeGraph &G,
                                     const Tables<C::SMEM> &T, const Shared &S, const Occ &O,
                                     const NatParams &p, float z, uint32_t u) {
  // star: live lanes with x <= 0 sit at the vertex (x = -start: a pending hit);
  // general: steps_left > 0 <=> strictly inside the edge (at-vertex lanes carry
  // steps_left < 0), so the common path tests one integer
  constexpr bool XSIGN = C::STAR && !GSDE_STAR_NEG;  // (the round-1 star encoding)
  const bool live = L.steps_left > 0;
  const bool run = XSIGN ? live && (L.x > 0.0f) : live;
  const bool vtx = XSIGN ? live && !run : L.steps_left < 0;  // (before this trip's hit)
  if constexpr (C::INJ)  // one injected normal per proposal
    z = run ? L.inj_gauss() : 0.0f;
  float xn = fmaf(L.sig_sqdt, z, C::ZD ? L.x : fmaf(L.drift(G, L.x), p.dt, L.x));
  const bool lo_ok = xn > 0.0f;
  const bool ok = run && lo_ok && (C::STAR || xn < L.len);
  const bool hit = run && !ok;
  if (C::REFLECT && xn > L.len) xn = fmaxf(2.0f * L.len - xn, 0.0f);
  if (hit) {
    L.pz = z;
    if (XSIGN)  // the flag and start point in x's sign
      L.x = -L.x;
    else  // the flag in the step count's sign, x stays the start
      L.steps_left = -L.steps_left;
  }
  if (ok) {
    L.x = xn;
    L.steps_left -= 1;
  }
  // star mirror wall: a proposal reflected onto the vertex itself (x == 0)
  // starts the next step there (kernels.py:185-188 then :196)
  if (C::REFLECT && !XSIGN && ok && !(xn > 0.0f) && L.steps_left > 0) {
    L.steps_left = -L.steps_left;
    L.pz = __int_as_float(0x7fffffff);
  }
  bool done = ok;
  if (SLOT && vtx) {
    done = rare_trip<C>(L, G, T, O, p, z, u);  // (general: leaves steps_left >= 0 when done)
    if (done) {
      L.step_done(S, p.cap, p.dt, p.sqdt);
      L.steps_left -= 1;  // (general: a step that ended at the vertex leaves it flagged)
    }
  }
  if (C::OCC) L.occ_tick(O, done);
  return done;
}

// Initial state of particle id (kernels.py:291-307, engine.py:194-203): the
// edge and position only.
// PerEdgeUniform from two raw 64-bit draws (kernels.py:298-305)
template <bool SMEM, bool STAR>
__device__ __forceinline__ void place_from_raw(const NativeGraph &G, const Tables<SMEM> &T,
                                               const NatParams &p, uint64_t r0, uint64_t r1,
                                               int &e, float &x) {
  const double u = (double)(r0 >> 11) * kInv2p53;
  const double u2 = (double)(r1 >> 11) * kInv2p53;
  e = (int)(u * (double)G.n_edges);
  if (e >= G.n_edges) e = G.n_edges - 1;
  // (star edges are semi-infinite; their records' x slot holds sig^2 / mu0^2)
  const double le = STAR ? (double)INFINITY : (double)T.E(e).x;
  x = (float)(u2 * (le < p.init_xmax ? le : p.init_xmax));
}

// Particle i of this call: native placement stream, or (Cfg::INJ) the
// reference's draws 0 and 1 of the particle's injected row.
template <class C>
__device__ __forceinline__ void place_values(const NativeGraph &G, const Tables<C::SMEM> &T,
                                             const NatParams &p, const InjParams &q, int64_t i,
                                             int &e, float &x) {
  if (p.init_kind == GSDE_INIT_POINT) {
    e = p.init_edge;
    x = C::STAR ? p.init_x : fminf(p.init_x, T.E(e).x);  // the FP32 edge, like every position
  } else if (C::STATE && p.init_kind == GSDE_INIT_STATE) {
    e = __ldg(q.st_e + i);  // coalesced: a warp refills 32 consecutive ids
    x = __ldg(q.st_x + i);
  } else if constexpr (C::INJ) {
    const uint64_t *r = q.raw + i * q.stride;
    place_from_raw<C::SMEM, C::STAR>(G, T, p, __ldg(r), __ldg(r + 1), e, x);
  } else {
    const Block r = native_block(p, 0u, kDomainPlace, (uint64_t)(p.id_offset + i));
    place_from_raw<C::SMEM, C::STAR>(G, T, p, ((uint64_t)r.x << 32) | r.y, ((uint64_t)r.z << 32) | r.w,
                            e, x);
  }
}

template <class C>
__device__ __forceinline__ void start_particle(Lane<C> &L, const Tables<C::SMEM> &T,
                                               const Occ &O, const NatParams &p, int e, float x,
                                               float star_len) {
  L.load_edge(T, O, e, p.sqdt, star_len);
  L.x = x;
  L.dtr = p.dt;
  L.sq = p.sqdt;
  L.M = 0;
  L.trunc = false;
  L.steps_left = p.n_steps;
  if (C::STAR ? GSDE_STAR_NEG && !(x > 0.0f) : !(x > 0.0f && x < L.len)) {  // at a vertex (trip)
    L.steps_left = -p.n_steps;
    L.pz = __int_as_float(0x7fffffff);
  }
  L.cross = L.events = L.truncs = 0;
  L.occ_left = O.start + O.every;
}

template <class C>
__device__ __forceinline__ void place_native(Lane<C> &L, const NativeGraph &G,
                                             const Tables<C::SMEM> &T, const Occ &O,
                                             const NatParams &p, const InjParams &q, uint64_t id,
                                             float star_len) {
  int e;
  float x;
  place_values<C>(G, T, p, q, (int64_t)(id - (uint64_t)p.id_offset), e, x);
  start_particle<C>(L, T, O, p, e, x, star_len);
}

// Per-warp shared queues of the ensemble kernel (64-entry rings):
//  * placements: particle index, edge and position of the next particles,
//    filled 32 at a time in one converged pass (one atomic, 32 Philox blocks
//    and 32 edge-record loads in flight together);
//  * finished states: edge and position awaiting the fused estimators --
//    and, in per-particle kernels, the particle's index and counters
//    awaiting its output stores -- handled 32 at a time in one converged
//    pass (the dependent grid loads / stores of 32 particles in flight
//    together; a store pass per finishing lane ran at ~1 active lane).
constexpr int kRing = 64;
template <class Cnt>
struct WarpQueues {
  long long *pid;
  int *pe;
  float *px;
  int *fe;
  float *fx;
  long long *fi;      // per-particle kernels: finished particle index
  Cnt *fc, *fv, *ft;  //   and its crossings / events / truncations
};
template <class C>
__host__ __device__ constexpr size_t queue_bytes_per_warp() {
  return kRing * (sizeof(long long) + 2 * sizeof(int) + 2 * sizeof(float) +
                  (C::PP ? sizeof(long long) + 3 * sizeof(typename C::Cnt) : 0));
}

// Random words of one Q-trip iteration with SLOTS vertex slots (trips
// k Q / SLOTS): word 0 = slot 0's exit uniform, words 1..Q = Box-Muller
// inputs of the Q Gaussians, word 4 NB - k = slot k's uniform (k >= 1).
// Philox blocks (counter: per-particle block index, domain, particle id) are
// generated as the trips need them; every helper below folds to a constant
// once the trip loop is unrolled.
template <int Q, int SLOTS>
struct IterWords {
  static constexpr int NB = (Q + SLOTS + 3) / 4;  // blocks per iteration
  static_assert(Q % 2 == 0, "Gaussians come in Box-Muller pairs");
  static_assert(SLOTS >= 1 && SLOTS <= 4 && Q % SLOTS == 0, "slots split the iteration evenly");
  __host__ __device__ static constexpr bool is_slot(int t) { return t % (Q / SLOTS) == 0; }
  __host__ __device__ static constexpr int uword(int t) {  // uniform word of slot trip t
    return t == 0 ? 0 : 4 * NB - t / (Q / SLOTS);
  }
  // bit b set: block b is read by some trip of the pairs 0..j
  __host__ __device__ static constexpr unsigned need(int j) {
    unsigned m = 0;
    for (int jj = 0; jj <= j; jj += 2) {
      m |= (1u << ((1 + jj) / 4)) | (1u << ((2 + jj) / 4));
      if (is_slot(jj)) m |= 1u << (uword(jj) / 4);
      if (is_slot(jj + 1)) m |= 1u << (uword(jj + 1) / 4);
    }
    return m;
  }
};

// Star graphs: 3 blocks / SM (up to 85 registers, no spills, more ILP per
// warp) measured +4% over 4 blocks / 64 registers; general graphs keep 4.
template <class C, int Q, int SLOTS>
__global__ void __launch_bounds__(kThreads, C::STAR ? kMinBlocksStar : kMinBlocks)
    native_ensemble_kernel(NativeGraph G, NatParams p, KOut o, int occ_smem_cells,
                           unsigned long long *work, unsigned queue_off,
                           unsigned occ_tab_off, InjParams q) {
  using IW = IterWords<Q, SLOTS>;
  constexpr int NB = IW::NB;
  const int nb = p.cap + 1;
  Shared S;
  Tables<C::SMEM> T;
  shared_setup<C::STAR, C::SMEM, C::FULL>(G, nb, o.m_hist, S, T, false,
                                          C::OCC ? occ_smem_cells : 0, p.mh_smem);
  Occ O{o.hist_offsets, o.hist_counts, o.hist_dx, o.occ, S.occ, (int32_t)o.occ_every,
        (int32_t)o.occ_start, nullptr};
  if (C::OCC && G.n_edges <= kOccTabEdges) {
    extern __shared__ __align__(16) unsigned char smem_t[];
    float4 *tab = reinterpret_cast<float4 *>(smem_t + occ_tab_off);
    for (int j = threadIdx.x; j < G.n_edges; j += blockDim.x)
      tab[j] = make_float4(__int_as_float((int)o.hist_offsets[j]),
                           __int_as_float((int)o.hist_counts[j] - 1),
                           (float)(1.0 / o.hist_dx[j]), 0.0f);
    __syncthreads();
    O.tab = tab;
  }
  const float star_len = C::REFLECT ? p.reflect : __int_as_float(0x7f800000);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Lane<C> L;
  L.x = 1.0f;
  L.e = 0;  // idle lanes still evaluate the predicated per-trip code: keep indices valid
  L.ev = make_int4(0, 0, 0, 0);
  L.len = star_len;
  L.mu_a = L.mu_b = L.sig = L.sig_sqdt = 0.0f;
  L.M = 0;
  L.steps_left = 0;  // no particle in flight: every trip is a no-op
  L.occ_left = 1 << 30;
  // Per-particle Philox block index: 32 bits in the counter's first word.
  // FULL kernels (runs that could pass 2^32 blocks per particle) carry the
  // wrap into bits 48.. of the stream-id word -- particle ids stay below 2^48
  // (checked by the host) -- so streams never repeat.
  uint32_t blk = 0;
  static_assert(!C::FULL || (NB & (NB - 1)) == 0,
                "2^32 must be a multiple of the blocks per iteration");
  uint64_t id = 0;
  int64_t t_cross = 0, t_events = 0, t_truncs = 0, t_over = 0;
  bool waiting = i < p.n;  // next particle not started yet
  bool active = false;     // a particle is in flight
  bool need = false;       // finished: fetch the next particle id
  bool queued = false;     // this lane's finished state awaits binning

  auto finish = [&]() {
    if constexpr (C::PP) {
      if (!C::HT) {
        t_cross += L.cross;
        t_events += L.events;
        t_truncs += L.truncs;
      }
    }
    if (C::INJ) t_over += L.over ? 1 : 0;
    if (C::STATE && q.counter)  // next block (NATIVE: carry in id's bits 48..) / draws used (INJ)
      q.counter[i] = C::INJ ? (uint64_t)L.k : ((id >> 48) << 32) | blk;
    queued = true;
    active = false;
    need = true;
  };

  // Placement only (engine.py:329-336): every particle placed and binned once
  // here; the host starts the particle counter past every id (launch below),
  // so the hand-out loop that follows starts nothing.
  if (p.n_steps == 0) {
    while (waiting) {
      id = (uint64_t)(p.id_offset + i);
      place_native(L, G, T, O, p, q, id, star_len);
      if constexpr (C::PP) {
        epilogue_particle(o, i, L.e, (double)L.x, 0, 0, 0);
        if (q.progress) publish_particle(q, i);
      }
      epilogue_bins(o, L.e, (double)L.x);
      i += stride;
      waiting = i < p.n;
    }
    L.steps_left = 0;
  }

  // Particles come from a grid-wide counter, 32 per warp refill, so warps the
  // schedulers favour take more particles and the SMs stay full until the end
  // (results are per particle id and integer sums: assignment-invariant).
  // Particles start on iteration boundaries, so the lanes of a warp share
  // their vertex slot.
  const int lane = threadIdx.x & 31;
  extern __shared__ __align__(16) unsigned char smem_q[];
  WarpQueues<typename C::Cnt> WQ;
  {
    unsigned char *q = smem_q + queue_off + (threadIdx.x >> 5) * queue_bytes_per_warp<C>();
    WQ.pid = reinterpret_cast<long long *>(q);
    WQ.pe = reinterpret_cast<int *>(q + kRing * sizeof(long long));
    WQ.px = reinterpret_cast<float *>(q + kRing * (sizeof(long long) + sizeof(int)));
    WQ.fe = reinterpret_cast<int *>(q + kRing * (sizeof(long long) + sizeof(int) + sizeof(float)));
    WQ.fx = reinterpret_cast<float *>(q + kRing * (sizeof(long long) + 2 * sizeof(int) + sizeof(float)));
    if constexpr (C::PP) {
      unsigned char *r = q + kRing * (sizeof(long long) + 2 * sizeof(int) + 2 * sizeof(float));
      WQ.fi = reinterpret_cast<long long *>(r);
      WQ.fc = reinterpret_cast<typename C::Cnt *>(r + kRing * sizeof(long long));
      WQ.fv = WQ.fc + kRing;
      WQ.ft = WQ.fv + kRing;
    }
  }
  uint32_t q_head = 0, q_tail = 0;  // placement ring (warp-uniform)
  int f_n = 0;                      // finished states queued (warp-uniform)
  const bool bins = o.edge_counts || o.hist;
  // shared-memory estimator counters (when the grid fits): the warp's 32
  // finished states are grouped by edge / cell with __match_any_sync, and
  // one lane per group adds the group's size -- one shared atomic per
  // distinct bin per 32 particles; flushed to global int64 once per block
  // (the counters' address is re-derived from the parameter at each use: a
  // pointer held across the stepping loop costs the loop registers)
  extern __shared__ __align__(16) unsigned char smem_b[];
  auto bin_base = [&]() { return reinterpret_cast<unsigned *>(smem_b + q.bin_off); };
  // (compiled for graphs staged in shared memory only: a network too large
  // to stage has more bins than fit, and the code would cost its loop)
  const bool sbins = C::SMEM && q.bin_off;
  if (sbins) {
    for (int j = threadIdx.x; j < q.bin_edges + q.bin_cells; j += blockDim.x) bin_base()[j] = 0u;
    __syncthreads();
  }
  auto flush_bins = [&](int n_take) {  // converged: bin entries 0..n_take-1
    const bool mine = lane < n_take;
    if (sbins) {
      unsigned *s_ec = bin_base(), *s_h = s_ec + q.bin_edges;
      const int e = mine ? WQ.fe[lane] : -1;
      if (o.edge_counts) {
        const unsigned grp = __match_any_sync(0xffffffffu, e);
        if (mine && lane == __ffs(grp) - 1) atomicAdd(&s_ec[e], (unsigned)__popc(grp));
      }
      if (o.hist) {
        const int c = mine ? (int)hist_cell(o.hist_offsets, o.hist_counts, o.hist_dx, e,
                                            (double)WQ.fx[lane])
                           : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, c);
        if (mine && lane == __ffs(grp) - 1) atomicAdd(&s_h[c], (unsigned)__popc(grp));
      }
    } else if (bins && mine) {
      epilogue_bins(o, WQ.fe[lane], (double)WQ.fx[lane]);
    }
    if constexpr (C::PP) {
      // the per-particle outputs, one particle per lane; then, for streamed
      // results, one GPU-scope fence for the warp and one relaxed add per
      // distinct progress range (a release add per particle stalled each
      // finishing warp on its own fence: +7% kernel time on C1)
      const long long fi = mine ? WQ.fi[lane] : 0;
      if (mine)
        epilogue_particle(o, fi, WQ.fe[lane], (double)WQ.fx[lane], WQ.fc[lane], WQ.fv[lane],
                          WQ.ft[lane]);
      if (q.progress) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncwarp();
        const int r = mine ? (int)((q.progress_base + fi) >> q.progress_shift) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, r);
        if (mine && lane == __ffs(grp) - 1) atomicAdd(q.progress + r, (unsigned)__popc(grp));
      }
    }
    __syncwarp();
    if (lane < f_n - n_take) {  // n_take == 32: sources and targets do not overlap
      WQ.fe[lane] = WQ.fe[n_take + lane];
      WQ.fx[lane] = WQ.fx[n_take + lane];
      if constexpr (C::PP) {
        WQ.fi[lane] = WQ.fi[n_take + lane];
        WQ.fc[lane] = WQ.fc[n_take + lane];
        WQ.fv[lane] = WQ.fv[n_take + lane];
        WQ.ft[lane] = WQ.ft[n_take + lane];
      }
    }
    __syncwarp();
    f_n -= n_take;
  };
  need = true;
  waiting = false;
  for (;;) {
    const unsigned nm = __ballot_sync(0xffffffffu, need);  // finished lanes (+ the start)
    if (nm) {
      if (C::PP || bins) {  // queue the finished states (i, L: still the old particle); 32 at a time
        const unsigned qm = __ballot_sync(0xffffffffu, queued);
        if (queued) {
          const int slot = f_n + __popc(qm & ((1u << lane) - 1u));
          WQ.fe[slot] = L.e;
          WQ.fx[slot] = L.x;
          if constexpr (C::PP) {
            WQ.fi[slot] = i;
            WQ.fc[slot] = L.cross;
            WQ.fv[slot] = L.events;
            WQ.ft[slot] = L.truncs;
          }
          queued = false;
        }
        f_n += __popc(qm);
        __syncwarp();
        if (!C::PP && f_n >= 32) flush_bins(32);
      }
      const int k = __popc(nm);
      if (q_tail - q_head < (uint32_t)k) {  // refill 32 placements
        unsigned long long base = 0;
        // (a warp past its budget -- q_tail counts the particles it took --
        // takes nothing more)
        if (lane == 0)
          base = (p.warp_budget == 0u || q_tail < p.warp_budget) ? atomicAdd(work, 32ull)
                                                                 : (unsigned long long)p.n;
        base = __shfl_sync(0xffffffffu, base, 0);
        const int64_t pi = (int64_t)base + lane;
        int e = 0;
        float x = 0.0f;
        if (pi < p.n) place_values<C>(G, T, p, q, pi, e, x);
        const int slot = (int)((q_tail + lane) & (kRing - 1));
        WQ.pid[slot] = pi;
        WQ.pe[slot] = e;
        WQ.px[slot] = x;
        q_tail += 32;
        __syncwarp();
      }
      if (need) {
        const int slot = (int)((q_head + __popc(nm & ((1u << lane) - 1u))) & (kRing - 1));
        i = WQ.pid[slot];
        waiting = i < p.n;
        if (waiting) {
          id = (uint64_t)(p.id_offset + i);
          start_particle<C>(L, T, O, p, WQ.pe[slot], WQ.px[slot], star_len);
          if constexpr (C::INJ) {
            L.thr = q.thresh;
            L.ved = q.vedges;
            L.vor = q.vorient;
            L.ir = q.raw + i * q.stride;
            L.inn = q.normal + i * q.stride;
            // PerEdgeUniform placement used the row's draws 0 and 1
            L.k = p.init_kind == GSDE_INIT_PER_EDGE_UNIFORM ? 2 : 0;
            L.kmax = (int)q.stride;
            L.over = false;
          }
          blk = 0;
          if (C::STATE && p.init_kind == GSDE_INIT_STATE && q.st_k) {  // resume: next block
            const uint64_t k0 = __ldg(q.st_k + i);
            blk = (uint32_t)k0;
            id += (k0 >> 32) << 48;
          }
          waiting = false;
          active = true;
        }
        need = false;
      }
      q_head += k;
      __syncwarp();
      // per-particle kernels flush here, after the refill (one call site);
      // out of work (idle lanes): store / publish what is queued now -- the
      // run's last particles would otherwise wait for the warp's exit
      if constexpr (C::PP) {
        const int t = f_n >= 32 ? 32 : (f_n > 0 && !__all_sync(0xffffffffu, active) ? f_n : 0);
        if (t > 0) flush_bins(t);
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
    uint32_t W[4 * NB];
    auto fill = [&](int kb) {
      const Block r = native_block(p, blk + (uint32_t)kb, kDomainEnsemble, id);
      W[4 * kb] = r.x;
      W[4 * kb + 1] = r.y;
      W[4 * kb + 2] = r.z;
      W[4 * kb + 3] = r.w;
    };
#pragma unroll
    for (int j = 0; j < Q; j += 2) {
      const unsigned fresh = IW::need(j) & ~(j ? IW::need(j - 2) : 0u);
      float z0 = 0.0f, z1 = 0.0f;
      if constexpr (!C::INJ) {  // (injected draws are taken per use inside the trips)
#pragma unroll
        for (int kb = 0; kb < NB; ++kb)
          if (fresh & (1u << kb)) fill(kb);
        box_muller(W[1 + j], W[2 + j], z0, z1);
      } else {
        for (int kb = 0; kb < 4 * NB; ++kb) W[kb] = 0u;
      }
      if (IW::is_slot(j))
        trip<C, true>(L, G, T, S, O, p, z0, W[IW::uword(j)]);
      else
        trip<C, false>(L, G, T, S, O, p, z0, 0u);
      if (IW::is_slot(j + 1))
        trip<C, true>(L, G, T, S, O, p, z1, W[IW::uword(j + 1)]);
      else
        trip<C, false>(L, G, T, S, O, p, z1, 0u);
    }
    blk += NB;
    if (C::FULL && blk == 0u) id += 1ull << 48;
    if (active && L.steps_left == 0) finish();
  }
  if ((C::PP || bins) && f_n > 0) flush_bins(f_n);
  if (sbins) {
    const unsigned *s_ec = bin_base(), *s_h = s_ec + q.bin_edges;
    __syncthreads();
    for (int j = threadIdx.x; j < q.bin_edges; j += blockDim.x)
      if (s_ec[j] && o.edge_counts) add_i64(&o.edge_counts[j], (int64_t)s_ec[j]);
    for (int j = threadIdx.x; j < q.bin_cells; j += blockDim.x)
      if (s_h[j] && o.hist) add_i64(&o.hist[j], (int64_t)s_h[j]);
  }
  if (o.totals && !C::HT) {
    warp_add_i64(&o.totals[0], t_cross);
    warp_add_i64(&o.totals[1], t_events);
    warp_add_i64(&o.totals[2], t_truncs);
    if (C::INJ) warp_add_i64(&o.totals[3], t_over);
  }
  shared_flush<C::FULL, C::HT>(S, nb, o.m_hist, C::OCC ? occ_smem_cells : 0, o.occ,
                               o.totals);
}

// Vertex trials: one macro step per trial from the vertex (kernels.py:447-521),
// fused exit counts per edge and M histogram including M = 0.
template <class C, bool OUT>
__global__ void __launch_bounds__(kThreads, kMinBlocksTrials)
    native_trials_kernel(NativeGraph G, NatParams p, gsde_trials_out o, int exit_cnt,
                         InjParams q) {
  // HT: run totals from the M histogram (every trial lands in bin M <= cap)
  // and a shared truncation counter, as in the lean ensemble kernel -- off:
  // per-lane sums measured 2% faster here (the lane's registers are free)
  constexpr bool HT = false;
  const int nb = p.cap + 1;
  Shared S;
  Tables<C::SMEM> T;
  shared_setup<C::STAR, C::SMEM, C::FULL>(G, nb, o.m_hist, S, T, exit_cnt != 0, 0, p.mh_smem);
  const Occ O{};
  const float inf = __int_as_float(0x7f800000);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool active = i < p.n;
  Lane<C> L;
  uint32_t pair = 0;
  uint64_t id = 0;
  // per-lane sums: trials per lane x cap < 2^31 unless the host chose FULL
  typename C::Cnt t_M = 0;
  int32_t t_ev = 0, t_tr = 0, t_over = 0;
  // the fused estimator (no per-trial arrays, native draws) walks its trials
  // by stream id alone: one 64-bit add and compare per trial
  constexpr bool BY_ID = !OUT && !C::INJ;
  const uint64_t id_end = (uint64_t)(p.id_offset + p.n);
  auto start = [&]() {
    if (!BY_ID) id = (uint64_t)(p.id_offset + i);
    // (star: every trial's first trip picks its exit edge, which loads that
    // edge's record, so the start needs none; general: the start edge's
    // endpoint record names the vertex's slots)
    if (!C::STAR) L.load_edge(T, O, p.start_edge, p.sqdt, inf);
    L.x = C::STAR ? 0.0f : p.start_x;
    L.dtr = p.dt;
    L.sq = p.sqdt;
    L.M = 0;
    L.trunc = false;
    L.steps_left = 1;  // (general: the sign carries a pending re-hit)
    pair = 0;
    if constexpr (C::INJ) {  // the trial's own injected row, from draw 0
      L.thr = q.thresh;
      L.ved = q.vedges;
      L.vor = q.vorient;
      L.ir = q.raw + i * q.stride;
      L.inn = q.normal + i * q.stride;
      L.k = 0;
      L.kmax = (int)q.stride;
      L.over = false;
    }
  };
  auto finish = [&]() {
    if (C::INJ) t_over += L.over ? 1 : 0;
    if (OUT) {  // per-trial arrays (vertex_crossing_trials); the fused estimator skips them
      if (o.M) o.M[i] = L.M;
      if (o.edge) o.edge[i] = L.e;
      if (o.x) o.x[i] = (double)L.x;
      if (o.trunc) o.trunc[i] = L.trunc ? 1 : 0;
    }
    if (S.exit_cnt) {
#if GSDE_EXIT_PRIV
      S.exit_cnt[L.e * kThreads + threadIdx.x] += 1;
#else
      atomicAdd(&S.exit_cnt[L.e], 1u);
#endif
    }
    else if (o.exit_counts)
      add_i64(&o.exit_counts[L.e], 1);
    mh_add<C::FULL>(S, L.M > p.cap ? p.cap : L.M);
    if constexpr (HT) {
      if (L.trunc) atomicAdd(reinterpret_cast<unsigned *>(&S.tot[2]), 1u);
    } else {
      t_M += L.M;
      t_ev += L.M > 0 ? 1 : 0;
      t_tr += L.trunc ? 1 : 0;
    }
    if constexpr (BY_ID) {
      id += (uint64_t)stride;
      active = id < id_end;
    } else {
      i += stride;
      active = i < p.n;
    }
    if (active) start();
  };
  L.x = 1.0f;
  L.e = 0;
  L.ev = make_int4(0, 0, 0, 0);
  L.len = inf;
  L.mu_a = L.mu_b = L.sig = L.sig_sqdt = 0.0f;
  if (BY_ID) id = (uint64_t)(p.id_offset + i);
  if (active) start();
  // a trial is one macro step started at the vertex: every trip is a vertex
  // trip, so the rare-path step functions run directly
  while (__any_sync(0xffffffffu, active)) {
    Block r{0u, 0u, 0u, 0u};
    float z0 = 0.0f, z1 = 0.0f;
    if constexpr (!C::INJ) {  // (injected draws are taken per use inside the trips)
      r = native_block(p, pair++, kDomainTrials, id);
      box_muller(r.x, r.y, z0, z1);
    }
    bool fin = false;
    if (active) fin = rare_trip<C, false>(L, G, T, O, p, z0, r.z);
    if (active && !fin) fin = rare_trip<C, false>(L, G, T, O, p, z1, r.w);
    if (fin) finish();
  }
  if (o.totals && !HT) {
    warp_add_i64(&o.totals[0], t_M);
    warp_add_i64(&o.totals[1], t_ev);
    warp_add_i64(&o.totals[2], t_tr);
    if (C::INJ) warp_add_i64(&o.totals[3], t_over);
  }
  shared_flush<C::FULL, HT>(S, nb, o.m_hist, 0, nullptr, o.totals);
  if (S.exit_cnt && o.exit_counts)
    for (int e = threadIdx.x; e < G.n_edges; e += blockDim.x) {
#if GSDE_EXIT_PRIV
      int64_t v = 0;
      for (int t = 0; t < kThreads; ++t) v += S.exit_cnt[e * kThreads + t];
      if (v) add_i64(&o.exit_counts[e], v);
#else
      if (S.exit_cnt[e]) add_i64(&o.exit_counts[e], (int64_t)S.exit_cnt[e]);
#endif
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

constexpr int kOccSmemCells = 8192;  // shared uint32 occupation counters up to 32 KB
constexpr int kBinSmemMax = 4096;    // shared uint32 final-state bins (edges + cells) up to 16 KB

size_t smem_bytes(const gsde_graph *g, int nb, bool stage, bool exit_cnt, int occ_cells) {
  size_t b = ((size_t)smem_bins(nb) * sizeof(int) + 15) & ~size_t(15);
  b += 4 * sizeof(unsigned long long);
  if (stage) b += (size_t)g->E * (g->is_star ? 16 : 32) + (size_t)g->S * 16;
  if (exit_cnt) b += align16((size_t)g->E * (GSDE_EXIT_PRIV ? kThreads : 1) * sizeof(unsigned));
  b += (size_t)occ_cells * sizeof(unsigned);
  return b;
}

template <class K>
int occupancy_grid(K kernel, size_t smem, int device, int64_t n_items, int waves = 1,
                   int max_per_sm = 1 << 30) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  if (per_sm > max_per_sm) per_sm = max_per_sm;
  if (per_sm < 1) per_sm = 1;
  const int64_t full = (int64_t)dev_info(device).sm_count * per_sm * waves;
  const int64_t need = (n_items + kThreads - 1) / kThreads;
  return (int)(need < full ? (need < 1 ? 1 : need) : full);
}

// Testing knob (tests/test_gpu_robustness.py): GSDE_FORCE_GLOBAL_BINS=1 takes
// the path of runs too large for 32-bit shared counters at any size.
bool force_global_bins() {
  static const bool f = std::getenv("GSDE_FORCE_GLOBAL_BINS") != nullptr;
  return f;
}
// Testing knob: GSDE_GENERIC_DRIFT=1 runs constant-drift graphs through the
// generic affine-drift kernel (the constant-drift variant must match it bit
// for bit: tests/test_gpu_robustness.py).
bool generic_drift() {
  static const bool f = std::getenv("GSDE_GENERIC_DRIFT") != nullptr;
  return f;
}
// Testing knob: GSDE_GENERIC_EXITS=1 picks exits through the alias columns even
// where every column keeps its own slot (the uniform-exit variant must match).
bool generic_exits() {
  static const bool f = std::getenv("GSDE_GENERIC_EXITS") != nullptr;
  return f;
}

NatParams make_params(uint64_t seed, int64_t n, int64_t off, double dt, int32_t cap) {
  NatParams p{};
  p.seed = seed;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r, k0 += kPhiloxW0, k1 += kPhiloxW1) {
    p.rk[2 * r] = k0;
    p.rk[2 * r + 1] = k1;
  }
  p.n = n;
  p.id_offset = off;
  p.cap = cap;
  p.dt = (float)dt;
  p.sqdt = sqrtf((float)dt);
  p.mh_smem = kMaxSmemBins;
  p.warp_budget = 0u;
  return p;
}

template <class K, class... Args>
cudaError_t launch(K kernel, size_t smem, int grid, cudaStream_t s, Args... args) {
  kernel<<<grid, kThreads, smem, s>>>(args...);
  count_launch();
  return cudaGetLastError();
}

template <class K>
cudaError_t prepare(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Runtime flags -> compile-time kernel variant (Cfg).
// ENS: ensemble launches (the lean, no-per-particle-counter kernels exist only there)
template <bool OCC, bool ENS = false, class F>
cudaError_t dispatch(bool star, bool smem, bool tab, bool zd, bool reflect, F &&f,
                     bool inj = false, bool full = false, bool pp = true, bool cd = false,
                     bool uni = false) {
  using T = std::true_type;
  using N = std::false_type;
  auto with = [&](auto st, auto sm) -> cudaError_t {
    constexpr bool ST = decltype(st)::value, SM = decltype(sm)::value;
    auto drift = [&](auto rf) -> cudaError_t {
      constexpr bool RF = decltype(rf)::value;
      // drift kind: tabulated / zero / constant (general-graph ensembles) / affine
      auto mk = [&](auto inj_t, auto full_t, auto pp_t) -> cudaError_t {
        constexpr bool I = decltype(inj_t)::value, FU = decltype(full_t)::value,
                       P = decltype(pp_t)::value;
        if (tab) return f(Cfg<ST, SM, true, RF, OCC, false, I, FU, P>{});
        if (zd) return f(Cfg<ST, SM, false, RF, OCC, true, I, FU, P>{});
        if constexpr (ENS && !ST)
          if (cd) return f(Cfg<ST, SM, false, RF, OCC, false, I, FU, P, true>{});
        return f(Cfg<ST, SM, false, RF, OCC, false, I, FU, P>{});
      };
      // uniform exits (general-graph native ensembles): same drift kinds
      auto mku = [&](auto inj_t, auto full_t, auto pp_t) -> cudaError_t {
        constexpr bool I = decltype(inj_t)::value, FU = decltype(full_t)::value,
                       P = decltype(pp_t)::value;
        // (general-graph ensembles and vertex trials; star ensembles only with
        // GSDE_STAR_UNI: measured -0.7% on C1, 23.46 -> 23.63 ms)
        if constexpr (!I && (ENS ? (!ST || GSDE_STAR_UNI) : ST)) {
          if (uni) {
            if (tab) return f(Cfg<ST, SM, true, RF, OCC, false, I, FU, P, false, true>{});
            if (zd) return f(Cfg<ST, SM, false, RF, OCC, true, I, FU, P, false, true>{});
            if (cd) return f(Cfg<ST, SM, false, RF, OCC, false, I, FU, P, true, true>{});
            return f(Cfg<ST, SM, false, RF, OCC, false, I, FU, P, false, true>{});
          }
        }
        return mk(inj_t, full_t, pp_t);
      };
      if (inj) {  // parity mode: no occupation sampling; state-in, counter, 32-bit counts
        if constexpr (!OCC) return mk(T{}, N{}, T{});
        return cudaErrorInvalidValue;
      }
      if (full) return mku(N{}, T{}, T{});
      if constexpr (ENS)
        if (!pp) return mku(N{}, N{}, N{});  // lean: fused estimators only
      return mku(N{}, N{}, T{});
    };
    if constexpr (ST)
      if (reflect) return drift(T{});
    return drift(N{});
  };
  if (star) return smem ? with(T{}, T{}) : with(T{}, N{});
  return smem ? with(N{}, T{}) : with(N{}, N{});
}

// Ensembles take the FULL kernel for state-in / counter output, or when a
// 32-bit per-lane count, the shared M histogram or the Philox block index
// could overflow: per particle at most n_steps x cap crossings, and at most
// (cap + 2) iterations (4 blocks each) per step.
bool ensemble_needs_full(const gsde_run &a, const gsde_out &o) {
  const double steps = (double)a.n_steps, cap = (double)a.cap;
  return a.init_kind == GSDE_INIT_STATE || o.counter != nullptr ||
         a.cap + 1 > kMaxSmemBins || steps * cap >= 2147483647.0 ||
         4.0 * steps * (cap + 2.0) >= 4294967296.0;
}

}  // namespace

namespace {
cudaError_t launch_native_ensemble_one(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                       cudaStream_t s) {
  NatParams p = make_params(a.seed, a.n_particles, a.pid_offset, a.dt, a.cap);
  p.n_steps = (int32_t)a.n_steps;
  p.reflect = (float)a.reflect_len;
  p.init_kind = a.init_kind;
  p.init_edge = (int32_t)a.init_edge;
  p.init_x = (float)a.init_x;
  p.init_xmax = a.init_xmax;
  const bool inj = a.stream == GSDE_STREAM_INJECT;  // (precision GSDE_PREC_NATIVE)
  InjParams q{a.inj_raw,         a.inj_normal,       a.inj_stride,
              g->ref32.v_thresh, g->ref32.v_edges,   g->ref32.v_orient,
              a.state_edge,      a.state_x,          a.state_counter,
              o.counter};
  q.progress = o.progress;
  q.progress_base = o.progress_base;
  q.progress_shift = o.progress_shift;
  const bool stage = g->nat_graph_smem > 0;
  const bool occ = o.occ != nullptr;
  const int d = g->device;
  const int64_t n = a.n_particles;
  // Shared 32-bit counters (M histogram, occupation, final-state bins) stay
  // exact: each warp takes at most 4 x its fair share of particles + 64 (the
  // kernel's warp_budget and its last refill), which bounds what one block
  // can count -- steps x that for the M histogram / occupation, that for the
  // final-state bins.  Runs past 2^32 keep those counters in global memory
  // (FULL kernel, no shared M bins).  (grid >= min(SMs, ceil(n / 256)))
  const double share = 8.0 * (std::max(256.0, 4.0 * std::ceil((double)n / (8.0 * dev_info(d).sm_count))) + 64.0);
  const bool big_steps = share * (double)std::max<int64_t>(a.n_steps, 1) >= 4294967295.0 ||
                         force_global_bins();
  const bool big_parts = share >= 4294967295.0 || force_global_bins();
  p.mh_smem = big_steps ? 0 : kMaxSmemBins;
  auto run = [&](auto cfg) -> cudaError_t {
    using C = decltype(cfg);
    // 14-trip iterations; one vertex slot on star graphs (rare, short vertex
    // visits), two on general graphs (a zero-time re-hit makes a lane wait for
    // the next slot).  Measured: (10,1) / (14,1) / (18,1) /
    // (22,1) on star3, (10,2) / (14,2) / (22,2) / (12,3) / (18,3) / (16,4)
    // on hub64 and vascular.
#ifndef GSDE_GQ
#define GSDE_GQ 14
#define GSDE_GS 2
#endif
    constexpr int kSlots = C::STAR ? 1 : ((C::FULL || C::INJ) ? 2 : GSDE_GS);
    constexpr int kQ = C::STAR ? kTrips : ((C::FULL || C::INJ) ? kTrips : GSDE_GQ);
    auto k = native_ensemble_kernel<C, kQ, kSlots>;
    // occupation counters in shared memory when the grid is small (shared
    // counters carry into the int64 arrays, so no run length overflows them)
    int occ_cells = 0;
    if (C::OCC && o.hist_n_cells <= kOccSmemCells) occ_cells = (int)o.hist_n_cells;
    const size_t queues = (kThreads / 32) * queue_bytes_per_warp<C>();
    const size_t occ_tab = (C::OCC && g->E <= kOccTabEdges) ? (size_t)g->E * sizeof(float4) : 0;
    size_t smem = align16(smem_bytes(g, a.cap + 1, stage, false, occ_cells)) + queues + occ_tab;
    cudaError_t err = prepare(k, smem);
    if (err != cudaSuccess) return err;
#ifndef GSDE_STAR_BLOCKS
#define GSDE_STAR_BLOCKS (1 << 30)
#endif
    // (GSDE_STAR_BLOCKS caps star grids per SM for experiments: 3 vs 4 resident
    // blocks of the 61-register driftless star kernel measured -0.3%)
    const int grid = occupancy_grid(k, smem, d, n, 1, C::STAR ? GSDE_STAR_BLOCKS : 1 << 30);
    if (big_steps) occ_cells = 0;
    const size_t qoff = align16(smem_bytes(g, a.cap + 1, stage, false, occ_cells));
    smem = qoff + queues + occ_tab;
    // fused final-state bins in shared memory when they fit
    InjParams qq = q;
    const int bin_e = o.edge_counts ? (int)g->E : 0;
    const int bin_c = o.hist ? (int)o.hist_n_cells : 0;
    if (C::SMEM && (bin_e || bin_c) && (int64_t)bin_e + bin_c <= kBinSmemMax && !big_parts) {
      qq.bin_off = (unsigned)align16(smem);
      qq.bin_edges = bin_e;
      qq.bin_cells = bin_c;
      smem = align16(smem) + (size_t)(bin_e + bin_c) * sizeof(unsigned);
      err = prepare(k, smem);
      if (err != cudaSuccess) return err;
    }
    // grid-wide particle counter: this call's slot of the handle's ring
    // (a per-call cudaMallocAsync here stalled running kernels for up to
    // hundreds of ms when the pool remapped memory).  A slot is reused only
    // after the kernel that last used it finished (its event), so any number
    // of calls may be in flight on any streams.
    gsde_graph *gm = const_cast<gsde_graph *>(g);
    const int slot = gm->next_work_slot();
    unsigned long long *work = gm->work + slot;
    cudaEvent_t &done = gm->work_done[slot];
    if (!done)
      err = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    else
      err = cudaStreamWaitEvent(s, done, 0);
    if (err != cudaSuccess) return err;
    // (placement-only runs: 0x7f7f... -- past every particle id, nothing handed out)
    err = cudaMemsetAsync(work, a.n_steps == 0 ? 0x7f : 0, sizeof(*work), s);
    if (err != cudaSuccess) return err;
    NatParams pk = p;  // a warp's budget: 4 x its fair share (+ one refill of 32)
    const double wb = 4.0 * std::ceil((double)n / ((double)grid * (kThreads / 32))) + 32.0;
    pk.warp_budget = wb < 4.0e9 ? (uint32_t)wb : 0u;
    err = launch(k, smem, grid, s, g->nat, pk, kernel_out(o), occ_cells, work, (unsigned)qoff,
                 (unsigned)(qoff + queues), qq);
    if (err != cudaSuccess) return err;
    return cudaEventRecord(done, s);
  };
  const bool full = ensemble_needs_full(a, o) || big_steps;
  // per-particle counters only when some per-particle array is requested
  const bool pp = o.edge || o.x || o.crossings || o.events || o.truncs;
  return occ ? dispatch<true, true>(g->is_star, stage, g->has_tab, g->zero_drift, p.reflect > 0.0f, run,
                                    inj, full, pp, g->const_drift && !generic_drift(),
                                    g->uniform_exits && !generic_exits())
             : dispatch<false, true>(g->is_star, stage, g->has_tab, g->zero_drift, p.reflect > 0.0f,
                                     run, inj, full, pp, g->const_drift && !generic_drift(),
                                     g->uniform_exits && !generic_exits());
}

}  // namespace

// A call whose particles would let one block count 2^32 events in a shared
// 32-bit counter (launch_native_ensemble_one's bound: per-warp budget x steps)
// runs as consecutive launches over contiguous particle-id chunks small enough
// to keep the shared counters -- results are bit-identical (streams are keyed
// by global id; estimators accumulate) -- instead of taking the FULL kernel's
// global-memory counters, whose same-address atomics would serialise a large
// run.  Only when a single chunk of the minimum size would still overflow
// (n_steps beyond ~1.6e6) does the run fall back to global counters.
// GSDE_CHUNK_PARTICLES=<n> forces chunks of n particles (testing).
cudaError_t launch_native_ensemble(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                   cudaStream_t s) {
  const int64_t n = a.n_particles;
  const double steps = (double)std::max<int64_t>(a.n_steps, 1);
  const double sm8 = 8.0 * dev_info(g->device).sm_count;
  // launch_native_ensemble_one's share(nc) = 8 (max(256, 4 ceil(nc / sm8)) + 64)
  // stays below 2^32 / steps for ceil(nc / sm8) <= lim
  // (share never drops below 8 (256 + 64): chunks help while that x steps fits)
  const double lim = std::floor((4294967295.0 / (8.0 * steps) - 64.0) / 4.0) - 1.0;
  int64_t chunk = 8.0 * (256.0 + 64.0) * steps < 4294967295.0
                      ? (int64_t)std::min(std::max(lim, 1.0) * sm8, 9.0e18)
                      : 0;
  static const char *forced = std::getenv("GSDE_CHUNK_PARTICLES");
  if (forced && std::atoll(forced) > 0) chunk = std::atoll(forced);
  if (chunk <= 0 || n <= chunk) return launch_native_ensemble_one(g, a, o, s);
  for (int64_t off = 0; off < n; off += chunk) {
    gsde_run ac = a;
    ac.n_particles = std::min(chunk, n - off);
    ac.pid_offset = a.pid_offset + off;
    if (ac.inj_raw) ac.inj_raw += off * a.inj_stride;
    if (ac.inj_normal) ac.inj_normal += off * a.inj_stride;
    if (ac.state_edge) ac.state_edge += off;
    if (ac.state_x) ac.state_x += off;
    if (ac.state_counter) ac.state_counter += off;
    gsde_out oc = o;
    if (oc.edge) oc.edge += off;
    if (oc.x) oc.x += off;
    if (oc.crossings) oc.crossings += off;
    if (oc.events) oc.events += off;
    if (oc.truncs) oc.truncs += off;
    if (oc.counter) oc.counter += off;
    oc.progress_base += off;
    const cudaError_t err = launch_native_ensemble_one(g, ac, oc, s);
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

cudaError_t launch_native_trials(const gsde_graph *g, const gsde_trials &a,
                                 const gsde_trials_out &o, cudaStream_t s) {
  NatParams p = make_params(a.seed, a.n_trials, a.trial_offset, a.dt, a.cap);
  p.start_edge = (int32_t)a.start_edge;
  p.start_x = (float)a.start_x;
  // Trials are assigned grid-stride: a block runs at most ceil(n / (grid x
  // 256)) x 256 of them, grid >= min(SMs, ceil(n / 256)).  Past 2^32 the
  // M histogram and exit counts stay in global memory (FULL, no shared bins).
  const double per_block = std::max(256.0, std::ceil((double)a.n_trials /
                                                     (dev_info(g->device).sm_count * 256.0)) * 256.0);
  const bool big = per_block >= 4294967295.0 || force_global_bins();
  if (big) p.mh_smem = 0;
  // exit counts in lane-private shared uint32 counters up to 32 edges (shared
  // atomics: 4096 edges, -0.6%); larger graphs add to the global int64 counts
  const int exit_cnt = (o.exit_counts && g->E <= (GSDE_EXIT_PRIV ? 32 : 4096) && !big) ? 1 : 0;
  const bool stage = g->nat_graph_smem > 0;
  const size_t smem = smem_bytes(g, a.cap + 1, stage, exit_cnt, 0);
  const int d = g->device;
  const int64_t n = a.n_trials;
  const bool inj = a.stream == GSDE_STREAM_INJECT;  // (precision GSDE_PREC_NATIVE)
  const InjParams q{a.inj_raw,        a.inj_normal,       a.inj_stride,
                    g->ref32.v_thresh, g->ref32.v_edges, g->ref32.v_orient};
  const bool out = o.M || o.edge || o.x || o.trunc;
  // FULL when a lane's sum of M (<= its trials x cap; conservatively one
  // block per SM) could pass 2^31 or the M histogram outgrows shared memory
  const double per_lane = std::ceil((double)n / ((double)dev_info(d).sm_count * kThreads));
  const bool full = a.cap + 1 > kMaxSmemBins || per_lane * (double)a.cap >= 2147483647.0 || big;
  return dispatch<false>(g->is_star, stage, g->has_tab, g->zero_drift, false,
                         [&](auto cfg) -> cudaError_t {
    auto k = out ? native_trials_kernel<decltype(cfg), true>
                 : native_trials_kernel<decltype(cfg), false>;
    cudaError_t err = prepare(k, smem);
    if (err != cudaSuccess) return err;
    // four waves of blocks: with one resident wave and a static share per
    // thread, the warp schedulers' favourites finished at about half time and
    // the SMs ran on with ~34 of 48 warps (measured per-warp exit times); later
    // waves refill the slots of early blocks (measured: 1 / 2 / 4 / 8 / 16
    // waves 48.8 / 46.8 / 46.0 / 46.0 / 46.4 ms on C3).  A per-lane dynamic
    // hand-out from a warp pool kept 40 registers but cost 7%.
    return launch(k, smem, occupancy_grid(k, smem, d, n, kTrialWaves), s, g->nat, p, o, exit_cnt,
                  q);
  }, inj, full, true, false, g->uniform_exits && !generic_exits());
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
