// gsde_abi.cu -- the extern "C" boundary (include/gsde.h): graph upload,
// argument checks, stream/mode dispatch and host-side scalar helpers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gsde_internal.h"

namespace gsde {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int set_error(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

DevInfo dev_info(int device) {
  static std::mutex mu;
  static std::vector<DevInfo> cache;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)cache.size() <= device) cache.resize(device + 1);
  if (cache[device].sm_count == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device].sm_count = v > 0 ? v : 1;
  }
  return cache[device];
}

namespace {

// Scoped device switch (restores the caller's current device).
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int cuda_fail(cudaError_t e, const char *what) {
  return set_error(GSDE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Vose alias table over one vertex's slot weights: column j keeps slot j
// with probability prob[j], else jumps to alias[j].
// (scratch vectors reused across vertices: a 1e5-vertex network otherwise
// spends its graph upload in the allocator)
void build_alias(const double *w, int deg, std::vector<double> &prob, std::vector<int> &alias) {
  static thread_local std::vector<double> p;
  static thread_local std::vector<int> small, large;
  prob.assign(deg, 1.0);
  alias.resize(deg);
  p.resize(deg);
  small.clear();
  large.clear();
  double tot = 0.0;
  for (int j = 0; j < deg; ++j) tot += w[j];
  for (int j = 0; j < deg; ++j) {
    alias[j] = j;
    p[j] = tot > 0.0 ? w[j] / tot * deg : 1.0;
    (p[j] < 1.0 ? small : large).push_back(j);
  }
  while (!small.empty() && !large.empty()) {
    const int s = small.back();
    small.pop_back();
    const int l = large.back();
    large.pop_back();
    prob[s] = p[s];
    alias[s] = l;
    p[l] = (p[l] + p[s]) - 1.0;
    (p[l] < 1.0 ? small : large).push_back(l);
  }
  for (int j : small) prob[j] = 1.0, alias[j] = j;
  for (int j : large) prob[j] = 1.0, alias[j] = j;
}

// Recycled device arenas (graph handles are often re-created per call with
// the same size): avoids cudaMalloc / cudaFree -- both device-synchronising
// and slow once the process holds large caching-allocator pools.
struct ArenaPool {
  struct Entry {
    int device;
    void *ptr;
    size_t bytes;
  };
  std::mutex mu;
  std::vector<Entry> free;
  void *take(int device, size_t bytes, size_t *got) {
    std::lock_guard<std::mutex> lock(mu);
    for (size_t i = 0; i < free.size(); ++i) {
      const Entry e = free[i];
      if (e.device == device && e.bytes >= bytes && e.bytes <= 2 * bytes + 4096) {
        free.erase(free.begin() + (long)i);
        *got = e.bytes;
        return e.ptr;
      }
    }
    return nullptr;
  }
  // returns false when the pool is full (caller frees)
  bool give(int device, void *ptr, size_t bytes) {
    std::lock_guard<std::mutex> lock(mu);
    if (free.size() >= 16) return false;
    free.push_back(Entry{device, ptr, bytes});
    return true;
  }
};
ArenaPool &arena_pool() {
  static ArenaPool *pool = new ArenaPool();  // never destroyed: outlives static teardown
  return *pool;
}

size_t g_is_general_size(int32_t is_star, int64_t S) { return is_star ? 0 : (size_t)S * 5; }

// Device-arena layout: 256-byte aligned slices, sizes known up front, so the
// packing loops write straight into the upload buffer.
struct Layout {
  size_t size = 0;
  size_t add(size_t bytes) {
    const size_t off = (size + 255) & ~size_t(255);
    size = off + (bytes ? bytes : 1);
    return off;
  }
};

// Process-wide pinned staging buffer for graph uploads, grown on demand and
// kept: every graph_create packs into warm, page-locked memory (a 1e5-edge
// network spent ~30 ms of its upload in first-touch page faults of fresh
// host vectors, and the copy from pageable memory ran at ~5 GB/s).
struct Staging {
  std::mutex mu;
  unsigned char *buf = nullptr;
  size_t cap = 0;
  unsigned char *get(size_t bytes) {  // caller holds mu
    if (bytes > cap) {
      if (buf) cudaFreeHost(buf);
      buf = nullptr;
      cap = 0;
      const size_t want = bytes + bytes / 4;
      if (cudaHostAlloc(&buf, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        buf = nullptr;
        return nullptr;
      }
      cap = want;
    }
    return buf;
  }
};
Staging &staging() {
  static Staging *s = new Staging();  // never destroyed
  return *s;
}

}  // namespace
}  // namespace gsde

using namespace gsde;

extern "C" {

int gsde_abi_version(void) { return GSDE_ABI_VERSION; }
const char *gsde_last_error(void) { return g_last_error.c_str(); }
int64_t gsde_launch_count(void) { return g_launches.load(); }

uint64_t gsde_raw64(uint64_t seed, uint64_t stream, uint64_t index) {
  return raw64(seed, stream, index);
}
double gsde_uniform01(uint64_t seed, uint64_t stream, uint64_t index) {
  return u53_to_uniform(raw64(seed, stream, index) >> 11);
}
double gsde_normal(uint64_t seed, uint64_t stream, uint64_t index) {
  return u64_to_normal(raw64(seed, stream, index));
}
double gsde_u64_to_uniform(uint64_t r) { return u53_to_uniform(r >> 11); }
double gsde_u64_to_normal(uint64_t r) { return u64_to_normal(r); }
double gsde_norm_ppf(double p) {
  const double q = p - 0.5;
  return norm_ppf_qt(q, q < 0.0 ? p : 1.0 - p);
}
double gsde_solve_first_passage_s(double a, double b, double c) {
  return solve_first_passage_s<double>(a, b, c);
}

int gsde_graph_create(const gsde_graph_desc *d, int device, gsde_graph **out) {
  if (!d || !out) return set_error(GSDE_EINVAL, "graph_create: null argument");
  *out = nullptr;
  const int64_t E = d->n_edges, V = d->n_vertices;
  if (E < 1 || V < 1 || E > (1ll << 30) || V > (1ll << 30))
    return set_error(GSDE_EINVAL, "graph_create: bad sizes E=%lld V=%lld", (long long)E,
                     (long long)V);
  const int64_t S = d->v_off[V];
  const int64_t T = d->n_tab;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return set_error(GSDE_ENODEV, "graph_create: CUDA device %d unavailable", device);
  DeviceGuard guard(device);
  if (!guard.ok) return set_error(GSDE_ENODEV, "graph_create: cannot select device %d", device);

  static const bool timing = std::getenv("GSDE_TIMING") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto lap = [&](const char *what) {
    if (!timing) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gsde] graph_create %s: %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_start).count());
    t_start = t;
  };
  // --- layout of the device arena ----------------------------------------
  const int64_t T1 = T ? T : 1;
  const size_t nfat = g_is_general_size(d->is_star, S);
  Layout Lo;
  const size_t o_len64 = Lo.add(E * 8), o_coef64 = Lo.add(E * 8), o_sig64 = Lo.add(E * 8),
               o_tabx64 = Lo.add(T1 * 8), o_tabmu64 = Lo.add(T1 * 8), o_len32 = Lo.add(E * 4),
               o_coef32 = Lo.add(E * 4), o_sig32 = Lo.add(E * 4), o_tabx32 = Lo.add(T1 * 4),
               o_tabmu32 = Lo.add(T1 * 4), o_einit = Lo.add(E * 4), o_eterm = Lo.add(E * 4),
               o_voff = Lo.add((V + 1) * 4), o_vedges = Lo.add(S * 4), o_vorient = Lo.add(S),
               o_thresh = Lo.add(S * 8), o_kind = Lo.add(E), o_taboff = Lo.add((E + 1) * 4),
               o_nedge = Lo.add(E * sizeof(float4)), o_nedgev = Lo.add(E * sizeof(int4)),
               o_ncol = Lo.add(S * sizeof(int4)), o_nfat = Lo.add(nfat * sizeof(int4)),
               o_nufat = Lo.add((d->is_star ? 0 : (size_t)S * 3) * sizeof(int4)),
               o_work = Lo.add(gsde_graph::kWorkSlots * sizeof(unsigned long long));
  Staging &st = staging();
  std::lock_guard<std::mutex> staging_lock(st.mu);
  unsigned char *H = st.get(Lo.size);
  if (!H) return set_error(GSDE_ENOMEM, "graph_create: cudaHostAlloc(%zu) failed", Lo.size);
  auto at = [&](size_t off, auto *type) { return reinterpret_cast<decltype(type)>(H + off); };
  double *len64 = at(o_len64, (double *)0), *coef64 = at(o_coef64, (double *)0),
         *sig64 = at(o_sig64, (double *)0), *tabx64 = at(o_tabx64, (double *)0),
         *tabmu64 = at(o_tabmu64, (double *)0);
  float *len32 = at(o_len32, (float *)0), *coef32 = at(o_coef32, (float *)0),
        *sig32 = at(o_sig32, (float *)0), *tabx32 = at(o_tabx32, (float *)0),
        *tabmu32 = at(o_tabmu32, (float *)0);
  int32_t *einit = at(o_einit, (int32_t *)0), *eterm = at(o_eterm, (int32_t *)0),
          *voff = at(o_voff, (int32_t *)0), *vedges = at(o_vedges, (int32_t *)0),
          *taboff = at(o_taboff, (int32_t *)0);
  uint8_t *vorient = at(o_vorient, (uint8_t *)0), *kind = at(o_kind, (uint8_t *)0);
  uint64_t *thresh = at(o_thresh, (uint64_t *)0);
  float4 *nedge = at(o_nedge, (float4 *)0);
  int4 *nedgev = at(o_nedgev, (int4 *)0), *ncol = at(o_ncol, (int4 *)0),
       *nfat4 = at(o_nfat, (int4 *)0), *nufat4 = at(o_nufat, (int4 *)0);
  memset(at(o_work, (unsigned char *)0), 0, gsde_graph::kWorkSlots * sizeof(unsigned long long));
  tabx64[0] = tabmu64[0] = 0.0;
  tabx32[0] = tabmu32[0] = 0.0f;

  // --- host-side packing (into the pinned staging buffer) -----------------
  // validation first (the packing loops below run in parallel: OpenMP over
  // edges / slots / vertices for large networks -- a 1e5-edge upload)
  for (int64_t e = 0; e < E; ++e)
    if (d->dkind[e] < 0 || d->dkind[e] > 2)
      return set_error(GSDE_EINVAL, "graph_create: bad drift kind on edge %lld", (long long)e);
  for (int64_t v = 0; v < V; ++v)
    if (d->v_off[v + 1] - d->v_off[v] < 1)
      return set_error(GSDE_EINVAL, "graph_create: vertex %lld has no slots", (long long)v);
  const bool par = E + S > 32768;
  bool has_tab = false, zero_drift = true, const_drift = true;
#pragma omp parallel for if (par) reduction(|| : has_tab) reduction(&& : zero_drift, const_drift)
  for (int64_t e = 0; e < E; ++e) {
    einit[e] = (int32_t)d->edge_init[e];
    eterm[e] = (int32_t)d->edge_term[e];
    len64[e] = d->edge_length[e];
    len32[e] = (float)d->edge_length[e];
    kind[e] = (uint8_t)d->dkind[e];
    coef64[e] = d->dcoef[e];
    coef32[e] = (float)d->dcoef[e];
    sig64[e] = d->sigma[e];
    sig32[e] = (float)d->sigma[e];
    has_tab = has_tab || kind[e] == 2;
    zero_drift = zero_drift && !(kind[e] == 2 || d->dcoef[e] != 0.0);
    const_drift = const_drift && !(kind[e] == 2 || (kind[e] == 1 && d->dcoef[e] != 0.0));
  }
  for (int64_t e = 0; e <= E; ++e) taboff[e] = (int32_t)d->tab_off[e];
  for (int64_t t = 0; t < T; ++t) {
    tabx64[t] = d->tab_x[t];
    tabmu64[t] = d->tab_mu[t];
    tabx32[t] = (float)d->tab_x[t];
    tabmu32[t] = (float)d->tab_mu[t];
  }
  for (int64_t v = 0; v <= V; ++v) voff[v] = (int32_t)d->v_off[v];
  const double two53 = 9007199254740992.0;
#pragma omp parallel for if (par)
  for (int64_t j = 0; j < S; ++j) {
    vedges[j] = (int32_t)d->v_edges[j];
    vorient[j] = (uint8_t)d->v_orient[j];
    double c = std::floor(d->v_cumw[j] * two53);  // exact: scaling by 2^53
    if (!(c > 0.0)) c = 0.0;
    if (c > two53) c = two53;
    thresh[j] = (uint64_t)c;
  }
  // native records
#pragma omp parallel for if (par)
  for (int64_t e = 0; e < E; ++e) {
    float4 r;
    // FP32 length rounded toward zero, so every native position (<= the FP32
    // length) also lies within the reference's FP64 edge [0, l]
    r.x = len32[e];
    if (std::isfinite(len64[e]) && (double)r.x > len64[e]) r.x = std::nextafter(r.x, 0.0f);
    // sigma * sqrt(2 ln 2): the native Box-Muller returns z / sqrt(2 ln 2)
    r.w = (float)(d->sigma[e] * 1.1774100225154747);
    if (kind[e] == 0) {
      r.y = coef32[e];
      r.z = 0.0f;
    } else if (kind[e] == 1) {
      r.y = 0.0f;
      r.z = coef32[e];
    } else {
      int32_t off = taboff[e];
      memcpy(&r.y, &off, sizeof(float));
      r.z = NAN;
    }
    if (d->is_star) {
      // star edges are semi-infinite: the x slot carries sig^2 / mu(0)^2 of the
      // native record (the failed-excursion time per w^2; constant drift mu0 =
      // the coefficient, linear mu0 = 0 -> inf; tabulated drifts keep the
      // generic formula in their kernel)
      const double mu0 = kind[e] == 0 ? (double)r.y : 0.0;
      r.x = kind[e] == 2 ? NAN
            : (mu0 != 0.0 ? (float)(((double)r.w * r.w) / (mu0 * mu0)) : INFINITY);
    }
    nedge[e] = r;
    const int32_t a = einit[e], b = eterm[e];
    nedgev[e] = make_int4(voff[a], voff[a + 1] - voff[a], b >= 0 ? voff[b] : 0,
                          b >= 0 ? voff[b + 1] - voff[b] : 0);
  }
#pragma omp parallel if (par)
  {
    std::vector<double> prob;
    std::vector<int> alias;
#pragma omp for schedule(static, 1024)
    for (int64_t v = 0; v < V; ++v) {
      const int lo = voff[v], deg = voff[v + 1] - voff[v];
      build_alias(d->v_weights + lo, deg, prob, alias);
      for (int j = 0; j < deg; ++j) {
        const int sp = lo + j, sa = lo + alias[j];
        const uint32_t prim = (uint32_t)vedges[sp] | ((uint32_t)vorient[sp] << 31);
        const uint32_t alt = (uint32_t)vedges[sa] | ((uint32_t)vorient[sa] << 31);
        double t = std::nearbyint(prob[j] * 4294967296.0);
        uint32_t th = t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)(t > 0.0 ? t : 0.0);
        int4 c;
        c.x = (int)th;
        c.y = (int)prim;
        c.z = (int)(prob[j] >= 1.0 ? prim : alt);
        c.w = 0;
        ncol[sp] = c;
      }
    }
  }
  lap("records + alias tables");
  // fat alias columns for general graphs (one L2 round trip per vertex event)
  if (!d->is_star) {
#pragma omp parallel for if (par)
    for (int64_t j = 0; j < S; ++j) {
      const int4 c = ncol[j];
      const int pe = c.y & 0x7fffffff, ae = c.z & 0x7fffffff;
      int4 pe4, ae4;
      memcpy(&pe4, &nedge[pe], sizeof(int4));
      memcpy(&ae4, &nedge[ae], sizeof(int4));
      nfat4[5 * j + 0] = c;
      nfat4[5 * j + 1] = pe4;
      nfat4[5 * j + 2] = nedgev[pe];
      nfat4[5 * j + 3] = ae4;
      nfat4[5 * j + 4] = nedgev[ae];
      nufat4[3 * j + 0] = make_int4(c.y, 0, 0, 0);
      nufat4[3 * j + 1] = pe4;
      nufat4[3 * j + 2] = nedgev[pe];
    }
  }
  // every column's alias is its own slot (prob >= 1: equal jump weights)?
  bool uniform_exits = true;
  for (int64_t j = 0; j < S && uniform_exits; ++j) uniform_exits = ncol[j].y == ncol[j].z;
  lap("fat columns");
  size_t arena_bytes = Lo.size;
  void *dev = arena_pool().take(device, Lo.size, &arena_bytes);
  cudaError_t err = cudaSuccess;
  if (!dev) {
    err = cudaMalloc(&dev, Lo.size);
    if (err != cudaSuccess) return set_error(GSDE_ENOMEM, "graph_create: cudaMalloc(%zu): %s",
                                             Lo.size, cudaGetErrorString(err));
  }
  err = cudaMemcpy(dev, H, Lo.size, cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(dev);
    return cuda_fail(err, "graph_create: upload");
  }
  lap("device arena + upload");
  auto P = [&](size_t off) { return (void *)((unsigned char *)dev + off); };
  gsde_graph *g = new gsde_graph();
  g->device = device;
  g->E = E;
  g->V = V;
  g->S = S;
  g->T = T;
  g->is_star = d->is_star != 0;
  g->has_tab = has_tab;
  g->zero_drift = zero_drift;
  g->const_drift = const_drift;
  g->arena = dev;
  g->arena_bytes = (int64_t)arena_bytes;
  g->work = (unsigned long long *)P(o_work);
  auto fill_ref = [&](auto &R, size_t ol, size_t oc, size_t os, size_t ox, size_t om) {
    using T_ = std::remove_pointer_t<decltype(R.edge_len)>;
    R.n_edges = (int32_t)E;
    R.edge_len = (const T_ *)P(ol);
    R.dcoef = (const T_ *)P(oc);
    R.sigma = (const T_ *)P(os);
    R.tab_x = (const T_ *)P(ox);
    R.tab_mu = (const T_ *)P(om);
    R.edge_init = (const int32_t *)P(o_einit);
    R.edge_term = (const int32_t *)P(o_eterm);
    R.v_off = (const int32_t *)P(o_voff);
    R.v_edges = (const int32_t *)P(o_vedges);
    R.v_orient = (const uint8_t *)P(o_vorient);
    R.v_thresh = (const uint64_t *)P(o_thresh);
    R.dkind = (const uint8_t *)P(o_kind);
    R.tab_off = (const int32_t *)P(o_taboff);
  };
  fill_ref(g->ref64, o_len64, o_coef64, o_sig64, o_tabx64, o_tabmu64);
  fill_ref(g->ref32, o_len32, o_coef32, o_sig32, o_tabx32, o_tabmu32);
  g->nat.n_edges = (int32_t)E;
  g->nat.n_slots = (int32_t)S;
  g->nat.edge = (const float4 *)P(o_nedge);
  g->nat.edgev = (const int4 *)P(o_nedgev);
  g->nat.col = (const int4 *)P(o_ncol);
  g->nat.fat = d->is_star ? nullptr : (const int4 *)P(o_nfat);
  g->nat.ufat = d->is_star ? nullptr : (const int4 *)P(o_nufat);
  g->uniform_exits = uniform_exits;
  g->nat.tab_off = (const int32_t *)P(o_taboff);
  g->nat.tab_x = (const float *)P(o_tabx32);
  g->nat.tab_mu = (const float *)P(o_tabmu32);
  g->nat.has_tab = has_tab ? 1 : 0;
  const int64_t stage = E * (g->is_star ? 16 : 32) + S * 16;
  g->nat_graph_smem = stage <= 32 * 1024 ? stage : 0;
  *out = g;
  return GSDE_OK;
}

int gsde_graph_destroy(gsde_graph *g) {
  if (!g) return GSDE_OK;
  DeviceGuard guard(g->device);
  // like cudaFree, wait for queued kernels that may still read the arena
  // (on any stream) before it can be recycled
  cudaError_t err = cudaDeviceSynchronize();
  if (err == cudaSuccess && !arena_pool().give(g->device, g->arena, (size_t)g->arena_bytes))
    err = cudaFree(g->arena);
  for (cudaEvent_t ev : g->work_done)
    if (ev) cudaEventDestroy(ev);
  delete g;
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "graph_destroy");
}

int64_t gsde_graph_device_bytes(const gsde_graph *g) { return g ? g->arena_bytes : 0; }

static int check_stream_args(int32_t stream, int32_t precision, const uint64_t *inj_raw,
                             const double *inj_normal, int64_t inj_stride, const char *who) {
  if (stream != GSDE_STREAM_NATIVE && stream != GSDE_STREAM_REFERENCE &&
      stream != GSDE_STREAM_INJECT)
    return set_error(GSDE_EINVAL, "%s: unknown stream mode %d", who, stream);
  if (stream == GSDE_STREAM_INJECT) {
    if (!inj_raw || !inj_normal || inj_stride < 1)
      return set_error(GSDE_EINVAL, "%s: INJECT needs inj_raw, inj_normal and inj_stride", who);
    if (precision != GSDE_PREC_F32 && precision != GSDE_PREC_F64 &&
        precision != GSDE_PREC_NATIVE)
      return set_error(GSDE_EINVAL, "%s: unknown precision %d", who, precision);
  }
  return GSDE_OK;
}

int gsde_ensemble(const gsde_graph *g, const gsde_run *a, const gsde_out *o, void *stream) {
  if (!g || !a || !o) return set_error(GSDE_EINVAL, "ensemble: null argument");
  if (a->n_particles < 0 || a->n_steps < 0)
    return set_error(GSDE_EINVAL, "ensemble: n_steps and n_particles must be nonnegative");
  if (!(a->dt > 0.0) || !std::isfinite(a->dt))
    return set_error(GSDE_EINVAL, "ensemble: dt must be positive and finite");
  if (a->cap < 1) return set_error(GSDE_EINVAL, "ensemble: cap must be >= 1");
  if (a->reflect_len < 0.0 || (a->reflect_len > 0.0 && !g->is_star))
    return set_error(GSDE_EINVAL, "ensemble: reflect_len applies to star graphs only");
  if (a->init_kind != GSDE_INIT_POINT && a->init_kind != GSDE_INIT_PER_EDGE_UNIFORM &&
      a->init_kind != GSDE_INIT_STATE)
    return set_error(GSDE_EINVAL, "ensemble: bad init_kind %d", a->init_kind);
  if (a->init_kind == GSDE_INIT_STATE) {
    if (!a->state_edge || !a->state_x)
      return set_error(GSDE_EINVAL, "ensemble: GSDE_INIT_STATE needs state_edge and state_x");
    if (!(a->stream == GSDE_STREAM_NATIVE ||
          (a->stream == GSDE_STREAM_INJECT && a->precision == GSDE_PREC_NATIVE)))
      return set_error(GSDE_EINVAL, "ensemble: GSDE_INIT_STATE runs the NATIVE or "
                                    "INJECT/NATIVE streams (REFERENCE states: gsde_step_batch)");
  }
  if (o->counter && !(a->stream == GSDE_STREAM_NATIVE ||
                      (a->stream == GSDE_STREAM_INJECT && a->precision == GSDE_PREC_NATIVE)))
    return set_error(GSDE_EINVAL, "ensemble: the counter output is a NATIVE / INJECT-NATIVE "
                                  "output");
  if (a->init_kind == GSDE_INIT_POINT && (a->init_edge < 0 || a->init_edge >= g->E))
    return set_error(GSDE_EINVAL, "ensemble: init_edge out of range");
  if ((o->hist || o->occ) && (!o->hist_offsets || !o->hist_counts || !o->hist_dx ||
                               o->hist_n_cells < 1))
    return set_error(GSDE_EINVAL, "ensemble: hist/occ need offsets, counts, dx and n_cells");
  if (o->occ && (o->occ_every < 1 || o->occ_start < 0 || o->occ_every > 0x7fffffff ||
                 o->occ_start > 0x7fffffff))
    return set_error(GSDE_EINVAL, "ensemble: occ_every must be >= 1 and occ_start >= 0");
  int rc = check_stream_args(a->stream, a->precision, a->inj_raw, a->inj_normal, a->inj_stride,
                             "ensemble");
  if (rc) return rc;
  if (a->stream == GSDE_STREAM_NATIVE && a->n_steps > 0x7fffffffll)
    return set_error(GSDE_EINVAL, "ensemble: NATIVE stream supports n_steps < 2^31");
  // NATIVE stream ids carry the block-counter carry in bits 48.. (gsde_native.cu)
  if (a->stream == GSDE_STREAM_NATIVE &&
      (a->pid_offset < 0 || a->pid_offset + a->n_particles > (1ll << 48)))
    return set_error(GSDE_EINVAL, "ensemble: NATIVE stream particle ids must lie in [0, 2^48)");
  const bool native_inj = a->stream == GSDE_STREAM_INJECT && a->precision == GSDE_PREC_NATIVE;
  if (native_inj && o->occ)
    return set_error(GSDE_EINVAL, "ensemble: INJECT/NATIVE does not sample the occupation "
                                  "histogram");
  if (native_inj && (a->n_steps > 0x7fffffffll || a->inj_stride > 0x7fffffffll))
    return set_error(GSDE_EINVAL, "ensemble: INJECT/NATIVE needs n_steps, inj_stride < 2^31");
  if (o->progress) {
    if (!(a->stream == GSDE_STREAM_NATIVE || native_inj))
      return set_error(GSDE_EINVAL, "ensemble: progress counters are a NATIVE / INJECT-NATIVE "
                                    "output");
    if (!(o->edge || o->x || o->crossings || o->events || o->truncs))
      return set_error(GSDE_EINVAL, "ensemble: progress counts per-particle outputs; none asked");
    if (o->progress_base < 0 || o->progress_shift < 0 || o->progress_shift > 62)
      return set_error(GSDE_EINVAL, "ensemble: progress_base >= 0, progress_shift in [0, 62]");
  }
  if (a->n_particles == 0) return GSDE_OK;
  DeviceGuard guard(g->device);
  const cudaStream_t s = (cudaStream_t)stream;
  const cudaError_t err = (a->stream == GSDE_STREAM_NATIVE || native_inj)
                              ? launch_native_ensemble(g, *a, *o, s)
                              : launch_ref_ensemble(g, *a, *o, s);
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "ensemble launch");
}

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda
// link); resolved once
int gsde_stream_wait_geq32(void *stream, const uint32_t *addr, uint32_t value) {
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<WaitFn>(f);
  }();
  if (!addr) return set_error(GSDE_EINVAL, "stream_wait_geq32: null address");
  if (!fn) return set_error(GSDE_ECUDA, "stream_wait_geq32: cuStreamWaitValue32 unavailable");
  const CUresult r = fn((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS)
    return set_error(GSDE_ECUDA, "stream_wait_geq32: cuStreamWaitValue32 failed (%d)", (int)r);
  return GSDE_OK;
}

int gsde_vertex_trials(const gsde_graph *g, const gsde_trials *a, const gsde_trials_out *o,
                       void *stream) {
  if (!g || !a || !o) return set_error(GSDE_EINVAL, "vertex_trials: null argument");
  if (a->n_trials < 0) return set_error(GSDE_EINVAL, "vertex_trials: n_trials must be >= 0");
  if (!(a->dt > 0.0)) return set_error(GSDE_EINVAL, "vertex_trials: dt must be positive");
  if (a->cap < 1) return set_error(GSDE_EINVAL, "vertex_trials: cap must be >= 1");
  if (!g->is_star && (a->start_edge < 0 || a->start_edge >= g->E))
    return set_error(GSDE_EINVAL, "vertex_trials: start_edge out of range");
  int rc = check_stream_args(a->stream, a->precision, a->inj_raw, a->inj_normal, a->inj_stride,
                             "vertex_trials");
  if (rc) return rc;
  const bool native_inj = a->stream == GSDE_STREAM_INJECT && a->precision == GSDE_PREC_NATIVE;
  if (native_inj && a->inj_stride > 0x7fffffffll)
    return set_error(GSDE_EINVAL, "vertex_trials: INJECT/NATIVE needs inj_stride < 2^31");
  if (a->n_trials == 0) return GSDE_OK;
  DeviceGuard guard(g->device);
  const cudaStream_t s = (cudaStream_t)stream;
  const cudaError_t err = (a->stream == GSDE_STREAM_NATIVE || native_inj)
                              ? launch_native_trials(g, *a, *o, s)
                              : launch_ref_trials(g, *a, *o, s);
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "vertex_trials launch");
}

int gsde_step_batch(const gsde_graph *g, const gsde_step_args *a, int64_t *edge, double *x,
                    uint64_t *k, int64_t *M, int64_t *trunc, void *stream) {
  if (!g || !a || !edge || !x || !k) return set_error(GSDE_EINVAL, "step_batch: null argument");
  if (a->n < 0 || !(a->dt > 0.0) || a->cap < 1)
    return set_error(GSDE_EINVAL, "step_batch: bad n / dt / cap");
  if (a->stream == GSDE_STREAM_NATIVE)
    return set_error(GSDE_EINVAL, "step_batch: REFERENCE or INJECT streams only");
  if (a->stream == GSDE_STREAM_REFERENCE && (!a->seed || !a->pid))
    return set_error(GSDE_EINVAL, "step_batch: REFERENCE needs seed and pid arrays");
  int rc = check_stream_args(a->stream, a->precision, a->inj_raw, a->inj_normal, a->inj_stride,
                             "step_batch");
  if (rc) return rc;
  if (a->stream == GSDE_STREAM_INJECT && a->precision == GSDE_PREC_NATIVE)
    return set_error(GSDE_EINVAL, "%s: INJECT/NATIVE is an ensemble mode", "step_batch");
  DeviceGuard guard(g->device);
  const cudaError_t err = launch_step_batch(g, *a, edge, x, k, M, trunc, (cudaStream_t)stream);
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "step_batch launch");
}

int gsde_histogram(int64_t n, const int64_t *edge, const double *x, const int64_t *offsets,
                   const int64_t *counts, const double *dx, int64_t n_cells, int64_t *hist,
                   void *stream) {
  if (n < 0 || n_cells < 1 || (n > 0 && (!edge || !x)) || !offsets || !counts || !dx || !hist)
    return set_error(GSDE_EINVAL, "histogram: bad arguments");
  const cudaError_t err =
      launch_histogram(n, edge, x, offsets, counts, dx, n_cells, hist, (cudaStream_t)stream);
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "histogram launch");
}

int gsde_fvm_run(const gsde_fvm_desc *d, double *rho, double *scratch, int64_t n_steps,
                 double dt, double neg_floor, int64_t *neg_step, uint64_t *red, void *stream) {
  if (!d || !rho || !scratch || !neg_step || !red || n_steps < 0 || !(dt > 0.0) ||
      d->n_edges < 1 || d->n_cells < 1 || d->n_vertices < 0 || d->n_pslot < 0 || d->n_vser < 0 ||
      !d->cell_mu_l || !d->cell_mu_r || !d->cell_D || !d->cell_dx || !d->cell_flags ||
      !d->v_off || (d->n_pslot && (!d->pslot || !d->slot_vertex || !d->tstart ||
                                   !d->rstart || !d->rpos || (d->n_terms && !d->terms))) ||
      (d->n_vser && !d->vser))
    return set_error(GSDE_EINVAL, "fvm_run: bad arguments");
  if (n_steps == 0) {
    const cudaError_t err = cudaMemsetAsync(neg_step, 0, sizeof(int64_t), (cudaStream_t)stream);
    return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "fvm_run memset");
  }
  const cudaError_t err =
      launch_fvm(*d, rho, scratch, n_steps, dt, neg_floor, neg_step, red, (cudaStream_t)stream);
  return err == cudaSuccess ? GSDE_OK : cuda_fail(err, "fvm launch");
}

}  // extern "C"
