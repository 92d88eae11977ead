/*
 * oracle/gsde_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the reference graphsde hot path
 * (/root/reference/pkg/src/graphsde/{rng,kernels,engine}.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product path (paper_2512_02175_b200) never does.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference here): Random123
 * Philox KATs, raw64/uniform/normal grids, solve_first_passage_s triples,
 * per-step em_step_* tuples, run_ensemble / vertex_crossing_trials outputs.
 *
 * Parallelism mirrors the reference: ensembles are split into CHUNK=4096
 * particle chunks with private M-histogram rows (kernels.py:41-43,339-369)
 * distributed over OpenMP threads; trials are distributed per trial
 * (kernels.py:468,509).  Results are thread-count independent.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_CHUNK 4096 /* kernels.py:43 */
#define INIT_POINT 0   /* kernels.py:49 */

/* ---- rng.py:19-22 Philox constants ---------------------------------- */
#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
#define PH_W0 0x9E3779B9u
#define PH_W1 0xBB67AE85u

/* rng.py:29-42 */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)PH_M0 * c0;
    uint64_t p1 = (uint64_t)PH_M1 * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PH_W0;
    k1 += PH_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.py:45-66: block = index>>1, ctr = (blk, stream), key = seed */
uint64_t orc_raw64(uint64_t seed, uint64_t stream, uint64_t index) {
  uint64_t blk = index >> 1;
  uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)stream,
                     (uint32_t)(stream >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, key, x);
  if ((index & 1u) == 0) return ((uint64_t)x[0] << 32) | x[1];
  return ((uint64_t)x[2] << 32) | x[3];
}

static const double INV_2_53 = 1.0 / 9007199254740992.0;

/* rng.py:69-72 */
double orc_u64_to_uniform(uint64_t r) { return (double)(r >> 11) * INV_2_53; }

/* rng.py:81-134: AS241 layout, two Newton polishes in the far tail.
 * Written on (q = p - 1/2, pt = min(p, 1-p)) so the lattice map below can pass
 * both exactly. */
static double norm_ppf_qt(double q, double pt) {
  if (fabs(q) <= 0.425) {
    double r = 0.180625 - q * q;
    double num = (((((((2.5090809287301226727e3 * r + 3.3430575583588128105e4) * r +
                       6.7265770927008700853e4) * r + 4.5921953931549871457e4) * r +
                     1.3731693765509461125e4) * r + 1.9715909503065514427e3) * r +
                   1.3314166789178437745e2) * r + 3.3871328727963666080e0);
    double den = (((((((5.2264952788528545610e3 * r + 2.8729085735721942674e4) * r +
                       3.9307895800092710610e4) * r + 2.1213794301586595867e4) * r +
                     5.3941960214247511077e3) * r + 6.8718700749205790830e2) * r +
                   4.2313330701600911252e1) * r + 1.0);
    return q * num / den;
  }
  double r = sqrt(-log(pt));
  if (r <= 5.0) {
    double rr = r - 1.6;
    double num = (((((((7.74545014278341407640e-4 * rr + 2.27238449892691845833e-2) * rr +
                       2.41780725177450611770e-1) * rr + 1.27045825245236838258e0) * rr +
                     3.64784832476320460504e0) * rr + 5.76949722146069140550e0) * rr +
                   4.63033784615654529590e0) * rr + 1.42343711074968357734e0);
    double den = (((((((1.05075007164441684324e-9 * rr + 5.47593808499534494600e-4) * rr +
                       1.51986665636164571966e-2) * rr + 1.48103976427480074590e-1) * rr +
                     6.89767334985100004550e-1) * rr + 1.67638483018380384940e0) * rr +
                   2.05319162663775882187e0) * rr + 1.0);
    double val = num / den;
    return q < 0.0 ? -val : val;
  }
  double rr = r - 5.0;
  double num = (((((((2.01033439929228813265e-7 * rr + 2.71155556874348757815e-5) * rr +
                     1.24266094738807843860e-3) * rr + 2.65321895265761230930e-2) * rr +
                   2.96560571828504891230e-1) * rr + 1.78482653991729133580e0) * rr +
                 5.46378491116411436990e0) * rr + 6.65790464350110377720e0);
  double den = (((((((2.04426310338993978564e-15 * rr + 1.42151175831644588870e-9) * rr +
                     1.84631831751005468180e-6) * rr + 7.86869131145613259100e-4) * rr +
                   1.48753612908506148525e-2) * rr + 1.36929880922735805310e-1) * rr +
                 5.99832206555887937690e-1) * rr + 1.0);
  double val = num / den;
  double x = -val;
  for (int i = 0; i < 2; ++i) {
    double cdf = 0.5 * erfc(-x / 1.4142135623730951);
    double pdf = 0.3989422804014327 * exp(-0.5 * x * x);
    x -= (cdf - pt) / pdf;
  }
  val = -x;
  return q < 0.0 ? -val : val;
}

double orc_norm_ppf(double p) {
  double q = p - 0.5;
  return norm_ppf_qt(q, q < 0.0 ? p : 1.0 - p);
}

/* rng.py:137-143: p = (n + 1/2) 2^-53 on the centred 53-bit lattice.  Evaluated
 * exactly: q = (n - 2^52 + 1/2) 2^-53 and min(p, 1-p) are both representable,
 * whereas rounding p first (strict IEEE reading of the Python source) maps the
 * top lattice point to p = 1 and returns NaN.  The reference's compiled
 * (numba fastmath) code returns the finite quantile there, as does this. */
double orc_u64_to_normal(uint64_t r) {
  int64_t n = (int64_t)(r >> 11);
  double q = ((double)(n - 4503599627370496LL) + 0.5) * INV_2_53;
  /* upper half: 1 - p as the reference's compiled (fastmath) code forms it,
   * 1 - n 2^-53 (the 2^-54 term is reassociated away; tests/golden/validators.json) */
  double pt = q < 0.0 ? ((double)n + 0.5) * INV_2_53
                      : (double)(9007199254740992LL - n) * INV_2_53;
  return norm_ppf_qt(q, pt);
}

void orc_histogram(int64_t n, const int64_t *edges, const double *x, const int64_t *offsets,
                   const int64_t *counts, const double *dx, int64_t *hist);

/* ---- draw lookahead buffer (kernels.py:46, :55-64): value-neutral ---------- */
#define ORC_BUF 64
typedef struct {
  uint64_t seed, pid, k, kbase;
  uint64_t buf[ORC_BUF];
} orc_draws;

/* Refill: ORC_BUF/2 independent Philox blocks (each block is draws 2b and
 * 2b+1, rng.py:45-66) in a branch-free loop the compiler vectorises; the
 * buffer starts at an even draw index so every block is computed once. */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void draws_refill(orc_draws *d) {
  const uint64_t base = d->k & ~(uint64_t)1;
  const uint32_t s0 = (uint32_t)d->seed, s1 = (uint32_t)(d->seed >> 32);
  const uint32_t p0 = (uint32_t)d->pid, p1 = (uint32_t)(d->pid >> 32);
  for (int j = 0; j < ORC_BUF / 2; ++j) {
    const uint64_t blk = (base >> 1) + (uint64_t)j;
    uint32_t c0 = (uint32_t)blk, c1 = (uint32_t)(blk >> 32), c2 = p0, c3 = p1;
    uint32_t k0 = s0, k1 = s1;
    for (int r = 0; r < 10; ++r) {
      const uint64_t q0 = (uint64_t)PH_M0 * c0;
      const uint64_t q1 = (uint64_t)PH_M1 * c2;
      const uint32_t n0 = (uint32_t)(q1 >> 32) ^ c1 ^ k0;
      const uint32_t n2 = (uint32_t)(q0 >> 32) ^ c3 ^ k1;
      c1 = (uint32_t)q1;
      c3 = (uint32_t)q0;
      c0 = n0;
      c2 = n2;
      k0 += PH_W0;
      k1 += PH_W1;
    }
    d->buf[2 * j] = ((uint64_t)c0 << 32) | c1;
    d->buf[2 * j + 1] = ((uint64_t)c2 << 32) | c3;
  }
  d->kbase = base;
}

static inline uint64_t draw(orc_draws *d) {
  if (d->k - d->kbase >= ORC_BUF) draws_refill(d);
  return d->buf[d->k++ - d->kbase];
}

static inline void draws_init(orc_draws *d, uint64_t seed, uint64_t pid, uint64_t k) {
  d->seed = seed;
  d->pid = pid;
  d->k = k;
  d->kbase = k - ORC_BUF; /* empty: first draw refills */
}

/* ---- packed graph + field (graph.py:102-125, coefficients.py:121-152) -- */
typedef struct {
  int64_t n_edges, n_vertices;
  const double *edge_len;
  const int64_t *edge_init, *edge_term;
  const int64_t *v_off, *v_edges;
  const int8_t *v_orient;
  const double *v_cumw;
  const int8_t *dkind;
  const double *dcoef;
  const int64_t *tab_off;
  const double *tab_x, *tab_mu, *sigma;
} orc_graph;

/* kernels.py:67-85 */
static double drift_at(const orc_graph *g, int64_t e, double x) {
  int kd = g->dkind[e];
  if (kd == 0) return g->dcoef[e];
  if (kd == 1) return g->dcoef[e] * x;
  int64_t lo = g->tab_off[e], hi = g->tab_off[e + 1];
  if (x <= g->tab_x[lo]) return g->tab_mu[lo];
  if (x >= g->tab_x[hi - 1]) return g->tab_mu[hi - 1];
  int64_t j = lo + 1;
  while (g->tab_x[j] < x) ++j;
  double x0 = g->tab_x[j - 1];
  double t = (x - x0) / (g->tab_x[j] - x0);
  return g->tab_mu[j - 1] + t * (g->tab_mu[j] - g->tab_mu[j - 1]);
}

/* kernels.py:88-131 */
double orc_solve_first_passage_s(double a, double b, double c) {
  if (c < 0.0) return 0.0;
  if (c == 0.0) {
    if (b <= 0.0) return 0.0;
    if (a >= 0.0) return -1.0;
    double s = -b / a;
    return s < 1.0 ? s : 1.0;
  }
  if (a == 0.0) {
    if (b >= 0.0) return -1.0;
    double s = -c / b;
    return s < 1.0 ? s : 1.0;
  }
  double disc = b * b - 4.0 * a * c;
  if (disc < 0.0) disc = 0.0;
  double sq = sqrt(disc);
  double q = b >= 0.0 ? -0.5 * (b + sq) : -0.5 * (b - sq);
  double s = -1.0;
  double r1 = q / a;
  if (r1 >= 0.0) s = r1;
  if (q != 0.0) {
    double r2 = c / q;
    if (r2 >= 0.0 && (s < 0.0 || r2 < s)) s = r2;
  }
  if (s < 0.0) return -1.0;
  return s < 1.0 ? s : 1.0;
}

/* kernels.py:134-143 */
static int64_t pick_slot(const orc_graph *g, int64_t v, double u) {
  int64_t lo = g->v_off[v], hi = g->v_off[v + 1];
  for (int64_t j = lo; j < hi; ++j)
    if (u <= g->v_cumw[j]) return j;
  return hi - 1;
}

typedef struct {
  int64_t edge;
  double x;
  int64_t M;
  int32_t trunc;
  uint64_t k;
  /* diagnostics (not reference output): the smallest relative margin of the
   * step's continuous decisions -- |proposal - boundary| over the magnitude
   * of the terms that formed it (free / excursion accept tests, mirror
   * wall), |1 - alpha| (excursion residual time), |1 - s| for a split root
   * clamped near 1.  An FP32 evaluation can only take another branch where
   * this is within FP32 rounding (~1e-7 of the terms). */
  double margin;
} orc_step_out;

static inline double rel_margin(double v, double t0, double t1, double t2) {
  double s = fabs(t0);
  if (fabs(t1) > s) s = fabs(t1);
  if (fabs(t2) > s) s = fabs(t2);
  return s > 0.0 ? fabs(v) / s : INFINITY;
}
#define MG(m, v) do { double m_ = (v); if (m_ < (m)) (m) = m_; } while (0)

/* kernels.py:146-220 (draws: N on a free step; then U,N per vertex iteration) */
static orc_step_out step_star(const orc_graph *g, int64_t edge, double x, double dt,
                              orc_draws *d, int64_t cap, double reflect_len) {
  orc_step_out o;
  int64_t M = 0;
  double mg = INFINITY;
  if (x > 0.0) {
    double w = orc_u64_to_normal(draw(d));
    double mu = drift_at(g, edge, x);
    double a = mu * dt;
    double b = g->sigma[edge] * sqrt(dt) * w;
    double xn = x + a + b;
    MG(mg, rel_margin(xn, x, a, b));
    if (xn > 0.0) {
      if (reflect_len > 0.0) MG(mg, rel_margin(xn - reflect_len, x, a, b) /* wall */);
      if (reflect_len > 0.0 && xn > reflect_len) {
        xn = 2.0 * reflect_len - xn;
        if (xn < 0.0) xn = 0.0;
      }
      o.edge = edge; o.x = xn; o.M = 0; o.trunc = 0; o.k = d->k; o.margin = mg;
      return o;
    }
    double s = orc_solve_first_passage_s(a, b, x);
    if (s < 0.0) s = 1.0;
    if (s < 1.0) MG(mg, 1.0 - s);
    dt = (1.0 - s * s) * dt;
    if (dt < 0.0) dt = 0.0;
  }
  for (;;) {
    ++M;
    double u = orc_u64_to_uniform(draw(d));
    edge = g->v_edges[pick_slot(g, 0, u)];
    double w = orc_u64_to_normal(draw(d));
    double mu0 = drift_at(g, edge, 0.0);
    double sig0 = g->sigma[edge];
    double xn = mu0 * dt + sig0 * sqrt(dt) * fabs(w);
    MG(mg, rel_margin(xn, mu0 * dt, sig0 * sqrt(dt) * w, 0.0));
    if (xn >= 0.0) {
      if (reflect_len > 0.0) MG(mg, rel_margin(xn - reflect_len, mu0 * dt, sig0 * sqrt(dt) * w,
                                                reflect_len));
      if (reflect_len > 0.0 && xn > reflect_len) {
        xn = 2.0 * reflect_len - xn;
        if (xn < 0.0) xn = 0.0;
      }
      o.edge = edge; o.x = xn; o.M = M; o.trunc = 0; o.k = d->k; o.margin = mg;
      return o;
    }
    double alpha = (w * w * sig0 * sig0) / (mu0 * mu0 * dt);
    MG(mg, fabs(1.0 - alpha));
    dt = (1.0 - alpha) * dt;
    if (dt <= 0.0) {
      o.edge = edge; o.x = 0.0; o.M = M; o.trunc = 0; o.k = d->k; o.margin = mg;
      return o;
    }
    if (M >= cap) {
      o.edge = edge; o.x = 0.0; o.M = M; o.trunc = 1; o.k = d->k; o.margin = mg;
      return o;
    }
  }
}

/* kernels.py:223-288 (draws per iteration: [U if at a vertex], N) */
static orc_step_out step_general(const orc_graph *g, int64_t edge, double x, double dt,
                                 orc_draws *d, int64_t cap) {
  orc_step_out o;
  int64_t M = 0;
  double mg = INFINITY;
  for (;;) {
    double l = g->edge_len[edge];
    if (x <= 0.0 || x >= l) {
      int64_t v = x <= 0.0 ? g->edge_init[edge] : g->edge_term[edge];
      double u = orc_u64_to_uniform(draw(d));
      int64_t slot = pick_slot(g, v, u);
      edge = g->v_edges[slot];
      l = g->edge_len[edge];
      x = g->v_orient[slot] == 0 ? 0.0 : l;
    }
    double w = orc_u64_to_normal(draw(d));
    double mu = drift_at(g, edge, x);
    double a = mu * dt;
    double b = g->sigma[edge] * sqrt(dt) * w;
    double xn = x + a + b;
    MG(mg, rel_margin(xn, x, a, b));
    MG(mg, rel_margin(l - xn, l, a, b));
    if (0.0 < xn && xn < l) {
      o.edge = edge; o.x = xn; o.M = M; o.trunc = 0; o.k = d->k; o.margin = mg;
      return o;
    }
    ++M;
    double s;
    if (xn <= 0.0) {
      s = orc_solve_first_passage_s(a, b, x);
      x = 0.0;
    } else {
      s = orc_solve_first_passage_s(-a, -b, l - x);
      x = l;
    }
    if (s < 0.0) s = 1.0;
    if (s < 1.0) MG(mg, 1.0 - s);
    dt = (1.0 - s * s) * dt;
    if (dt <= 0.0) {
      o.edge = edge; o.x = x; o.M = M; o.trunc = 0; o.k = d->k; o.margin = mg;
      return o;
    }
    if (M >= cap) {
      o.edge = edge; o.x = x; o.M = M; o.trunc = 1; o.k = d->k; o.margin = mg;
      return o;
    }
  }
}

/* Single step, the per-step golden oracle (engine.py:206-270). */
void orc_step(const orc_graph *g, int32_t star, int64_t edge, double x, double dt,
              uint64_t seed, uint64_t pid, uint64_t k, int64_t cap, double reflect_len,
              int64_t *o_edge, double *o_x, int64_t *o_M, int32_t *o_trunc, uint64_t *o_k,
              double *o_margin) {
  orc_draws d;
  draws_init(&d, seed, pid, k);
  orc_step_out o = star ? step_star(g, edge, x, dt, &d, cap, reflect_len)
                        : step_general(g, edge, x, dt, &d, cap);
  *o_edge = o.edge; *o_x = o.x; *o_M = o.M; *o_trunc = o.trunc; *o_k = o.k;
  if (o_margin) *o_margin = o.margin;
}

/* Batched single steps from per-row states and streams (the golden em_step
 * rows) with each step's decision margin. */
void orc_step_rows(const orc_graph *g, int32_t star, int64_t n, const int64_t *edge,
                   const double *x, const double *dt, const uint64_t *seed, const uint64_t *pid,
                   const uint64_t *k, const int64_t *cap, const double *reflect_len,
                   int64_t *o_edge, double *o_x, int64_t *o_M, int32_t *o_trunc, uint64_t *o_k,
                   double *o_margin) {
  for (int64_t i = 0; i < n; ++i)
    orc_step(g, star, edge[i], x[i], dt[i], seed[i], pid[i], k[i], cap[i], reflect_len[i],
             o_edge + i, o_x + i, o_M + i, o_trunc + i, o_k + i, o_margin + i);
}

/* Whole trajectories recorded per step (run_ensemble's particles,
 * kernels.py:310-444): after step s of particle i, [i * n_steps + s] holds
 * the edge, position, M, truncation flag, next draw index and the step's
 * decision margin. */
void orc_trace(const orc_graph *g, int32_t star, uint64_t seed, int64_t n_particles,
               int64_t pid_offset, int64_t n_steps, double dt, int32_t init_kind,
               int64_t init_edge, double init_x, double init_xmax, int64_t cap,
               double reflect_len, int64_t *t_edge, double *t_x, int64_t *t_M, int32_t *t_trunc,
               uint64_t *t_k, double *t_margin, int32_t n_threads);

/* kernels.py:291-307 */
static void place(const orc_graph *g, uint64_t seed, uint64_t pid, int32_t init_kind,
                  int64_t init_edge, double init_x, double init_xmax, int64_t *edge,
                  double *x, uint64_t *k) {
  if (init_kind == INIT_POINT) {
    *edge = init_edge; *x = init_x; *k = 0;
    return;
  }
  double u = orc_u64_to_uniform(orc_raw64(seed, pid, 0));
  int64_t m = g->n_edges;
  int64_t e = (int64_t)(u * (double)m);
  if (e >= m) e = m - 1;
  double u2 = orc_u64_to_uniform(orc_raw64(seed, pid, 1));
  double span = init_xmax;
  if (g->edge_len[e] < span) span = g->edge_len[e];
  *edge = e; *x = u2 * span; *k = 2;
}

/* kernels.py:310-444: ensembles; m_hist is [n_chunks][cap+1] like the reference */
void orc_ensemble(const orc_graph *g, int32_t star, uint64_t seed, int64_t n_particles,
                  int64_t pid_offset, int64_t n_steps, double dt, int32_t init_kind,
                  int64_t init_edge, double init_x, double init_xmax, int64_t cap,
                  double reflect_len, int64_t *out_edge, double *out_x, int64_t *out_cross,
                  int64_t *out_events, int64_t *out_trunc, int64_t *m_hist, int32_t n_threads) {
  int64_t n_chunks = (n_particles + ORC_CHUNK - 1) / ORC_CHUNK;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t c = 0; c < n_chunks; ++c) {
    int64_t lo = c * ORC_CHUNK, hi = lo + ORC_CHUNK;
    if (hi > n_particles) hi = n_particles;
    int64_t *row = m_hist + c * (cap + 1);
    for (int64_t i = lo; i < hi; ++i) {
      uint64_t pid = (uint64_t)(i + pid_offset);
      int64_t edge;
      double x;
      uint64_t k;
      place(g, seed, pid, init_kind, init_edge, init_x, init_xmax, &edge, &x, &k);
      orc_draws d;
      draws_init(&d, seed, pid, k);
      int64_t cross = 0, events = 0, truncs = 0;
      for (int64_t s = 0; s < n_steps; ++s) {
        orc_step_out o = star ? step_star(g, edge, x, dt, &d, cap, reflect_len)
                              : step_general(g, edge, x, dt, &d, cap);
        edge = o.edge; x = o.x;
        if (o.M > 0) {
          cross += o.M;
          events += 1;
          row[o.M > cap ? cap : o.M] += 1;
          if (o.trunc) truncs += 1;
        }
      }
      if (out_edge) out_edge[i] = edge;
      if (out_x) out_x[i] = x;
      if (out_cross) out_cross[i] = cross;
      if (out_events) out_events[i] = events;
      if (out_trunc) out_trunc[i] = truncs;
    }
  }
}

void orc_trace(const orc_graph *g, int32_t star, uint64_t seed, int64_t n_particles,
               int64_t pid_offset, int64_t n_steps, double dt, int32_t init_kind,
               int64_t init_edge, double init_x, double init_xmax, int64_t cap,
               double reflect_len, int64_t *t_edge, double *t_x, int64_t *t_M, int32_t *t_trunc,
               uint64_t *t_k, double *t_margin, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t i = 0; i < n_particles; ++i) {
    uint64_t pid = (uint64_t)(i + pid_offset);
    int64_t edge;
    double x;
    uint64_t k;
    place(g, seed, pid, init_kind, init_edge, init_x, init_xmax, &edge, &x, &k);
    orc_draws d;
    draws_init(&d, seed, pid, k);
    for (int64_t s = 0; s < n_steps; ++s) {
      orc_step_out o = star ? step_star(g, edge, x, dt, &d, cap, reflect_len)
                            : step_general(g, edge, x, dt, &d, cap);
      edge = o.edge; x = o.x;
      const int64_t j = i * n_steps + s;
      t_edge[j] = edge; t_x[j] = x; t_M[j] = o.M; t_trunc[j] = o.trunc; t_k[j] = o.k;
      t_margin[j] = o.margin;
    }
  }
}

/* Time-integrated occupation histogram (the
 * reference only snapshots, analysis.py:61-79): the ensemble loop of
 * kernels.py:310-444 with (edge, x) binned exactly like histogram_accumulate
 * after every `every`-th step beyond step `start`. */
void orc_ensemble_occupation(const orc_graph *g, int32_t star, uint64_t seed,
                             int64_t n_particles, int64_t pid_offset, int64_t n_steps, double dt,
                             int32_t init_kind, int64_t init_edge, double init_x,
                             double init_xmax, int64_t cap, double reflect_len,
                             const int64_t *offsets, const int64_t *counts, const double *dx,
                             int64_t every, int64_t start, int64_t *occ, int32_t n_threads) {
  int64_t n_cells = offsets[g->n_edges];
  int64_t n_chunks = (n_particles + ORC_CHUNK - 1) / ORC_CHUNK;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel
#endif
  {
    int64_t *loc = calloc((size_t)n_cells, sizeof(int64_t));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t c = 0; c < n_chunks; ++c) {
      int64_t lo = c * ORC_CHUNK, hi = lo + ORC_CHUNK;
      if (hi > n_particles) hi = n_particles;
      for (int64_t i = lo; i < hi; ++i) {
        uint64_t pid = (uint64_t)(i + pid_offset);
        int64_t edge;
        double x;
        uint64_t k;
        place(g, seed, pid, init_kind, init_edge, init_x, init_xmax, &edge, &x, &k);
        orc_draws d;
        draws_init(&d, seed, pid, k);
        for (int64_t s = 0; s < n_steps; ++s) {
          orc_step_out o = star ? step_star(g, edge, x, dt, &d, cap, reflect_len)
                                : step_general(g, edge, x, dt, &d, cap);
          edge = o.edge; x = o.x;
          int64_t kk = s + 1 - start;
          if (kk > 0 && kk % every == 0) orc_histogram(1, &edge, &x, offsets, counts, dx, loc);
        }
      }
    }
#ifdef _OPENMP
#pragma omp critical
#endif
    for (int64_t j = 0; j < n_cells; ++j) occ[j] += loc[j];
    free(loc);
  }
}

/* kernels.py:447-521: one macro step per trial from the vertex, fresh stream */
void orc_vertex_trials(const orc_graph *g, int32_t star, uint64_t seed, int64_t n_trials,
                       int64_t trial_offset, double dt, int64_t start_edge, double start_x,
                       int64_t cap, int64_t *out_M, int64_t *out_edge, double *out_x,
                       int64_t *out_trunc, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(static, 4096)
#endif
  for (int64_t i = 0; i < n_trials; ++i) {
    uint64_t pid = (uint64_t)(i + trial_offset);
    orc_draws d;
    draws_init(&d, seed, pid, 0);
    orc_step_out o = star ? step_star(g, 0, 0.0, dt, &d, cap, 0.0)
                          : step_general(g, start_edge, start_x, dt, &d, cap);
    if (out_M) out_M[i] = o.M;
    if (out_edge) out_edge[i] = o.edge;
    if (out_x) out_x[i] = o.x;
    if (out_trunc) out_trunc[i] = o.trunc;
  }
}

/* analysis.py:61-79: floor(x/dx[e]) clipped to [0, counts[e]-1], bincount */
void orc_histogram(int64_t n, const int64_t *edges, const double *x, const int64_t *offsets,
                   const int64_t *counts, const double *dx, int64_t *hist) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t e = edges[i];
    double f = floor(x[i] / dx[e]);
    int64_t local = (int64_t)f;
    if (local < 0) local = 0;
    if (local > counts[e] - 1) local = counts[e] - 1;
    hist[offsets[e] + local] += 1;
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Injected-draw arrays for the INJECT parity mode: row i holds the
 * reference stream's draws k0 .. k0+K-1 of particle pid0+i, as raw 64-bit
 * words and as reference normals (rng.py:45-66, :137-143). */
void orc_fill_draws(uint64_t seed, uint64_t pid0, int64_t n, uint64_t k0, int64_t K,
                    uint64_t *raw, double *nrm, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < K; ++j) {
      uint64_t r = orc_raw64(seed, pid0 + (uint64_t)i, k0 + (uint64_t)j);
      raw[i * K + j] = r;
      nrm[i * K + j] = orc_u64_to_normal(r);
    }
  }
}

/* Same for per-row (seed, pid, k0) triples (per-step parity). */
void orc_fill_draws_rows(const uint64_t *seed, const uint64_t *pid, const uint64_t *k0,
                         int64_t n, int64_t K, uint64_t *raw, double *nrm) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < K; ++j) {
      uint64_t r = orc_raw64(seed[i], pid[i], k0[i] + (uint64_t)j);
      raw[i * K + j] = r;
      nrm[i * K + j] = orc_u64_to_normal(r);
    }
}

/* Finite-volume Fokker-Planck stepper: restatement of _fvm_step_loop
 * (fvm.py:254-340) over the packed arrays of _pack_static (fvm.py:343-382).
 * Explicit Euler, upwind drift + central diffusion on interior faces, then
 * the pairwise vertex exchange; rho updated in place.  Returns the 1-based
 * step at which min(0, min rho) < neg_floor * max(1, max |rho|), 0 if none
 * (the state is left at that step, like the reference). */
int64_t orc_fvm_steps(double *rho, int64_t n_cells, int64_t n_steps, double dt,
                      const int64_t *offs, int64_t n_edges, const double *dx_edge,
                      const double *D_edge, const double *face_mu, const int64_t *face_off,
                      const int64_t *v_off, int64_t n_vertices, const int64_t *v_cells,
                      const double *v_b, const double *v_dx, const double *v_speed_in,
                      const double *v_D, double neg_floor) {
  double *nw = (double *)malloc((size_t)(n_cells > 0 ? n_cells : 1) * sizeof(double));
  int64_t result = 0;
  for (int64_t step = 0; step < n_steps && !result; ++step) {
    for (int64_t i = 0; i < n_cells; ++i) nw[i] = rho[i];
    for (int64_t e = 0; e < n_edges; ++e) { /* interior faces, fvm.py:282-295 */
      const int64_t lo = offs[e], hi = offs[e + 1];
      const double dx = dx_edge[e], D = D_edge[e], scale = dt / dx;
      for (int64_t j = lo + 1; j < hi; ++j) {
        const double mu = face_mu[face_off[e] + (j - lo - 1)];
        double F = mu > 0.0 ? mu * rho[j - 1] : mu * rho[j];
        F -= D * (rho[j] - rho[j - 1]) / dx;
        nw[j] += scale * F;
        nw[j - 1] -= scale * F;
      }
    }
    for (int64_t v = 0; v < n_vertices; ++v) { /* vertex exchange, fvm.py:296-328 */
      const int64_t lo = v_off[v], hi = v_off[v + 1];
      if (hi - lo < 2) continue;
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t ci = v_cells[i];
        const double bi = v_b[i], rho_i = rho[ci];
        if (v_speed_in[i] > 0.0) {
          const double others = 1.0 - bi;
          if (others > 0.0) {
            const double total = v_speed_in[i] * rho_i;
            for (int64_t j = lo; j < hi; ++j) {
              if (j == i) continue;
              const double f = total * v_b[j] / others;
              nw[v_cells[j]] += dt * f / v_dx[j];
              nw[ci] -= dt * f / v_dx[i];
            }
          }
        }
        const double conc_i = rho_i / bi;
        for (int64_t j = i + 1; j < hi; ++j) {
          const int64_t cj = v_cells[j];
          const double dpair = 0.5 * (v_D[i] + v_D[j]);
          const double dxh = 2.0 * v_dx[i] * v_dx[j] / (v_dx[i] + v_dx[j]);
          const double g = dpair * (conc_i - rho[cj] / v_b[j]) / dxh;
          if (g >= 0.0) {
            const double f = g * v_b[j];
            nw[cj] += dt * f / v_dx[j];
            nw[ci] -= dt * f / v_dx[i];
          } else {
            const double f = -g * v_b[i];
            nw[ci] += dt * f / v_dx[i];
            nw[cj] -= dt * f / v_dx[j];
          }
        }
      }
    }
    double mx = 1.0, mn = 0.0; /* fvm.py:329-337 */
    for (int64_t i = 0; i < n_cells; ++i) {
      rho[i] = nw[i];
      const double a = fabs(rho[i]);
      if (a > mx) mx = a;
      if (rho[i] < mn) mn = rho[i];
    }
    if (mn < neg_floor * mx) result = step + 1;
  }
  free(nw);
  return result;
}
