/*
 * gsde.h -- C ABI of the B200-native graph-SDE simulator (libgsde.so).
 *
 * Drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/graphsde).  Every entry point names the reference
 * interface it replaces.  Plain pointers and sizes only; "device" pointers
 * are CUDA device memory (e.g. torch tensors' data_ptr()), "stream" is a
 * cudaStream_t passed as void*.  All calls are stream-ordered and re-entrant;
 * the library never frees caller memory.  Return 0 on success, a negative
 * GSDE_E* code otherwise (message via gsde_last_error()).  Argument
 * validation with the reference's exception types happens in the Python
 * host layer before dispatch; the library re-checks what it relies on.
 */
#ifndef GSDE_H
#define GSDE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSDE_ABI_VERSION 3

enum {
  GSDE_OK = 0,
  GSDE_EINVAL = -1,  /* bad argument */
  GSDE_ECUDA = -2,   /* CUDA runtime / launch failure */
  GSDE_ENOMEM = -3,  /* device allocation failed */
  GSDE_ENODEV = -4,  /* no usable sm_100 device */
};

/* Random-stream modes.
 *  REFERENCE: the reference's own streams -- Philox4x32-10 keyed
 *             (seed, particle, draw index) exactly as rng.py:45-66, AS241
 *             normals (rng.py:81-143), FP64 arithmetic, inverse-CDF exit
 *             slots (kernels.py:134-143).  Bit-compatible edge ids / M.
 *  INJECT:    draws supplied by the caller per (particle, draw index) --
 *             raw 64-bit words for uniforms, reference normals for Gaussians
 *             -- arithmetic in FP32 or FP64 (`precision`).
 *  NATIVE:    the B200 production stream -- FP32, Philox4x32-10 feeding
 *             Box-Muller Gaussians per proposal and 32-bit uniforms per vertex
 *             slot, alias tables for exit slots, flattened per-lane state
 *             machine in 14-proposal iterations.
 *             Statistically equivalent, not bit-identical, to REFERENCE. */
enum { GSDE_STREAM_NATIVE = 0, GSDE_STREAM_REFERENCE = 1, GSDE_STREAM_INJECT = 2 };
/* INJECT precisions: F32 / F64 run the reference-order stepper (gsde_ref.cu)
 * in that precision; NATIVE runs the production FP32 kernel itself (the
 * NATIVE stream's kernel with each proposal's normal and each exit uniform
 * taken from the injected rows in the reference's order, exit slots by the
 * reference's inverse CDF): ensembles (without the occupation histogram)
 * and vertex trials. */
enum { GSDE_PREC_F32 = 0, GSDE_PREC_F64 = 1, GSDE_PREC_NATIVE = 2 };

/* Initial placement codes (kernels.py:48-50), plus per-particle state-in:
 * GSDE_INIT_STATE takes particle i's (edge, x) from the SoA device arrays
 * state_edge / state_x of the run arguments (read coalesced, a warp's 32 particles
 * per refill) -- the batched form of em_step_*'s ParticleState
 * (engine.py:60-67, :206-270) and the resume point of a checkpointed run.
 * NATIVE and INJECT/NATIVE streams only; the caller guarantees
 * 0 <= edge < n_edges and 0 <= x <= length (x > 0 on a star edge unless at
 * the vertex). */
enum { GSDE_INIT_POINT = 0, GSDE_INIT_PER_EDGE_UNIFORM = 1, GSDE_INIT_STATE = 2 };

typedef struct gsde_graph_s gsde_graph; /* opaque, device-resident graph + field */

/* Packed graph + coefficient field in the reference's own layout and dtypes
 * (HOST memory): MetricGraph packed arrays graph.py:102-125 and
 * CoefficientField.packed() coefficients.py:121-152. */
typedef struct {
  int64_t n_edges, n_vertices, n_tab;
  const double *edge_length; /* [E] inf = semi-infinite */
  const int64_t *edge_init;  /* [E] */
  const int64_t *edge_term;  /* [E] -1 = vertex at infinity */
  const int64_t *v_off;      /* [V+1] CSR over finite vertices */
  const int64_t *v_edges;    /* [S] incident edge per slot (edge-id order) */
  const int8_t *v_orient;    /* [S] 0 = vertex at init, 1 = at term */
  const double *v_cumw;      /* [S] cumulative jump weights */
  const double *v_weights;   /* [S] jump weights (native alias tables) */
  const int8_t *dkind;       /* [E] 0 constant, 1 linear, 2 tabulated */
  const double *dcoef;       /* [E] */
  const int64_t *tab_off;    /* [E+1] */
  const double *tab_x;       /* [T] */
  const double *tab_mu;      /* [T] */
  const double *sigma;       /* [E] */
  int32_t is_star;           /* graph.py:254-258 */
} gsde_graph_desc;

/* Upload a graph + field to `device` (one-time; replaces the per-call
 * field.packed() / graph arrays handed to the numba kernels,
 * engine.py:304-328).  Builds FP32 copies, 53-bit integer slot thresholds and
 * per-vertex alias tables on the host, then copies once. */
int gsde_graph_create(const gsde_graph_desc *desc, int device, gsde_graph **out);
int gsde_graph_destroy(gsde_graph *g);
/* Device bytes held by the handle. */
int64_t gsde_graph_device_bytes(const gsde_graph *g);

/* Ensemble run parameters (kernels.py:310-444 arguments). */
typedef struct {
  uint64_t seed;
  int64_t n_particles;  /* particles handled by this call */
  int64_t pid_offset;   /* global id of this call's first particle (sharding) */
  int64_t n_steps;
  double dt;
  int32_t init_kind;    /* GSDE_INIT_* */
  int64_t init_edge;
  double init_x, init_xmax;
  int32_t cap;          /* max_splits_per_step */
  double reflect_len;   /* star mirror wall, 0 = off (engine.py:111-112) */
  int32_t stream;       /* GSDE_STREAM_* */
  int32_t precision;    /* GSDE_PREC_* (INJECT only; REFERENCE = F64, NATIVE = F32) */
  const uint64_t *inj_raw;    /* device [n_particles][inj_stride] */
  const double *inj_normal;   /* device [n_particles][inj_stride] */
  int64_t inj_stride;
  /* GSDE_INIT_STATE (device, [n_particles]): edge ids, positions, and for the
   * NATIVE stream optionally each particle's next Philox block (NULL = 0) --
   * gsde_out.counter of the run being resumed */
  const int32_t *state_edge;
  const float *state_x;
  const uint64_t *state_counter;
} gsde_run;

/* Ensemble outputs: device pointers, each optional (NULL = skip).  Per-particle
 * arrays use the reference dtypes (engine.py:296-300).  Reductions are
 * ACCUMULATED (+=) so shards / repeated calls merge; zero them first. */
typedef struct {
  int64_t *edge, *crossings, *events, *truncs; /* [n_particles] */
  double *x;                                    /* [n_particles] */
  int64_t *m_hist;      /* [cap+1] steps with M>0 by M (kernels.py:361-369) */
  int64_t *totals;      /* [4] crossings, events, truncations, inject overruns */
  int64_t *edge_counts; /* [E] final-edge occupancy */
  int64_t *hist;        /* [n_cells] snapshot histogram of final positions */
  const int64_t *hist_offsets; /* device [E+1]  (EdgeGrid.offsets) */
  const int64_t *hist_counts;  /* device [E]    (EdgeGrid.counts) */
  const double *hist_dx;       /* device [E]    (EdgeGrid.dx) */
  int64_t hist_n_cells;
  /* Time-integrated occupation histogram on the same grid: after every
   * occ_every-th completed macro step beyond step occ_start, each particle's
   * (edge, x) is binned into occ (accumulated).  Requires the hist grid
   * arrays; occ may be used with hist == NULL. */
  int64_t *occ;                /* [n_cells] */
  int64_t occ_every;           /* >= 1 */
  int64_t occ_start;           /* steps before the first sample (burn-in) */
  /* [n_particles]: NATIVE -- the particle's next unused Philox block (resume
   * with GSDE_INIT_STATE + state_counter); INJECT/NATIVE -- the number of
   * injected draws the particle consumed (the reference's RngStream.counter
   * advance, engine.py:228) */
  uint64_t *counter;
  /* Streamed results (optional; per-particle arrays asked for): the kernel
   * adds 1 to progress[(progress_base + i) >> progress_shift] after particle
   * i's per-particle outputs are stored (release order, GPU scope), so a copy
   * stream can wait for a particle-id range (gsde_stream_wait_geq32) and move
   * it to the host while the launch still runs.  Counters are accumulated:
   * zero them first.  (No reference counterpart: the reference returns
   * host arrays once the whole run has finished, engine.py:338-352.) */
  uint32_t *progress;
  int64_t progress_base;
  int32_t progress_shift;
} gsde_out;

/* run_ensemble's kernel call: kernels.ensemble_star / ensemble_general
 * (engine.py:309-328).  n_steps == 0 performs placement only
 * (engine.py:329-336). */
int gsde_ensemble(const gsde_graph *g, const gsde_run *run, const gsde_out *out, void *stream);

/* Make `stream` wait until the 32-bit word at device address `addr` is >=
 * `value` (cuStreamWaitValue32, GEQ) -- the consumer side of gsde_out's
 * progress counters.  Returns GSDE_OK, or an error when the driver has no
 * stream memory operations (callers then wait for the whole launch). */
int gsde_stream_wait_geq32(void *stream, const uint32_t *addr, uint32_t value);

/* Vertex-trial parameters (kernels.py:447-521 arguments). */
typedef struct {
  uint64_t seed;
  int64_t n_trials;
  int64_t trial_offset; /* global id of this call's first trial (sharding) */
  double dt;
  int64_t start_edge;   /* general graphs: first slot of the start vertex */
  double start_x;
  int32_t cap;
  int32_t stream;
  int32_t precision;
  const uint64_t *inj_raw;
  const double *inj_normal;
  int64_t inj_stride;
} gsde_trials;

/* Trial outputs (device, optional).  exit_counts / m_hist / totals are the
 * fused estimator for exit_probability_experiment (analysis.py:348-384): no
 * per-trial arrays need to exist. m_hist here includes M = 0 (engine.py:379-388). */
typedef struct {
  int64_t *M, *edge, *trunc; /* [n_trials] */
  double *x;                 /* [n_trials] */
  int64_t *exit_counts;      /* [E] */
  int64_t *m_hist;           /* [cap+1] */
  int64_t *totals;           /* [4] sum M, #(M>0), truncations, inject overruns */
} gsde_trials_out;

/* vertex_crossing_trials' kernel call: kernels.vertex_trials_star /
 * vertex_trials_general (engine.py:411-433). */
int gsde_vertex_trials(const gsde_graph *g, const gsde_trials *tr, const gsde_trials_out *out,
                       void *stream);

/* Batched single macro steps (em_step_star / em_step_general,
 * engine.py:206-270 -> kernels.step_star / step_general, kernels.py:146-288).
 * Per particle i: state (edge[i], x[i]) advanced by dt using stream
 * (seed[i], pid[i]) from draw index k[i] (REFERENCE) or injected draws.
 * edge, x, k are updated in place; M, trunc written.  All device pointers. */
typedef struct {
  int64_t n;
  double dt;
  int32_t cap;
  double reflect_len;
  int32_t stream;    /* REFERENCE or INJECT */
  int32_t precision; /* INJECT only */
  const uint64_t *seed, *pid; /* [n] */
  const uint64_t *inj_raw;
  const double *inj_normal;
  int64_t inj_stride;
} gsde_step_args;

int gsde_step_batch(const gsde_graph *g, const gsde_step_args *a, int64_t *edge, double *x,
                    uint64_t *k, int64_t *M, int64_t *trunc, void *stream);

/* Snapshot histogram of (edge, x) samples on an EdgeGrid
 * (histogram_accumulate, analysis.py:61-79): floor(x/dx[e]) clipped to
 * [0, counts[e]-1], accumulated into hist[offsets[e] + local].  Device arrays. */
int gsde_histogram(int64_t n, const int64_t *edge, const double *x, const int64_t *offsets,
                   const int64_t *counts, const double *dx, int64_t n_cells, int64_t *hist,
                   void *stream);

/* Finite-volume Fokker-Planck baseline (fvm.py): the packed static arrays of
 * fvm._pack_static (fvm.py:343-382) re-laid per cell, plus an ownership split
 * of the vertex exchange; all DEVICE pointers.  Cell c of edge e carries the
 * drift on its left / right interior face, D = sigma_e^2 / 2 and dx_e, and
 * flags: bit 0 = has a left interior face, bit 1 = has a right one, bit 2 =
 * vertex-adjacent cell of a vertex of degree >= 2 (that vertex's item
 * updates it).  Vertex v's slots are v_off[v]..v_off[v+1]; pslot lists the
 * slots of the vertices whose cells no other vertex touches (one thread per
 * slot), vser (ascending) the other degree >= 2 vertices (cells shared
 * through single-cell edges), processed in vertex order by one thread. */
typedef struct {
  int64_t n_edges, n_cells, n_vertices, n_pslot, n_vser, n_terms;
  const double *cell_mu_l;   /* [C] drift on the left face (0 if none) */
  const double *cell_mu_r;   /* [C] drift on the right face (0 if none) */
  const double *cell_D;      /* [C] */
  const double *cell_dx;     /* [C] */
  const uint8_t *cell_flags; /* [C] */
  const int64_t *v_off;      /* [V+1] */
  const int64_t *v_cells;    /* [S] vertex-adjacent cell per slot */
  const double *v_b;         /* [S] jump weight */
  const double *v_dx;        /* [S] */
  const double *v_speed_in;  /* [S] inward drift speed (>= 0) */
  const double *v_D;         /* [S] */
  const int64_t *slot_vertex; /* [S] vertex of each slot */
  const int64_t *pslot;      /* [n_pslot] slots of the vertices whose cells no other vertex touches */
  const int64_t *vser;       /* [n_vser] the other degree >= 2 vertices, ascending */
  /* two-phase exchange (fvm._term_layout): cell of pslot[t] sums the signed terms
   * terms[tstart[t] .. tstart[t+1]) in the reference's order; exchange row pslot[t]
   * writes its (j-side, i-side) term pairs to the positions rpos[rstart[t] ..
   * rstart[t+1]) */
  const int64_t *tstart;     /* [n_pslot+1] */
  const int64_t *rstart;     /* [n_pslot+1] */
  const int64_t *rpos;       /* [rstart[n_pslot]] */
  double *terms;             /* [n_terms] device workspace */
} gsde_fvm_desc;

/* fvm_run's stepper (_fvm_step_loop, fvm.py:254-340): n_steps explicit Euler
 * steps of rho (device [n_cells], updated in place; scratch: device
 * [n_cells]) in the reference's floating-point operation order (bit-identical
 * FP64).  After each step the run stops if min(0, min rho) <
 * neg_floor * max(1, max |rho|); *neg_step (device int64) receives the
 * 1-based step index, 0 if none.  red: caller-owned device scratch of 8
 * uint64.  Two kernels per step (exchange terms per vertex slot, then one
 * thread per cell / slot summing them), stream-ordered and replayed from a CUDA
 * graph; the stop test runs in the last block of each step. */
int gsde_fvm_run(const gsde_fvm_desc *d, double *rho, double *scratch, int64_t n_steps,
                 double dt, double neg_floor, int64_t *neg_step, uint64_t *red, void *stream);

/* Native reader for the "metric-graph v1" text format (graphfile.py:69-186),
 * happy path only: returns GSDE_OK and an opaque result, or a nonzero code for
 * any input it does not accept verbatim -- the caller then re-parses with the
 * Python parser, which raises the reference's exact ParseError.  Host-only. */
typedef struct gsde_parsed_s gsde_parsed;
int gsde_parse_graph_text(const char *text, int64_t len, gsde_parsed **out);
/* sizes[7]: vertex declarations, edges, weight directives, weight values,
 * drift directives, tabulated samples, sigma directives */
void gsde_parsed_sizes(const gsde_parsed *p, int64_t *sizes);
void gsde_parsed_export(const gsde_parsed *p, int64_t *vdecl, int64_t *e_id, int64_t *e_init,
                        int64_t *e_term, double *e_len, int64_t *w_vertex, int64_t *w_n,
                        double *w_val, int64_t *d_id, int8_t *d_kind, double *d_a, double *d_b,
                        int64_t *d_tab_n, double *tab_x, double *tab_mu, int64_t *s_id,
                        double *s_val);
void gsde_parsed_free(gsde_parsed *p);

/* Host-side scalar helpers, compiled from the same sources as the kernels. */
uint64_t gsde_raw64(uint64_t seed, uint64_t stream, uint64_t index); /* rng.py:45-66 */
double gsde_uniform01(uint64_t seed, uint64_t stream, uint64_t index); /* rng.py:75-78 */
double gsde_normal(uint64_t seed, uint64_t stream, uint64_t index);    /* rng.py:146-149 */
double gsde_u64_to_uniform(uint64_t r);                                /* rng.py:69-72 */
double gsde_u64_to_normal(uint64_t r);                                 /* rng.py:137-143 */
double gsde_norm_ppf(double p);                                        /* rng.py:81-134 */
double gsde_solve_first_passage_s(double a, double b, double c);     /* kernels.py:88-131 */

/* Number of kernels this library has launched (instrumentation for bench.py). */
int64_t gsde_launch_count(void);
int gsde_abi_version(void);
const char *gsde_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GSDE_H */
