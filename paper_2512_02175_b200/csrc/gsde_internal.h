// gsde_internal.h -- declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/gsde.h"
#include "gsde_core.cuh"

struct gsde_graph_s {
  int device = 0;
  int64_t E = 0, V = 0, S = 0, T = 0;
  bool is_star = false;
  bool has_tab = false;
  bool zero_drift = false;  // every edge driftless (kind 0/1 with coefficient 0)
  bool const_drift = false; // every edge's drift constant in x (kind 0, or kind 1 with 0)
  bool uniform_exits = false; // every alias column keeps its own slot (equal jump weights)
  void *arena = nullptr;
  int64_t arena_bytes = 0;
  gsde::RefGraph<double> ref64{};
  gsde::RefGraph<float> ref32{};
  gsde::NativeGraph nat{};
  // native smem staging size for the whole graph (0 = too large, read via L2)
  int64_t nat_graph_smem = 0;
  // work-distribution counters of the native kernels: a ring of slots in the
  // arena, one per call (zeroed stream-ordered before the launch).  A slot is
  // reused only after the kernel that last used it has finished: each launch
  // records the slot's event, and the next user's stream waits on it before
  // the memset (cheap: a slot comes round again only after kWorkSlots calls).
  static constexpr int kWorkSlots = 64;
  unsigned long long *work = nullptr;
  cudaEvent_t work_done[kWorkSlots] = {};
  std::atomic<uint32_t> work_ticket{0};
  int next_work_slot() { return (int)(work_ticket++ % kWorkSlots); }
};

namespace gsde {

// Kernel-side view of gsde_out: the estimator / output pointers the ensemble
// kernels take by value.  Its layout is deliberately frozen -- the kernel
// parameter layout feeds the register allocator, and growing this struct
// moved the headline kernel from 64 to 67 registers (one CTA per SM fewer).
// Later outputs (the per-particle counter) travel in the kernels' last
// parameter instead.
struct KOut {
  int64_t *edge, *crossings, *events, *truncs;
  double *x;
  int64_t *m_hist, *totals, *edge_counts, *hist;
  const int64_t *hist_offsets, *hist_counts;
  const double *hist_dx;
  int64_t hist_n_cells;
  int64_t *occ;
  int64_t occ_every, occ_start;
};

inline KOut kernel_out(const gsde_out &o) {
  return KOut{o.edge,        o.crossings,   o.events,   o.truncs,       o.x,
              o.m_hist,      o.totals,      o.edge_counts, o.hist,      o.hist_offsets,
              o.hist_counts, o.hist_dx,     o.hist_n_cells, o.occ,      o.occ_every,
              o.occ_start};
}

// Per-call device properties (cached per device).
struct DevInfo {
  int sm_count = 0;
};
DevInfo dev_info(int device);

void count_launch(int n = 1);
int set_error(int code, const char *fmt, ...);

// gsde_ref.cu (FP64 / injected streams; strict IEEE, no FMA contraction)
cudaError_t launch_ref_ensemble(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                cudaStream_t s);
cudaError_t launch_ref_trials(const gsde_graph *g, const gsde_trials &a,
                              const gsde_trials_out &o, cudaStream_t s);
cudaError_t launch_step_batch(const gsde_graph *g, const gsde_step_args &a, int64_t *edge,
                              double *x, uint64_t *k, int64_t *M, int64_t *trunc,
                              cudaStream_t s);

// gsde_native.cu (FP32 production stream)
cudaError_t launch_native_ensemble(const gsde_graph *g, const gsde_run &a, const gsde_out &o,
                                   cudaStream_t s);
cudaError_t launch_native_trials(const gsde_graph *g, const gsde_trials &a,
                                 const gsde_trials_out &o, cudaStream_t s);
// gsde_fvm.cu (finite-volume baseline; strict IEEE, no FMA contraction)
cudaError_t launch_fvm(const gsde_fvm_desc &d, double *rho, double *scratch, int64_t n_steps,
                       double dt, double neg_floor, int64_t *neg_step, uint64_t *red,
                       cudaStream_t s);

cudaError_t launch_histogram(int64_t n, const int64_t *edge, const double *x,
                             const int64_t *offsets, const int64_t *counts, const double *dx,
                             int64_t n_cells, int64_t *hist, cudaStream_t s);

}  // namespace gsde
