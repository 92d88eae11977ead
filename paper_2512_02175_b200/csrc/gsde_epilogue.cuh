// gsde_epilogue.cuh -- per-particle output / estimator helpers shared by kernels.
#pragma once
#include "gsde_internal.h"

namespace gsde {

__device__ __forceinline__ void add_i64(int64_t *p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}

// Snapshot-histogram cell of (e, x) on an EdgeGrid (analysis.py:75-78):
// floor(x / dx[e]) clipped to [0, counts[e]-1], in FP64 like the reference.
__device__ __forceinline__ int64_t hist_cell(const int64_t *offsets, const int64_t *counts,
                                            const double *dx, int e, double x) {
  const double f = floor(x / dx[e]);
  const int64_t top = counts[e] - 1;
  int64_t local;
  if (!(f > 0.0))
    local = 0;
  else if (f >= (double)top)
    local = top;
  else
    local = (int64_t)f;
  return offsets[e] + local;
}

// Per-particle result arrays of one ensemble particle (kernels.py:370-374).
__device__ __forceinline__ void epilogue_particle(const KOut &o, int64_t i, int e, double x,
                                                  int64_t cross, int64_t events,
                                                  int64_t truncs) {
  if (o.edge) o.edge[i] = e;
  if (o.x) o.x[i] = x;
  if (o.crossings) o.crossings[i] = cross;
  if (o.events) o.events[i] = events;
  if (o.truncs) o.truncs[i] = truncs;
}

// Fused estimators of one final state: final-edge occupancy and the snapshot
// histogram (analysis.py:61-79).
__device__ __forceinline__ void epilogue_bins(const KOut &o, int e, double x) {
  if (o.edge_counts) add_i64(&o.edge_counts[e], 1);
  if (o.hist) add_i64(&o.hist[hist_cell(o.hist_offsets, o.hist_counts, o.hist_dx, e, x)], 1);
}

__device__ __forceinline__ void ensemble_epilogue(const KOut &o, int64_t i, int e, double x,
                                                  int64_t cross, int64_t events,
                                                  int64_t truncs) {
  epilogue_particle(o, i, e, x, cross, events, truncs);
  epilogue_bins(o, e, x);
}

// Block-wide sum of per-thread int64 values, one atomic per warp.
__device__ __forceinline__ void warp_add_i64(int64_t *dst, int64_t v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0 && v != 0) add_i64(dst, v);
}

}  // namespace gsde
