// mrep_screen.cuh -- device helpers shared by the curve and surface
// projection pipelines: AABB lower bounds against the table's hierarchy,
// the exact cut-off radius, warp-aggregated append slots and counters.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "mrep_common.cuh"

namespace mrep {

template <int D>
__device__ __forceinline__ double box_lb2(const TableView& T, int64_t box, const double (&q)[D]) {
  const double* b = T.box + box * 6;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double g = fmax(0.0, fmax(__ldg(b + k) - q[k], q[k] - __ldg(b + 3 + k)));
    acc += g * g;
  }
  return acc;
}

// Cut-off radius: a box whose lower bound exceeds it cannot hold a candidate
// inside dmin + 1e-12 (margins cover rounding of the box bound and of the
// foot-point evaluation; they only ever keep extra work).
__device__ __forceinline__ double cut2(double dmin, double scale) {
  double c = dmin * (1.0 + 1e-7) + 1e-11 + 1e-13 * scale;
  return c * c;
}

__device__ __forceinline__ void warp_count(uint64_t* counters, int slot, uint64_t v) {
  if (!counters) return;
  unsigned lo = (unsigned)(v & 0xffffffffu), hi = (unsigned)(v >> 32);
  unsigned mask = __activemask();
  unsigned slo = __reduce_add_sync(mask, lo);
  unsigned shi = __reduce_add_sync(mask, hi);
  int leader = __ffs(mask) - 1;
  if ((threadIdx.x & 31) == leader)
    atomicAdd((unsigned long long*)&counters[slot], (unsigned long long)slo +
                                                        ((unsigned long long)shi << 32));
}

// warp-aggregated slot allocation (works in divergent code)
__device__ __forceinline__ unsigned long long wave_append(unsigned long long* counter, bool want) {
  unsigned act = __activemask();
  unsigned bal = __ballot_sync(act, want);
  if (!bal) return ~0ull;
  int leader = __ffs(bal) - 1;
  unsigned long long base = 0;
  if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(counter, (unsigned long long)__popc(bal));
  base = __shfl_sync(act, base, leader);
  return want ? base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1)) : ~0ull;
}

__device__ __forceinline__ unsigned long long tkey_of(double t) {
  if (t == 0.0) t = 0.0;  // -0.0 and +0.0 compare equal in the reference
  unsigned long long b = (unsigned long long)__double_as_longlong(t);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

}  // namespace mrep
