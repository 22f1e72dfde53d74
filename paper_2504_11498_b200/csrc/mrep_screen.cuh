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

// The same lower bound from the float copy of the box, on the FP32 pipe.
// The float box encloses the double box and q is rounded to float once per
// lane (FQ); every axis gap is shrunk by m = 6e-7 * scale (scale >= |q|
// and every box coordinate), more than the float roundings of q and of the
// subtraction can add, and the sum by 1e-6 relative -- so the result never
// exceeds the exact squared distance: a box it prunes is also pruned by
// box_lb2.  Tables/queries near the float range use box_lb2 (fbox_ok).
template <int D>
struct FQ {
  float lo[D], hi[D];  // q + m and q - m in float
};

template <int D>
__device__ __forceinline__ FQ<D> make_fq(const double (&q)[D], double scale) {
  FQ<D> f;
  const float m = (float)(6e-7 * scale);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float qf = __double2float_rn(q[k]);
    f.lo[k] = qf + m;
    f.hi[k] = qf - m;
  }
  return f;
}

template <int D>
__device__ __forceinline__ double box_lb2f(const TableView& T, int64_t box, const FQ<D>& f) {
  const float* b = T.fbox + box * 6;
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float g = fmaxf(0.0f, fmaxf(__ldg(b + k) - f.lo[k], f.hi[k] - __ldg(b + 3 + k)));
    acc += g * g;
  }
  return (double)acc * (1.0 - 1e-6);
}

// float copy of n boxes: lo rounded down, hi rounded up (encloses the box)
static __global__ void boxes_to_float_kernel(const double* box, float* fbox, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    fbox[i * 6 + k] = __double2float_rd(box[i * 6 + k]);
    fbox[i * 6 + 3 + k] = __double2float_ru(box[i * 6 + 3 + k]);
  }
}

// float boxes are usable while every coordinate stays far inside float range
__device__ __forceinline__ bool fbox_ok(double scale) { return scale < 1e15; }

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
