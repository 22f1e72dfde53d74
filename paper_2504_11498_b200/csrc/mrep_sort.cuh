// mrep_sort.cuh -- query ordering for warp coherence: a counting sort of the
// queries by the Morton code of their bucket in a uniform grid over the
// table's root box (+10% each side, outside queries clamped to the border
// buckets).  Only locality matters here (every result is independent of the
// query order: tests/test_gpu_project.py sorted-vs-unsorted), so queries of
// one bucket keep no particular order.  Three kernels (keys + histogram,
// scan, scatter) instead of the 5-kernel 24-bit radix sort: the fixed cost
// per projection call drops from ~60 us to ~15 us, which is what chunked
// host pipelines pay per chunk.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include <cub/cub.cuh>

#include "mrep_common.cuh"

namespace mrep {

// bits per axis: ~2 queries per bucket, between 2^12 and 2^18 buckets
inline int bucket_bits(int64_t n, int D) {
  int lg = 0;
  while (lg < 40 && ((int64_t)1 << (lg + 1)) <= n) ++lg;  // floor(log2 n)
  int b = (lg - 1 + D / 2) / D;
  static const int hi3 = [] {
    const char* e = getenv("MREP_BUCKET_MAX");  // A/B: finest bits per axis (3-D)
    const int v = e ? atoi(e) : 6;
    return v < 4 ? 4 : (v > 9 ? 9 : v);
  }();
  const int lo = D == 3 ? 4 : 6, hi = D == 3 ? hi3 : 9;
  return b < lo ? lo : (b > hi ? hi : b);
}

// spread the low 10 bits of x to every third (D = 3) / second (D = 2) bit
__device__ __forceinline__ uint32_t spread_bits(uint32_t x, int D) {
  if (D == 3) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
  }
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// Only locality matters here (any order gives the same results), so the
// bucket coordinates are computed in float with a reciprocal, and the Morton
// interleave is the constant bit spread: the kernel was instruction-bound on
// three FP64 divisions and a bit-by-bit loop per query (16 us per 10^6).
template <int D>
__global__ void bucket_key_kernel(const double* __restrict__ q, int64_t n,
                                  const double* __restrict__ root, int bits,
                                  uint32_t* __restrict__ key, int32_t* __restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t G = 1u << bits;
  uint32_t code = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double lo = root[k], hi = root[3 + k];
    const double ext = fmax(hi - lo, 1e-300);
    const float inv = __frcp_rn((float)(1.2 * ext)) * (float)G;
    float u = (float)(q[i * D + k] - (lo - 0.1 * ext)) * inv;
    u = fminf(fmaxf(u, 0.0f), (float)(G - 1));  // NaN -> 0
    code |= spread_bits((uint32_t)u, D) << k;
  }
  key[i] = code;
  atomicAdd(cnt + code, 1);
}

static __global__ void bucket_scatter_kernel(const uint32_t* __restrict__ key, int64_t n,
                                      int32_t* __restrict__ off, uint32_t* __restrict__ perm,
                                      uint32_t* __restrict__ inv) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t pos = atomicAdd(off + key[i], 1);
  perm[pos] = (uint32_t)i;
  if (inv) inv[i] = (uint32_t)pos;  // caller -> sorted position (coalesced)
}

// workspace bytes of bucket_sort for n queries in D dimensions
inline size_t bucket_sort_bytes(int64_t n, int D) {
  const int64_t B = (int64_t)1 << (bucket_bits(n, D) * D);
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (const int32_t*)nullptr, (int32_t*)nullptr, (int)B);
  return 4 * (size_t)n + 8 * (size_t)B + scan + 1024;
}

// perm[j] = the query at sorted position j (device, n entries)
inline int bucket_sort(const double* q, int64_t n, int D, const double* root, void* ws,
                       size_t ws_bytes, uint32_t* perm, cudaStream_t st,
                       uint32_t* inv = nullptr) {
  const int bits = bucket_bits(n, D);
  const int64_t B = (int64_t)1 << (bits * D);
  char* p = (char*)ws;
  auto take = [&](size_t b) {
    char* r = p;
    p += (b + 255) & ~(size_t)255;
    return r;
  };
  uint32_t* key = (uint32_t*)take(4 * (size_t)n);
  int32_t* cnt = (int32_t*)take(4 * (size_t)B);
  int32_t* off = (int32_t*)take(4 * (size_t)B);
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, cnt, off, (int)B, st);
  void* tmp = take(scan);
  if ((size_t)(p - (char*)ws) > ws_bytes) {
    set_error("bucket_sort: workspace too small");
    return MREP_ERR_ARG;
  }
  MREP_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 4 * (size_t)B, st));
  if (D == 3)
    bucket_key_kernel<3><<<grid_for(n, 256), 256, 0, st>>>(q, n, root, bits, key, cnt);
  else
    bucket_key_kernel<2><<<grid_for(n, 256), 256, 0, st>>>(q, n, root, bits, key, cnt);
  MREP_LAUNCH_CHECK();
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, scan, cnt, off, (int)B, st));
  bucket_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(key, n, off, perm, inv);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

}  // namespace mrep
