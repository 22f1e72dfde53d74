// mrep_peak.cu -- FP64 FMA throughput probe (the roofline denominator for the
// FP64-bound projection solve; MEASURED_PEAKS.json carries no FP64 figure).
// 8 independent DFMA chains per thread, 148 x 8 blocks of 256 threads.
#include <cuda_runtime.h>

#include "mrep_common.cuh"

namespace mrep {
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// FP64 tensor-core probe: 8 independent m8n8k4 accumulation chains per warp
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace mrep

using namespace mrep;

// measured FP64 tensor-core (DMMA m8n8k4) throughput, TFLOP/s: the roofline
// denominator of the exact-cand sign screen (mrep_cand.cuh)
extern "C" MREP_API int mrep_dmma_peak(double* tflops) {
  int dev = 0, sms = 0;
  MREP_CUDA_CHECK(cudaGetDevice(&dev));
  MREP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&out, sizeof(double)));
  const int iters = 1 << 12, threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  MREP_CUDA_CHECK(cudaEventCreate(&e0));
  MREP_CUDA_CHECK(cudaEventCreate(&e1));
  dmma_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    MREP_CUDA_CHECK(cudaEventRecord(e0));
    dmma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    MREP_CUDA_CHECK(cudaEventRecord(e1));
    MREP_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    MREP_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  MREP_LAUNCH_CHECK();
  // per warp and MMA: 8 x 8 x 4 multiply-adds
  double flops = 2.0 * 256.0 * 8.0 * iters * (double)(threads / 32) * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return MREP_OK;
}

extern "C" MREP_API int mrep_fp64_peak(double* tflops) {
  int dev = 0, sms = 0;
  MREP_CUDA_CHECK(cudaGetDevice(&dev));
  MREP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&out, sizeof(double)));
  const int iters = 1 << 14, threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  MREP_CUDA_CHECK(cudaEventCreate(&e0));
  MREP_CUDA_CHECK(cudaEventCreate(&e1));
  dfma_kernel<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    MREP_CUDA_CHECK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    MREP_CUDA_CHECK(cudaEventRecord(e1));
    MREP_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    MREP_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  MREP_LAUNCH_CHECK();
  double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return MREP_OK;
}
