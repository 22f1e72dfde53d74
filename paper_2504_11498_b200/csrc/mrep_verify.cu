// mrep_verify.cu -- the reference's brute-force verification oracle on the
// GPU: oracle_project_batch (/root/reference/pkg/src/splinemat/oracle.py:95-128),
// the dense-grid + ternary-search projection the CLI's --verify runs
// (cli.py:169-182).  It is the slowest step of a verified run in the
// reference; here:
//   * dense scan: thread per query, grid points staged through shared memory
//     in tiles, first index of the minimum squared distance (np.argmin);
//   * ternary search: lock-step iterations over all queries (the reference
//     loops while max(b - a) > 1e-10 over the whole batch), each step one
//     kernel that also reduces the new maximum width for the host's check;
//   * curve points by Cox-de Boor on the p+1 live functions with a binary
//     span search (same values as the reference's full basis table).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "mrep_common.cuh"

namespace mrep {

__device__ void deboor_point(int p, const double* kn, int64_t m, const double* ctrl, int64_t ncp,
                             int d, double t, double* out) {
  // span: the largest j with kn[j] <= t (then kn[j+1] > t: a nonzero span);
  // t == kn[m-1] maps onto the final nonzero span
  int64_t s;
  if (t == kn[m - 1]) {
    s = m - 2;
    while (s > 0 && !(kn[s] < kn[s + 1])) --s;
  } else {
    int64_t lo = 0, hi = m;  // first index with kn[idx] > t
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (kn[mid] <= t) lo = mid + 1;
      else hi = mid;
    }
    s = lo - 1;
  }
  double N[32];
  for (int j = 0; j <= p; ++j) N[j] = 0.0;
  if (s < 0 || s >= m - 1) {
    for (int k = 0; k < d; ++k) out[k] = 0.0;
    return;
  }
  N[p] = 1.0;
  for (int lvl = 1; lvl <= p; ++lvl) {
    for (int j = p - lvl; j <= p; ++j) {
      int64_t b = s - p + j;
      double acc = 0.0;
      double d1 = kn[b + lvl] - kn[b];
      if (d1 > 0.0) acc += (t - kn[b]) / d1 * N[j];
      double d2 = kn[b + lvl + 1] - kn[b + 1];
      if (d2 > 0.0 && j + 1 <= p) acc += (kn[b + lvl + 1] - t) / d2 * N[j + 1];
      N[j] = acc;
    }
  }
  for (int k = 0; k < d; ++k) {
    double acc = 0.0;
    for (int j = 0; j <= p; ++j) {
      int64_t b = s - p + j;
      if (b >= 0 && b < ncp) acc = fma(N[j], ctrl[b * d + k], acc);
    }
    out[k] = acc;
  }
}

// the p + 1 nonzero basis values of every t, written into its row of the
// zero-filled (n, m - 1 - p) matrix (oracle.py:13-42's _basis_rows): same
// span rule and two-term recursion as deboor_point
__global__ void basis_rows_kernel(int p, const double* kn, int64_t m, const double* ts, int64_t n,
                                  double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double t = ts[i];
  const int64_t ncol = m - 1 - p;
  int64_t s;
  if (t == kn[m - 1]) {
    s = m - 2;
    while (s > 0 && !(kn[s] < kn[s + 1])) --s;
  } else {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (kn[mid] <= t) lo = mid + 1;
      else hi = mid;
    }
    s = lo - 1;
  }
  if (s < 0 || s >= m - 1 || !(kn[s] < kn[s + 1])) return;  // outside every half-open span
  double N[32];
  for (int j = 0; j <= p; ++j) N[j] = 0.0;
  N[p] = 1.0;
  for (int lvl = 1; lvl <= p; ++lvl) {
    for (int j = p - lvl; j <= p; ++j) {
      int64_t b = s - p + j;
      double acc = 0.0;
      double d1 = kn[b + lvl] - kn[b];
      if (d1 > 0.0) acc += (t - kn[b]) / d1 * N[j];
      double d2 = kn[b + lvl + 1] - kn[b + 1];
      if (d2 > 0.0 && j + 1 <= p) acc += (kn[b + lvl + 1] - t) / d2 * N[j + 1];
      N[j] = acc;
    }
  }
  for (int j = 0; j <= p; ++j) {
    const int64_t b = s - p + j;
    if (b >= 0 && b < ncol) out[i * ncol + b] = N[j];
  }
}

constexpr int NB_TILE = 512;

__global__ void __launch_bounds__(256) dense_nearest_kernel(const double* pts, int64_t m,
                                                            const double* q, int64_t n, int d,
                                                            int64_t* best) {
  __shared__ double tile[NB_TILE * 3];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double qq[3] = {0.0, 0.0, 0.0};
  if (i < n)
    for (int k = 0; k < d; ++k) qq[k] = q[i * d + k];
  double bd = __longlong_as_double(0x7ff0000000000000LL);
  int64_t bi = 0;
  for (int64_t t0 = 0; t0 < m; t0 += NB_TILE) {
    int64_t cnt = m - t0 < NB_TILE ? m - t0 : NB_TILE;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < cnt * d; j += blockDim.x) tile[j] = pts[t0 * d + j];
    __syncthreads();
    if (i < n) {
      for (int64_t j = 0; j < cnt; ++j) {
        double acc = 0.0;
        for (int k = 0; k < d; ++k) {
          double df = tile[j * d + k] - qq[k];
          acc += df * df;
        }
        if (acc < bd) {  // strict: the first index of the minimum (np.argmin)
          bd = acc;
          bi = t0 + j;
        }
      }
    }
  }
  if (i < n) best[i] = bi;
}

struct TernaryArgs {
  int p, d;
  const double* kn;
  int64_t m;
  const double* ctrl;
  int64_t ncp;
  const double* q;
  int64_t n;
  double* a;
  double* b;
  unsigned long long* maxw;  // bits of the largest b - a after this step
};

__device__ __forceinline__ double qdist(const TernaryArgs& A, int64_t i, double t) {
  double pt[3];
  deboor_point(A.p, A.kn, A.m, A.ctrl, A.ncp, A.d, t, pt);
  double acc = 0.0;
  for (int k = 0; k < A.d; ++k) {
    double df = pt[k] - A.q[i * A.d + k];
    acc += df * df;
  }
  return sqrt(acc);
}

// bracket [ts[best-1], ts[best+1]] (clamped) and the initial max width
__global__ void ternary_init_kernel(TernaryArgs A, const double* ts, int64_t grid,
                                    const int64_t* best) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int64_t bi = best[i];
  A.a[i] = ts[bi > 0 ? bi - 1 : 0];
  A.b[i] = ts[bi + 1 < grid ? bi + 1 : grid - 1];
  atomicMax(A.maxw, (unsigned long long)__double_as_longlong(fmax(A.b[i] - A.a[i], 0.0)));
}

__global__ void ternary_step_kernel(TernaryArgs A) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double a = A.a[i], b = A.b[i];
  double m1 = a + (b - a) / 3.0;
  double m2 = b - (b - a) / 3.0;
  double f1 = qdist(A, i, m1), f2 = qdist(A, i, m2);
  if (f1 < f2) b = m2;
  else a = m1;
  A.a[i] = a;
  A.b[i] = b;
  atomicMax(A.maxw, (unsigned long long)__double_as_longlong(fmax(b - a, 0.0)));
}

__global__ void ternary_final_kernel(TernaryArgs A, double* t_out, double* d_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double tm = 0.5 * (A.a[i] + A.b[i]);
  t_out[i] = tm;
  d_out[i] = qdist(A, i, tm);
}

}  // namespace mrep

using namespace mrep;

extern "C" {

int mrep_oracle_project_batch(int p, const double* knots, int64_t m, const double* ctrl,
                              int64_t ncp, int d, const double* ts, const double* grid_pts,
                              int64_t grid, const double* queries, int64_t n, double* out_t,
                              double* out_dist, void* stream) {
  if (p < 0 || p > 31 || (d != 2 && d != 3) || grid < 2 || n < 0) {
    set_error("mrep_oracle_project_batch: bad arguments");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = nullptr;
  const size_t o_best = 0, o_a = 8 * (size_t)n, o_b = 16 * (size_t)n, o_w = 24 * (size_t)n;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&ws, o_w + 64, st));
  int64_t* best = (int64_t*)(ws + o_best);
  TernaryArgs A{p, d, knots, m, ctrl, ncp, queries, n, (double*)(ws + o_a), (double*)(ws + o_b),
                (unsigned long long*)(ws + o_w)};
  dense_nearest_kernel<<<grid_for(n, 256), 256, 0, st>>>(grid_pts, grid, queries, n, d, best);
  MREP_LAUNCH_CHECK();
  MREP_CUDA_CHECK(cudaMemsetAsync(A.maxw, 0, 8, st));
  ternary_init_kernel<<<grid_for(n, 256), 256, 0, st>>>(A, ts, grid, best);
  MREP_LAUNCH_CHECK();
  for (int it = 0; it < 400; ++it) {
    unsigned long long wbits = 0;
    MREP_CUDA_CHECK(cudaMemcpyAsync(&wbits, A.maxw, 8, cudaMemcpyDeviceToHost, st));
    MREP_CUDA_CHECK(cudaStreamSynchronize(st));
    double w;
    memcpy(&w, &wbits, 8);
    if (!(w > 1e-10)) break;  // while np.max(b - a) > 1e-10 (oracle.py:117)
    MREP_CUDA_CHECK(cudaMemsetAsync(A.maxw, 0, 8, st));
    ternary_step_kernel<<<grid_for(n, 256), 256, 0, st>>>(A);
    MREP_LAUNCH_CHECK();
  }
  ternary_final_kernel<<<grid_for(n, 256), 256, 0, st>>>(A, out_t, out_dist);
  MREP_LAUNCH_CHECK();
  MREP_CUDA_CHECK(cudaFreeAsync(ws, st));
  return MREP_OK;
}

int mrep_basis_rows(int p, const double* knots, int64_t m, const double* ts, int64_t n,
                    double* out, void* stream) {
  if (p < 1 || p > 31 || m < p + 2 || n < 0) {
    set_error("mrep_basis_rows: need 1 <= p <= 31, m >= p + 2, n >= 0");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  basis_rows_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(p, knots, m, ts, n, out);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

}  // extern "C"
