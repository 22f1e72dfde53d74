// mrep_prep.cu -- per-curve preprocessing on the GPU: B-spline -> Bezier
// decomposition and error-controlled G1 cubic approximation, batched over
// many curves, plus curve / Bezier evaluation.
//
// Replaces (reference = /root/reference/pkg/src/splinemat):
//   decompose.py:19-67        decompose_to_bezier / batched_decompose
//   basis.py:110-149           symbolic_basis_matrix (per-span Cox-de Boor)
//   reduce_approx.py:60-301    G1 reduction, elevation, max-error check,
//                              restriction, level-synchronous subdivision
//   oracle.py:13-52            eval_de_boor_many (curve evaluation)
//   core.py:248-258            eval_bezier
//
// Mapping: one warp per span (decomposition; lanes = polynomial coefficient
// index, p + 1 <= 32) and one warp per approximation item (lanes = error
// samples for the 64/1024-sample checks, = control-point rows for the
// subdivision-matrix products).  The level loop of
// approximate_error_controlled (reduce_approx.py:243-296) is a C++ runtime
// in this library: a device FIFO queue of pending cubics processed in
// batches of at most batch_cap, child slots allocated by an exclusive scan of
// child counts (the reference's prefix-sum slot allocation), accepted cubics
// appended and finally radix-sorted by (curve, ta).
//
// Arithmetic order follows the numpy expressions; small dot products and
// matrix products use a sequential FMA chain, which is what numpy/OpenBLAS
// does for the sizes that occur (measured), and integer powers
// are correctly rounded (powi_cr).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mrep_common.cuh"
#include "mrep_prep_math.cuh"

namespace mrep {

static std::mutex g_pascal_mu;
static int g_pascal_dev = -1;

// basis.py:17-22: PASCAL[:, 0] = 1; row n = row n-1 shifted + row n-1
static int ensure_pascal() {
  std::lock_guard<std::mutex> lk(g_pascal_mu);
  int dev = 0;
  MREP_CUDA_CHECK(cudaGetDevice(&dev));
  if (g_pascal_dev == dev) return MREP_OK;
  std::vector<double> P(PASCAL_ROWS * PASCAL_ROWS, 0.0);
  for (int n = 0; n < PASCAL_ROWS; ++n) P[n * PASCAL_ROWS] = 1.0;
  for (int n = 1; n < PASCAL_ROWS; ++n)
    for (int k = 1; k <= n; ++k)
      P[n * PASCAL_ROWS + k] = P[(n - 1) * PASCAL_ROWS + k - 1] + P[(n - 1) * PASCAL_ROWS + k];
  MREP_CUDA_CHECK(cudaMemcpyToSymbol(g_pascal, P.data(), P.size() * sizeof(double)));
  g_pascal_dev = dev;
  return MREP_OK;
}

constexpr int WARPS_PER_BLOCK = 2;
constexpr int LEVW = 33;  // padded row of the Cox-de Boor level buffer

// ---------------------------------------------------------------- spans
__global__ void span_count_kernel(const int32_t* degree, const int64_t* knot_ofs,
                                  const double* knots, int64_t nc, int64_t* nseg,
                                  int64_t* nrows) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  int p = degree[c];
  const double* k = knots + knot_ofs[c];
  int64_t m = knot_ofs[c + 1] - knot_ofs[c];
  int64_t cnt = 0;
  for (int64_t q = p; q < m - p - 1; ++q)
    if (k[q] < k[q + 1]) ++cnt;  // core.py:108-112
  nseg[c] = cnt;
  nrows[c] = cnt * (p + 1);
}

__global__ void span_list_kernel(const int32_t* degree, const int64_t* knot_ofs,
                                 const double* knots, int64_t nc, const int64_t* seg_ofs,
                                 int32_t* span, int32_t* seg_curve) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  int p = degree[c];
  const double* k = knots + knot_ofs[c];
  int64_t m = knot_ofs[c + 1] - knot_ofs[c];
  int64_t o = seg_ofs[c];
  for (int64_t q = p; q < m - p - 1; ++q)
    if (k[q] < k[q + 1]) {
      span[o] = (int32_t)q;
      seg_curve[o] = (int32_t)c;
      ++o;
    }
}

// basis.py:110-149, warp-cooperative: lane k owns polynomial coefficient k.
// Returns the final level buffer: slot j (row stride LEVW) holds the
// coefficients of N_{q-p+j,p} in powers of (t - center).
__device__ const double* span_basis_warp(const double* kn, int p, int q, double center, double* L0,
                                         double* L1) {
  const int k = threadIdx.x & 31;
  const bool act = k <= p;
  if (act) L0[0 * LEVW + k] = (k == 0) ? 1.0 : 0.0;
  __syncwarp();
  double* cur = L0;
  double* nxt = L1;
  for (int j = 1; j <= p; ++j) {
    for (int si = 0; si <= j; ++si) {
      int i = q - j + si;
      double cv = 0.0;
      if (si >= 1) {  // left = N_{i, j-1} at previous slot si-1
        double den = kn[i + j] - kn[i];
        if (act && k >= 1) cv += cur[(si - 1) * LEVW + k - 1] / den;
        double s1 = (center - kn[i]) / den;
        if (act) cv += s1 * cur[(si - 1) * LEVW + k];
      }
      if (si <= j - 1) {  // right = N_{i+1, j-1} at previous slot si
        double den = kn[i + j + 1] - kn[i + 1];
        if (act && k >= 1) cv -= cur[si * LEVW + k - 1] / den;
        double s2 = (kn[i + j + 1] - center) / den;
        if (act) cv += s2 * cur[si * LEVW + k];
      }
      if (act) nxt[si * LEVW + k] = cv;
    }
    __syncwarp();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  return cur;
}

// decompose.py:19-46 + basis.py:110-149: one warp per nonzero span
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
    decompose_kernel(const int32_t* degree, const int64_t* knot_ofs, const double* knots,
                     const int64_t* ctrl_ofs, const double* ctrl, int d, const int64_t* seg_ofs,
                     const int64_t* row_base, const int32_t* span, const int32_t* seg_curve,
                     int64_t nseg, double* out_rows, int64_t* out_row_ofs, double* out_iv) {
  __shared__ double lev[WARPS_PER_BLOCK][2][32 * LEVW];
  __shared__ double Rsh[WARPS_PER_BLOCK][32 * 3];
  int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t gs = (int64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
  if (gs >= nseg) return;
  int c = seg_curve[gs];
  int p = degree[c];
  int q = span[gs];
  const double* kn = knots + knot_ofs[c];
  const double* cp = ctrl + ctrl_ofs[c] * d;
  int64_t ncp = ctrl_ofs[c + 1] - ctrl_ofs[c];
  int64_t j_local = gs - seg_ofs[c];
  int64_t nseg_c = seg_ofs[c + 1] - seg_ofs[c];
  const int k = lane;
  const bool act = k <= p;
  const double* cur = span_basis_warp(kn, p, q, kn[q], lev[wib][0], lev[wib][1]);
  // row k of M1 = diag(h^k) A, then R[k] = M1[k] @ cp[q-p .. q] (FMA chain)
  double h = kn[q + 1] - kn[q];
  double hk = powi_cr(h, k);
  double R[3] = {0.0, 0.0, 0.0};
  if (act) {
    for (int col = 0; col <= p; ++col) {
      double m1 = hk * cur[col * LEVW + k];
      const double* row = cp + (int64_t)(q - p + col) * d;
      for (int dim = 0; dim < d; ++dim) R[dim] = fma(m1, row[dim], R[dim]);
    }
    for (int dim = 0; dim < d; ++dim) Rsh[wib][k * 3 + dim] = R[dim];
  }
  __syncwarp();
  // Q[i] = T_p[i] @ R, T_p[i][k] = C(i,k) / C(p,k) (basis.py:76-92)
  if (act) {
    const int i = k;
    double Qv[3] = {0.0, 0.0, 0.0};
    for (int kk = 0; kk <= i; ++kk) {
      double t = binom(i, kk) / binom(p, kk);
      for (int dim = 0; dim < d; ++dim) Qv[dim] = fma(t, Rsh[wib][kk * 3 + dim], Qv[dim]);
    }
    // clamping makes the outer endpoints exact (decompose.py:40-44)
    if (j_local == 0 && i == 0)
      for (int dim = 0; dim < d; ++dim) Qv[dim] = cp[dim];
    if (j_local == nseg_c - 1 && i == p)
      for (int dim = 0; dim < d; ++dim) Qv[dim] = cp[(ncp - 1) * d + dim];
    int64_t r0 = row_base[c] + j_local * (p + 1);
    for (int dim = 0; dim < d; ++dim) out_rows[(r0 + i) * d + dim] = Qv[dim];
    if (i == 0) {
      out_row_ofs[gs] = r0;
      out_iv[gs * 2] = kn[q];
      out_iv[gs * 2 + 1] = kn[q + 1];
    }
  }
  if (gs == nseg - 1 && lane == 0) out_row_ofs[nseg] = row_base[c] + nseg_c * (p + 1);
}

// ------------------------------------------------------------ evaluation
// core.py:248-258 (de Casteljau of one Bezier at many u): thread per u
__global__ void eval_bezier_kernel(const double* pts, int np1, int d, const double* u, int64_t m,
                                   double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double uu = u[i];
  double b[32 * 3];
  for (int r = 0; r < np1; ++r)
    for (int dim = 0; dim < d; ++dim) b[r * 3 + dim] = pts[r * d + dim];
  for (int lv = 0; lv < np1 - 1; ++lv)
    for (int r = 0; r < np1 - 1 - lv; ++r)
      for (int dim = 0; dim < d; ++dim)
        b[r * 3 + dim] = (1.0 - uu) * b[r * 3 + dim] + uu * b[(r + 1) * 3 + dim];
  for (int dim = 0; dim < d; ++dim) out[i * d + dim] = b[dim];
}

// oracle.py:13-52: Cox-de Boor recursion restricted to the p+1 functions
// alive at t (the others are exactly zero in the reference's full table)
__global__ void eval_curve_kernel(int p, const double* kn, int64_t m, const double* ctrl,
                                  int64_t ncp, int d, const double* ts, int64_t nt, double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  double t = ts[i];
  // span: last nonzero [k_s, k_s+1) containing t; at t == k[-1] the final nonzero span
  int64_t s = -1, last = -1;
  for (int64_t j = 0; j < m - 1; ++j)
    if (kn[j] < kn[j + 1]) {
      last = j;
      if (kn[j] <= t && t < kn[j + 1]) s = j;
    }
  if (t == kn[m - 1] && last >= 0) s = last;
  double N[33];
  for (int j = 0; j <= p; ++j) N[j] = 0.0;
  if (s < 0) {
    for (int dim = 0; dim < d; ++dim) out[i * d + dim] = 0.0;
    return;
  }
  // N[j] holds N_{s-p+j, level}; level 0: indicator at s
  N[p] = 1.0;
  for (int lvl = 1; lvl <= p; ++lvl) {
    for (int j = p - lvl; j <= p; ++j) {
      int64_t b = s - p + j;  // function index i
      double acc = 0.0;
      double d1 = kn[b + lvl] - kn[b];
      if (d1 > 0.0) acc += (t - kn[b]) / d1 * N[j];
      double d2 = kn[b + lvl + 1] - kn[b + 1];
      if (d2 > 0.0 && j + 1 <= p) acc += (kn[b + lvl + 1] - t) / d2 * N[j + 1];
      N[j] = acc;
    }
  }
  for (int dim = 0; dim < d; ++dim) {
    double acc = 0.0;
    for (int j = 0; j <= p; ++j) {
      int64_t b = s - p + j;
      if (b >= 0 && b < ncp) acc = fma(N[j], ctrl[b * d + dim], acc);
    }
    out[i * d + dim] = acc;
  }
}

// ------------------------------------------------------- approximation
struct ApproxDev {
  // originals (degree >= 1), CSR rows of stride d
  const double* orow;
  const int64_t* orow_ofs;
  const double* oiv;
  const int32_t* ocurve;
  int64_t norig;
  int d;
  // queue (stride 3 for points)
  int64_t* q_orig;
  double* q_la;
  double* q_lb;
  int32_t* q_depth;
  double* q_P;
  // batch scratch
  int32_t* b_status;  // 0 accepted, 1 failing
  double* b_mx;       // record error (64-sample mx, or 1024-sample if verify failed)
  int64_t* b_nchild;
  uint32_t* b_mask;   // [B][mwords]
  int32_t* b_nsamp;
  int mwords;
  // output
  double* o_P;
  double* o_iv;
  double* o_err;
  int32_t* o_curve;
  unsigned long long* o_count;
  int64_t o_cap;
  // error reporting: first failing item index that hit max_depth
  unsigned long long* depth_fail;
};

__device__ __forceinline__ double lin_sample(int i, int ns) {
  // numpy.linspace(0, 1, ns)[i]
  if (ns == 1) return 0.0;
  if (i == ns - 1) return 1.0;
  return (double)i * (1.0 / (double)(ns - 1));
}

// reduce_approx.py:80-121, single thread; Q rows stride 3
__device__ void g1_reduce(const double* Q, int p, int d, double* R, double* d0o, double* d1o) {
  double dQ0[3], dQp[3], ext[3];
  for (int k = 0; k < d; ++k) {
    dQ0[k] = Q[1 * 3 + k] - Q[0 * 3 + k];
    dQp[k] = Q[p * 3 + k] - Q[(p - 1) * 3 + k];
    double lo = Q[k], hi = Q[k];
    for (int j = 1; j <= p; ++j) {
      lo = fmin(lo, Q[j * 3 + k]);
      hi = fmax(hi, Q[j * 3 + k]);
    }
    ext[k] = hi - lo;
  }
  auto dot = [&](const double* a, const double* b) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc = fma(a[k], b[k], acc);
    return acc;
  };
  double scale = sqrt(dot(ext, ext));
  double eps = 1e-12 * fmax(scale, 1e-300);
  double dd0 = 1.0, dd1 = 1.0;
  bool fallback = sqrt(dot(dQ0, dQ0)) <= eps || sqrt(dot(dQp, dQp)) <= eps;
  if (!fallback) {
    // Gram rows G(3,p)[1], G(3,p)[2] and G(3,3) (basis.py:95-107)
    auto gram = [&](int m, int n, int i, int j) {
      return binom(m, i) * binom(n, j) / ((double)(m + n + 1) * binom(m + n, i + j));
    };
    double V1[3], V2[3];
    for (int k = 0; k < d; ++k) {
      double a1 = 0.0, a2 = 0.0;
      for (int j = 0; j <= p; ++j) {
        a1 = fma(gram(3, p, 1, j), Q[j * 3 + k], a1);
        a2 = fma(gram(3, p, 2, j), Q[j * 3 + k], a2);
      }
      double e1 = 0.0, e2 = 0.0;
      double ends[4] = {Q[k], Q[k], Q[p * 3 + k], Q[p * 3 + k]};
      for (int j = 0; j < 4; ++j) {
        e1 = fma(gram(3, 3, 1, j), ends[j], e1);
        e2 = fma(gram(3, 3, 2, j), ends[j], e2);
      }
      V1[k] = a1 - e1;
      V2[k] = a2 - e2;
    }
    double c = (double)p / 3.0;
    double a11 = gram(3, 3, 1, 1) * c * dot(dQ0, dQ0);
    double a12 = -gram(3, 3, 1, 2) * c * dot(dQp, dQ0);
    double a21 = gram(3, 3, 2, 1) * c * dot(dQ0, dQp);
    double a22 = -gram(3, 3, 2, 2) * c * dot(dQp, dQp);
    double b1 = dot(V1, dQ0);
    double b2 = dot(V2, dQp);
    double det = a11 * a22 - a12 * a21;
    if (!(fabs(det) <= 1e-12 * (fabs(a11 * a22) + fabs(a12 * a21)))) {
      dd0 = (b1 * a22 - a12 * b2) / det;
      dd1 = (a11 * b2 - a21 * b1) / det;
    }
  }
  // _g1_cubic (reduce_approx.py:60-66)
  double c = (double)p / 3.0;
  for (int k = 0; k < d; ++k) {
    R[0 * 3 + k] = Q[k];
    R[1 * 3 + k] = Q[k] + c * (Q[3 + k] - Q[k]) * dd0;
    R[2 * 3 + k] = Q[p * 3 + k] - c * (Q[p * 3 + k] - Q[(p - 1) * 3 + k]) * dd1;
    R[3 * 3 + k] = Q[p * 3 + k];
  }
  if (d0o) *d0o = dd0;
  if (d1o) *d1o = dd1;
}

// sum_j bern(p, j, v) Q_j with bern as bernstein_design builds it
// ((C(p,j) * v**j) * (1-v)**(p-j), basis.py:192-196; FMA accumulation in j
// order).  The powers come from one double-double chain per base instead of
// a binary powering per (j, base): the same correctly rounded values (both
// carry ~2^-100 relative error before the final rounding) at a quarter of
// the work.
__device__ __forceinline__ void bern_comb(const double* Q, int p, int d, double v, double* o) {
  double wp[32];
  {
    const double w = 1.0 - v;
    double h = 1.0, l = 0.0;
    wp[0] = 1.0;
    for (int k = 1; k <= p; ++k) {
      dd_mul(h, l, w, 0.0);
      wp[k] = (k == 1) ? w : h + l;
    }
  }
  double vh = 1.0, vl = 0.0;
  for (int j = 0; j <= p; ++j) {
    double vj;
    if (j == 0) {
      vj = 1.0;
    } else {
      dd_mul(vh, vl, v, 0.0);
      vj = (j == 1) ? v : vh + vl;
    }
    const double bj = binom(p, j) * vj * wp[p - j];
    for (int k = 0; k < d; ++k) o[k] = fma(bj, Q[j * 3 + k], o[k]);
  }
}

// reduce_approx.py:146-155 for one (cubic, original) pair, warp-cooperative.
// Writes the argmax mask (err >= mx - 1e-12) and returns mx.  With `errs`
// (shared memory, >= ns doubles) the second pass reads the errors back
// instead of recomputing them (same bits either way).
__device__ double max_error_warp(const double* P, double pa, double pb, const double* Q, int p,
                                 int d, double oa, double ob, int ns, uint32_t* mask,
                                 double* errs = nullptr) {
  int lane = threadIdx.x & 31;
  int nchunks = (ns + 31) / 32;
  double mx = -1.0;
  // pass 1: the maximum; pass 2: the argmax set
  for (int pass = 0; pass < 2; ++pass) {
    for (int ch = 0; ch < nchunks; ++ch) {
      int i = ch * 32 + lane;
      double err = -1.0;
      if (i < ns) {
        if (pass == 1 && errs) {
          err = errs[i];
        } else {
          double u = lin_sample(i, ns);
          double t = pa + u * (pb - pa);
          double v = (t - oa) / (ob - oa);
          double a[3] = {0.0, 0.0, 0.0}, o[3] = {0.0, 0.0, 0.0};
          for (int j = 0; j < 4; ++j) {
            double bj = bern(3, j, u);
            for (int k = 0; k < d; ++k) a[k] = fma(bj, P[j * 3 + k], a[k]);
          }
          bern_comb(Q, p, d, v, o);
          double s = 0.0;
          for (int k = 0; k < d; ++k) {
            double df = a[k] - o[k];
            s = (k == 0) ? df * df : s + df * df;
          }
          err = sqrt(s);
          if (errs) errs[i] = err;
        }
      }
      if (pass == 0) {
        mx = fmax(mx, err);
      } else {
        unsigned bits = __ballot_sync(0xffffffffu, i < ns && err >= mx - 1e-12);
        if (lane == 0) mask[ch] = bits;
      }
    }
    if (pass == 0) {
      for (int off = 16; off; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
  }
  return mx;
}

// load original row block into shared (stride 3)
__device__ __forceinline__ void load_rows(const double* rows, int np1, int d, double* sh) {
  int lane = threadIdx.x & 31;
  if (lane < np1)
    for (int k = 0; k < 3; ++k) sh[lane * 3 + k] = k < d ? rows[lane * d + k] : 0.0;
  __syncwarp();
}

// reduce_approx.py:229-240: seed the queue / output
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
    approx_init_kernel(ApproxDev A, const int64_t* qslot) {
  __shared__ double Qs[WARPS_PER_BLOCK][32 * 3];
  int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t i = (int64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
  if (i >= A.norig) return;
  int64_t r0 = A.orow_ofs[i];
  int p = (int)(A.orow_ofs[i + 1] - r0) - 1;
  int d = A.d;
  double* Q = Qs[wib];
  load_rows(A.orow + r0 * d, p + 1, d, Q);
  if (lane != 0) return;
  double oa = A.oiv[2 * i], ob = A.oiv[2 * i + 1];
  if (p <= 3) {
    double P[4 * 3];
    if (p == 3) {
      for (int j = 0; j < 12; ++j) P[j] = Q[j];
    } else {
      // elevate_degree (reduce_approx.py:129-143)
      double cur[4 * 3];
      for (int j = 0; j < (p + 1) * 3; ++j) cur[j] = Q[j];
      int pp = p;
      while (pp < 3) {
        double out[4 * 3];
        for (int k = 0; k < 3; ++k) out[k] = cur[k];
        for (int r = 1; r <= pp; ++r) {
          double w = (double)r / ((double)pp + 1.0);
          for (int k = 0; k < 3; ++k)
            out[r * 3 + k] = w * cur[(r - 1) * 3 + k] + (1.0 - w) * cur[r * 3 + k];
        }
        for (int k = 0; k < 3; ++k) out[(pp + 1) * 3 + k] = cur[pp * 3 + k];
        ++pp;
        for (int j = 0; j < (pp + 1) * 3; ++j) cur[j] = out[j];
      }
      for (int j = 0; j < 12; ++j) P[j] = cur[j];
    }
    unsigned long long slot = atomicAdd(A.o_count, 1ull);
    if ((int64_t)slot < A.o_cap) {
      for (int j = 0; j < 12; ++j) A.o_P[slot * 12 + j] = P[j];
      A.o_iv[slot * 2] = oa;
      A.o_iv[slot * 2 + 1] = ob;
      A.o_err[slot] = 0.0;
      A.o_curve[slot] = A.ocurve ? A.ocurve[i] : 0;
    }
    return;
  }
  int64_t s = qslot[i];
  double R[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  g1_reduce(Q, p, d, R, nullptr, nullptr);
  for (int j = 0; j < 12; ++j) A.q_P[s * 12 + j] = R[j];
  A.q_orig[s] = i;
  A.q_la[s] = 0.0;
  A.q_lb[s] = 1.0;
  A.q_depth[s] = 0;
}

__global__ void flag_kernel(const int64_t* orow_ofs, int64_t n, int64_t* flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (orow_ofs[i + 1] - orow_ofs[i] - 1) >= 4 ? 1 : 0;
}

// reduce_approx.py:248-272 for one batch [head, head + B)
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
    approx_eval_kernel(ApproxDev A, int64_t head, int64_t B, double tol, int ls, int vs,
                       int max_depth) {
  __shared__ double Qs[WARPS_PER_BLOCK][32 * 3];
  __shared__ double Ps[WARPS_PER_BLOCK][12];
  int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t bi = (int64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
  if (bi >= B) return;
  int64_t it = head + bi;
  int64_t oi = A.q_orig[it];
  int64_t r0 = A.orow_ofs[oi];
  int p = (int)(A.orow_ofs[oi + 1] - r0) - 1;
  int d = A.d;
  double* Q = Qs[wib];
  load_rows(A.orow + r0 * d, p + 1, d, Q);
  if (lane < 12) Ps[wib][lane] = A.q_P[it * 12 + lane];
  __syncwarp();
  double oa = A.oiv[2 * oi], ob = A.oiv[2 * oi + 1];
  double la = A.q_la[it], lb = A.q_lb[it];
  double pa = oa + la * (ob - oa), pb = oa + lb * (ob - oa);
  uint32_t* mask = A.b_mask + bi * A.mwords;
  double mx = max_error_warp(Ps[wib], pa, pb, Q, p, d, oa, ob, ls, mask);
  int nsamp = ls;
  bool accept = false;
  double rec = mx;
  if (mx <= tol) {
    double mx2 = max_error_warp(Ps[wib], pa, pb, Q, p, d, oa, ob, vs, mask);
    if (mx2 <= tol) {
      accept = true;
      if (lane == 0) {
        unsigned long long slot = atomicAdd(A.o_count, 1ull);
        if ((int64_t)slot < A.o_cap) {
          for (int j = 0; j < 12; ++j) A.o_P[slot * 12 + j] = Ps[wib][j];
          A.o_iv[slot * 2] = pa;
          A.o_iv[slot * 2 + 1] = pb;
          A.o_err[slot] = mx2;
          A.o_curve[slot] = A.ocurve ? A.ocurve[oi] : 0;
        }
      }
    } else {
      nsamp = vs;
      rec = mx2;
    }
  }
  if (lane != 0) return;
  A.b_status[bi] = accept ? 0 : 1;
  A.b_mx[bi] = rec;
  A.b_nsamp[bi] = nsamp;
  if (accept) {
    A.b_nchild[bi] = 0;
    return;
  }
  if (A.q_depth[it] >= max_depth) atomicMin(A.depth_fail, (unsigned long long)bi);
  int nz = 0;
  for (int w = 0; w < (nsamp + 31) / 32; ++w) {
    uint32_t bits = mask[w];
    while (bits) {
      int b = __ffs(bits) - 1;
      bits &= bits - 1;
      double z = lin_sample(w * 32 + b, nsamp);
      if (1e-9 < z && z < 1.0 - 1e-9) ++nz;
    }
  }
  A.b_nchild[bi] = (nz > 0 ? nz : 1) + 1;
}

// the k-th interior argmax parameter of batch item bi (or 0.5 if none)
__device__ double interior_z(const ApproxDev& A, int64_t bi, int k, int* nz_out) {
  int nsamp = A.b_nsamp[bi];
  const uint32_t* mask = A.b_mask + bi * A.mwords;
  int nz = 0;
  double zk = 0.5;
  for (int w = 0; w < (nsamp + 31) / 32; ++w) {
    uint32_t bits = mask[w];
    while (bits) {
      int b = __ffs(bits) - 1;
      bits &= bits - 1;
      double z = lin_sample(w * 32 + b, nsamp);
      if (1e-9 < z && z < 1.0 - 1e-9) {
        if (nz == k) zk = z;
        ++nz;
      }
    }
  }
  *nz_out = nz;
  return zk;
}

// de Casteljau of the original at u (core.py:248-258), lane-parallel
__device__ void warp_eval(const double* Q, int p, double u, double* out3) {
  int lane = threadIdx.x & 31;
  double b[3];
  for (int k = 0; k < 3; ++k) b[k] = lane <= p ? Q[lane * 3 + k] : 0.0;
  double omu = 1.0 - u;
  for (int lv = 0; lv < p; ++lv) {
    double nb[3];
    for (int k = 0; k < 3; ++k) {
      double right = __shfl_down_sync(0xffffffffu, b[k], 1);
      nb[k] = omu * b[k] + u * right;
    }
    for (int k = 0; k < 3; ++k) b[k] = nb[k];
  }
  for (int k = 0; k < 3; ++k) out3[k] = __shfl_sync(0xffffffffu, b[k], 0);
}

// reduce_approx.py:171-182: Q <- S_L((b-a)/(1-a)) S_R(a) Q, lane = row
__device__ void warp_restrict(double* Q, int p, double a, double b, double* tmp) {
  int lane = threadIdx.x & 31;
  int n = p;
  if (a > 0.0) {
    double v[3] = {0.0, 0.0, 0.0};
    if (lane <= n) {
      int i = lane;
      for (int j = i; j <= n; ++j) {
        double s = binom(n - i, j - i) * powi_cr(a, j - i) * powi_cr(1.0 - a, n - j);
        for (int k = 0; k < 3; ++k) v[k] = fma(s, Q[j * 3 + k], v[k]);
      }
    }
    __syncwarp();
    if (lane <= n)
      for (int k = 0; k < 3; ++k) tmp[lane * 3 + k] = v[k];
    __syncwarp();
    if (lane <= n)
      for (int k = 0; k < 3; ++k) Q[lane * 3 + k] = tmp[lane * 3 + k];
    __syncwarp();
    b = (b - a) / (1.0 - a);
  }
  if (b < 1.0) {
    double v[3] = {0.0, 0.0, 0.0};
    if (lane <= n) {
      int i = lane;
      for (int j = 0; j <= i; ++j) {
        double s = binom(i, j) * powi_cr(b, j) * powi_cr(1.0 - b, i - j);
        for (int k = 0; k < 3; ++k) v[k] = fma(s, Q[j * 3 + k], v[k]);
      }
    }
    __syncwarp();
    if (lane <= n)
      for (int k = 0; k < 3; ++k) tmp[lane * 3 + k] = v[k];
    __syncwarp();
    if (lane <= n)
      for (int k = 0; k < 3; ++k) Q[lane * 3 + k] = tmp[lane * 3 + k];
    __syncwarp();
  }
}

// reduce_approx.py:274-291: build child k of failing batch item `parent`
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
    approx_child_kernel(ApproxDev A, int64_t head, int64_t B, const int64_t* child_ofs,
                        int64_t nchildren, int64_t tail) {
  __shared__ double Qs[WARPS_PER_BLOCK][32 * 3];
  __shared__ double Ts[WARPS_PER_BLOCK][32 * 3];
  __shared__ double Os[WARPS_PER_BLOCK][32 * 3];
  int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t ci = (int64_t)blockIdx.x * WARPS_PER_BLOCK + wib;
  if (ci >= nchildren) return;
  // parent = last batch index with child_ofs[parent] <= ci
  int64_t lo = 0, hi = B;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (child_ofs[mid] <= ci) lo = mid;
    else hi = mid;
  }
  int64_t parent = lo;
  while (parent + 1 < B && child_ofs[parent + 1] <= ci) ++parent;
  int k = (int)(ci - child_ofs[parent]);
  int64_t it = head + parent;
  int64_t oi = A.q_orig[it];
  int64_t r0 = A.orow_ofs[oi];
  int p = (int)(A.orow_ofs[oi + 1] - r0) - 1;
  int d = A.d;
  double la = A.q_la[it], lb = A.q_lb[it];
  int nz;
  double zk = interior_z(A, parent, k, &nz);
  double zprev = 0.0;
  if (k > 0) {
    int dummy;
    zprev = interior_z(A, parent, k - 1, &dummy);
  }
  int ncuts = (nz > 0 ? nz : 1);  // interior cuts
  double ca = (k == 0) ? la : la + zprev * (lb - la);
  double cb = (k == ncuts) ? lb : la + zk * (lb - la);
  double* O = Os[wib];
  load_rows(A.orow + r0 * d, p + 1, d, O);
  // child fit: G1 reduction of the original restricted to [ca, cb]
  double* Q = Qs[wib];
  if (lane <= p)
    for (int kk = 0; kk < 3; ++kk) Q[lane * 3 + kk] = O[lane * 3 + kk];
  __syncwarp();
  warp_restrict(Q, p, ca, cb, Ts[wib]);
  double pin0[3], pin1[3];
  warp_eval(O, p, ca, pin0);
  warp_eval(O, p, cb, pin1);
  if (lane != 0) return;
  double R[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  g1_reduce(Q, p, d, R, nullptr, nullptr);
  // one stored point per interior cut keeps the seams C0 exact
  if (k > 0)
    for (int kk = 0; kk < 3; ++kk) R[kk] = pin0[kk];
  if (k < ncuts)
    for (int kk = 0; kk < 3; ++kk) R[9 + kk] = pin1[kk];
  for (int kk = 0; kk < 3; ++kk)
    if (kk >= d) R[kk] = R[3 + kk] = R[6 + kk] = R[9 + kk] = 0.0;
  int64_t s = tail + ci;
  for (int j = 0; j < 12; ++j) A.q_P[s * 12 + j] = R[j];
  A.q_orig[s] = oi;
  A.q_la[s] = ca;
  A.q_lb[s] = cb;
  A.q_depth[s] = A.q_depth[it] + 1;
}

__global__ void gather_out_kernel(const int64_t* idx, int64_t n, const double* P, const double* iv,
                                  const double* err, const int32_t* curve, int d, double* oP,
                                  double* oiv, double* oerr, int32_t* ocurve) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t s = idx[i];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < d; ++k) oP[(i * 4 + j) * d + k] = P[s * 12 + j * 3 + k];
  oiv[2 * i] = iv[2 * s];
  oiv[2 * i + 1] = iv[2 * s + 1];
  if (oerr) oerr[i] = err[s];
  if (ocurve) ocurve[i] = curve[s];
}

__global__ void iota_kernel(int64_t* a, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
__global__ void ta_key_kernel(const double* iv, int64_t n, double* key) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = iv[2 * i];
}
__global__ void curve_key_kernel(const int32_t* curve, const int64_t* idx, int64_t n,
                                 int32_t* key) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = curve[idx[i]];
}

// --------------------------------------------------- device buffer helper
template <typename T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  int reserve(int64_t want, bool keep, cudaStream_t st) {
    if (want <= n) return MREP_OK;
    int64_t cap = std::max<int64_t>(want, n * 2);
    T* q = nullptr;
    MREP_CUDA_CHECK(cudaMalloc(&q, sizeof(T) * (size_t)cap));
    if (keep && p && n) MREP_CUDA_CHECK(cudaMemcpyAsync(q, p, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
    if (p) {
      MREP_CUDA_CHECK(cudaStreamSynchronize(st));
      cudaFree(p);
    }
    p = q;
    n = cap;
    return MREP_OK;
  }
};

template <typename T>
static int exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, st));
  void* t = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync(&t, tmp > 0 ? tmp : 1, st));
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)n, st));
  MREP_CUDA_CHECK(cudaFreeAsync(t, st));
  return MREP_OK;
}

// ---------------------------------------------------- single-item kernels
// basis.py:110-149 for one span: A [p+1][p+1] row-major (A[k][j])
__global__ void span_basis_kernel(const double* kn, int p, int q, double center, double* A) {
  __shared__ double lev[2][32 * LEVW];
  const double* cur = span_basis_warp(kn, p, q, center, lev[0], lev[1]);
  int k = threadIdx.x;
  if (k <= p)
    for (int j = 0; j <= p; ++j) A[k * (p + 1) + j] = cur[j * LEVW + k];
}

// reduce_approx.py:69-121: reduce_points_g1 + _l2_error for n segments of
// equal degree (one thread each); Q [n][p+1][d] -> R [n][4][d], delta [n][2], l2 [n]
__global__ void reduce_g1_kernel(const double* Qg, int p, int d, int64_t n, double* Rg,
                                 double* delta, double* l2) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double Q[32 * 3], R[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k < 3; ++k) Q[j * 3 + k] = k < d ? Qg[(s * (p + 1) + j) * d + k] : 0.0;
  double d0, d1;
  g1_reduce(Q, p, d, R, &d0, &d1);
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < d; ++k) Rg[(s * 4 + j) * d + k] = R[j * 3 + k];
  delta[2 * s] = d0;
  delta[2 * s + 1] = d1;
  // eps = Q'GppQ - 2 Q'Gp3R + R'G33R (einsum "id,ij,jd->"), clamped at 0
  auto gram = [&](int m, int nn, int i, int j) {
    return binom(m, i) * binom(nn, j) / ((double)(m + nn + 1) * binom(m + nn, i + j));
  };
  double e1 = 0.0, e2 = 0.0, e3 = 0.0;
  for (int i = 0; i <= p; ++i)
    for (int j = 0; j <= p; ++j)
      for (int k = 0; k < d; ++k) e1 += Q[i * 3 + k] * gram(p, p, i, j) * Q[j * 3 + k];
  for (int i = 0; i <= p; ++i)
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < d; ++k) e2 += Q[i * 3 + k] * gram(p, 3, i, j) * R[j * 3 + k];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < d; ++k) e3 += R[i * 3 + k] * gram(3, 3, i, j) * R[j * 3 + k];
  double e = e1 - 2.0 * e2 + e3;
  l2[s] = e > 0.0 ? e : 0.0;
}

// reduce_approx.py:146-168: one (cubic, original) pair, one warp
__global__ void max_error_kernel(const double* Pg, double pa, double pb, const double* Qg, int p,
                                 int d, double oa, double ob, int ns, double* mx_out,
                                 uint32_t* mask) {
  __shared__ double Qs[32 * 3];
  __shared__ double Ps[12];
  int lane = threadIdx.x;
  load_rows(Qg, p + 1, d, Qs);
  if (lane < 12) Ps[lane] = (lane % 3) < d ? Pg[(lane / 3) * d + lane % 3] : 0.0;
  __syncwarp();
  double mx = max_error_warp(Ps, pa, pb, Qs, p, d, oa, ob, ns, mask);
  if (lane == 0) *mx_out = mx;
}

// reduce_approx.py:129-143: elevate one segment to `target`
__global__ void elevate_kernel(const double* Pg, int p, int d, int target, double* out) {
  double cur[33 * 3];
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k < d; ++k) cur[j * 3 + k] = Pg[j * d + k];
  int pp = p;
  while (pp < target) {
    double nxt[33 * 3];
    for (int k = 0; k < d; ++k) nxt[k] = cur[k];
    for (int r = 1; r <= pp; ++r) {
      double w = (double)r / ((double)pp + 1.0);
      for (int k = 0; k < d; ++k) nxt[r * 3 + k] = w * cur[(r - 1) * 3 + k] + (1.0 - w) * cur[r * 3 + k];
    }
    for (int k = 0; k < d; ++k) nxt[(pp + 1) * 3 + k] = cur[pp * 3 + k];
    ++pp;
    for (int j = 0; j <= pp; ++j)
      for (int k = 0; k < 3; ++k) cur[j * 3 + k] = nxt[j * 3 + k];
  }
  for (int j = 0; j <= target; ++j)
    for (int k = 0; k < d; ++k) out[j * d + k] = cur[j * 3 + k];
}

// reduce_approx.py:185-204 (snap != 0) and distance.py:84-90 (snap == 0):
// split a cubic at z with the subdivision matrices (basis.py:172-189),
// optionally snapping the shared point onto the original segment.
__global__ void split_cubic_kernel(const double* Pg, int d, double z, int snap, double aa,
                                   double ab, const double* Qg, int p, double oa, double ob,
                                   double* Lg, double* Rg) {
  __shared__ double Qs[32 * 3];
  int lane = threadIdx.x;
  double pin[3] = {0, 0, 0};
  if (snap) {
    load_rows(Qg, p + 1, d, Qs);
    double t_split = aa + z * (ab - aa);
    warp_eval(Qs, p, (t_split - oa) / (ob - oa), pin);
  }
  if (lane != 0) return;
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < d; ++k) {
      double l = 0.0, r = 0.0;
      for (int j = 0; j <= i; ++j)
        l = fma(binom(i, j) * powi_cr(z, j) * powi_cr(1.0 - z, i - j), Pg[j * d + k], l);
      for (int j = i; j <= 3; ++j)
        r = fma(binom(3 - i, j - i) * powi_cr(z, j - i) * powi_cr(1.0 - z, 3 - j), Pg[j * d + k], r);
      Lg[i * d + k] = l;
      Rg[i * d + k] = r;
    }
  if (snap)
    for (int k = 0; k < d; ++k) {
      Lg[3 * d + k] = pin[k];
      Rg[k] = pin[k];
    }
}

}  // namespace mrep (kernels)
namespace mrep {

}  // namespace mrep

// ============================================================ approximation handle
struct mrep_approx {
  int d = 3;
  int64_t count = 0;
  mrep::DBuf<double> P, iv, err;
  mrep::DBuf<int32_t> curve;
  mrep::DBuf<int64_t> order;  // sorted order of the raw outputs
  // collect_levels records (host)
  struct Level {
    std::vector<double> P, iv, err;
    std::vector<int64_t> prefix, keys;
  };
  std::vector<Level> levels;
};

using namespace mrep;

extern "C" {

MREP_API int mrep_decompose_plan(const int32_t* degree, const int64_t* knot_ofs,
                                 const double* knots, int64_t nc, int64_t* seg_ofs,
                                 int64_t* row_base, int64_t* total_segs, int64_t* total_rows,
                                 void* stream) {
  if (nc < 1) {
    set_error("mrep_decompose_plan: need at least one curve");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_pascal();
  if (rc) return rc;
  int64_t *cnt = nullptr, *rows = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync(&cnt, sizeof(int64_t) * (nc + 1), st));
  MREP_CUDA_CHECK(cudaMallocAsync(&rows, sizeof(int64_t) * (nc + 1), st));
  MREP_CUDA_CHECK(cudaMemsetAsync(cnt + nc, 0, sizeof(int64_t), st));
  MREP_CUDA_CHECK(cudaMemsetAsync(rows + nc, 0, sizeof(int64_t), st));
  span_count_kernel<<<grid_for(nc, 128), 128, 0, st>>>(degree, knot_ofs, knots, nc, cnt, rows);
  MREP_LAUNCH_CHECK();
  if ((rc = exclusive_scan<int64_t>(cnt, seg_ofs, nc + 1, st))) return rc;
  if ((rc = exclusive_scan<int64_t>(rows, row_base, nc + 1, st))) return rc;
  MREP_CUDA_CHECK(cudaMemcpyAsync(total_segs, seg_ofs + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaMemcpyAsync(total_rows, row_base + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaFreeAsync(cnt, st));
  MREP_CUDA_CHECK(cudaFreeAsync(rows, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  return MREP_OK;
}

MREP_API int mrep_decompose(const int32_t* degree, const int64_t* knot_ofs, const double* knots,
                            const int64_t* ctrl_ofs, const double* ctrl, int64_t nc, int d,
                            const int64_t* seg_ofs, const int64_t* row_base, int64_t nseg,
                            double* out_rows, int64_t* out_row_ofs, double* out_iv,
                            int32_t* out_curve, int32_t* out_span, void* stream) {
  if (nseg < 1 || (d != 2 && d != 3)) {
    set_error("mrep_decompose: need nseg >= 1 and d in {2,3}");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_pascal();
  if (rc) return rc;
  span_list_kernel<<<grid_for(nc, 128), 128, 0, st>>>(degree, knot_ofs, knots, nc, seg_ofs,
                                                      out_span, out_curve);
  MREP_LAUNCH_CHECK();
  decompose_kernel<<<grid_for(nseg, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, st>>>(
      degree, knot_ofs, knots, ctrl_ofs, ctrl, d, seg_ofs, row_base, out_span, out_curve, nseg,
      out_rows, out_row_ofs, out_iv);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_eval_bezier(const double* pts, int degree, int d, const double* u, int64_t m,
                              double* out, void* stream) {
  if (degree < 0 || degree > 31 || (d != 2 && d != 3)) {
    set_error("mrep_eval_bezier: degree in [0,31], d in {2,3}");
    return MREP_ERR_ARG;
  }
  if (m <= 0) return MREP_OK;
  eval_bezier_kernel<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(pts, degree + 1, d, u, m,
                                                                         out);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_eval_curve(int p, const double* knots, int64_t m, const double* ctrl,
                             int64_t ncp, int d, const double* ts, int64_t nt, double* out,
                             void* stream) {
  if (p < 0 || p > 31 || (d != 2 && d != 3)) {
    set_error("mrep_eval_curve: degree in [0,31], d in {2,3}");
    return MREP_ERR_ARG;
  }
  if (nt <= 0) return MREP_OK;
  eval_curve_kernel<<<grid_for(nt, 128), 128, 0, (cudaStream_t)stream>>>(p, knots, m, ctrl, ncp, d,
                                                                         ts, nt, out);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_approx_run(const double* orow, const int64_t* orow_ofs, const double* oiv,
                             const int32_t* ocurve, int64_t norig, int d, double tol,
                             int64_t batch_cap, int loop_samples, int verify_samples,
                             int max_depth, int collect_levels, mrep_approx** out,
                             void* stream) {
  *out = nullptr;
  if (norig < 0 || (d != 2 && d != 3) || loop_samples < 1 || verify_samples < 1) {
    set_error("mrep_approx_run: bad arguments");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_pascal();
  if (rc) return rc;
  auto* H = new mrep_approx();
  H->d = d;
  auto fail = [&](int code) {
    delete H;
    return code;
  };
  if (norig == 0) {
    *out = H;
    return MREP_OK;
  }
  if (batch_cap < 1) batch_cap = 1;
  ApproxDev A{};
  A.orow = orow;
  A.orow_ofs = orow_ofs;
  A.oiv = oiv;
  A.ocurve = ocurve;
  A.norig = norig;
  A.d = d;
  A.mwords = (std::max(loop_samples, verify_samples) + 31) / 32;
  // queue slots for the degree >= 4 originals
  DBuf<int64_t> flag, qslot;
  if ((rc = flag.reserve(norig + 1, false, st)) || (rc = qslot.reserve(norig + 1, false, st)))
    return fail(rc);
  MREP_CUDA_CHECK(cudaMemsetAsync(flag.p + norig, 0, sizeof(int64_t), st));
  flag_kernel<<<grid_for(norig, 128), 128, 0, st>>>(orow_ofs, norig, flag.p);
  if ((rc = exclusive_scan<int64_t>(flag.p, qslot.p, norig + 1, st))) return fail(rc);
  int64_t nq0 = 0;
  MREP_CUDA_CHECK(cudaMemcpyAsync(&nq0, qslot.p + norig, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  DBuf<int64_t> q_orig;
  DBuf<double> q_la, q_lb, q_P;
  DBuf<int32_t> q_depth;
  int64_t qcap = std::max<int64_t>(nq0 * 2, 1024);
  if ((rc = q_orig.reserve(qcap, false, st)) || (rc = q_la.reserve(qcap, false, st)) ||
      (rc = q_lb.reserve(qcap, false, st)) || (rc = q_P.reserve(qcap * 12, false, st)) ||
      (rc = q_depth.reserve(qcap, false, st)))
    return fail(rc);
  int64_t ocap = std::max<int64_t>(norig * 4, 1024);
  DBuf<double> oP, oiv2, oerr;
  DBuf<int32_t> ocur;
  DBuf<unsigned long long> counters;  // [0] out count, [1] depth fail
  if ((rc = oP.reserve(ocap * 12, false, st)) || (rc = oiv2.reserve(ocap * 2, false, st)) ||
      (rc = oerr.reserve(ocap, false, st)) || (rc = ocur.reserve(ocap, false, st)) ||
      (rc = counters.reserve(2, false, st)))
    return fail(rc);
  unsigned long long init[2] = {0ull, ~0ull};
  MREP_CUDA_CHECK(cudaMemcpyAsync(counters.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  auto bind = [&]() {
    A.q_orig = q_orig.p;
    A.q_la = q_la.p;
    A.q_lb = q_lb.p;
    A.q_depth = q_depth.p;
    A.q_P = q_P.p;
    A.o_P = oP.p;
    A.o_iv = oiv2.p;
    A.o_err = oerr.p;
    A.o_curve = ocur.p;
    A.o_count = counters.p;
    A.o_cap = ocap;
    A.depth_fail = counters.p + 1;
  };
  bind();
  approx_init_kernel<<<grid_for(norig, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, st>>>(A, qslot.p);
  MREP_LAUNCH_CHECK();
  int64_t head = 0, tail = nq0;
  DBuf<int32_t> b_status, b_nsamp;
  DBuf<double> b_mx;
  DBuf<int64_t> b_nchild, child_ofs;
  DBuf<uint32_t> b_mask;
  while (head < tail) {
    int64_t B = std::min<int64_t>(batch_cap, tail - head);
    if ((rc = b_status.reserve(B, false, st)) || (rc = b_nsamp.reserve(B, false, st)) ||
        (rc = b_mx.reserve(B, false, st)) || (rc = b_nchild.reserve(B + 1, false, st)) ||
        (rc = child_ofs.reserve(B + 1, false, st)) ||
        (rc = b_mask.reserve(B * A.mwords, false, st)))
      return fail(rc);
    A.b_status = b_status.p;
    A.b_nsamp = b_nsamp.p;
    A.b_mx = b_mx.p;
    A.b_nchild = b_nchild.p;
    A.b_mask = b_mask.p;
    // make room for accepted outputs of this batch
    unsigned long long ocount = 0;
    MREP_CUDA_CHECK(cudaMemcpyAsync(&ocount, counters.p, sizeof(ocount), cudaMemcpyDeviceToHost, st));
    MREP_CUDA_CHECK(cudaStreamSynchronize(st));
    if ((int64_t)ocount + B > ocap) {
      int64_t nc2 = std::max<int64_t>(ocap * 2, (int64_t)ocount + B);
      if ((rc = oP.reserve(nc2 * 12, true, st)) || (rc = oiv2.reserve(nc2 * 2, true, st)) ||
          (rc = oerr.reserve(nc2, true, st)) || (rc = ocur.reserve(nc2, true, st)))
        return fail(rc);
      ocap = nc2;
      bind();
    }
    approx_eval_kernel<<<grid_for(B, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, st>>>(
        A, head, B, tol, loop_samples, verify_samples, max_depth);
    MREP_LAUNCH_CHECK();
    MREP_CUDA_CHECK(cudaMemsetAsync(b_nchild.p + B, 0, sizeof(int64_t), st));
    if ((rc = exclusive_scan<int64_t>(b_nchild.p, child_ofs.p, B + 1, st))) return fail(rc);
    int64_t nch = 0;
    unsigned long long dfail = 0;
    MREP_CUDA_CHECK(cudaMemcpyAsync(&nch, child_ofs.p + B, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MREP_CUDA_CHECK(cudaMemcpyAsync(&dfail, counters.p + 1, sizeof(dfail), cudaMemcpyDeviceToHost, st));
    MREP_CUDA_CHECK(cudaStreamSynchronize(st));
    if (dfail != ~0ull) {
      double iv[2] = {0, 0}, la = 0, lb = 0;
      int64_t oi = 0;
      cudaMemcpy(&oi, q_orig.p + head + dfail, sizeof(oi), cudaMemcpyDeviceToHost);
      cudaMemcpy(&la, q_la.p + head + dfail, sizeof(la), cudaMemcpyDeviceToHost);
      cudaMemcpy(&lb, q_lb.p + head + dfail, sizeof(lb), cudaMemcpyDeviceToHost);
      cudaMemcpy(iv, oiv + 2 * oi, sizeof(iv), cudaMemcpyDeviceToHost);
      char msg[256];
      snprintf(msg, sizeof msg,
               "tolerance %g not reached after %d levels on source interval (%.17g, %.17g)", tol,
               max_depth, iv[0] + la * (iv[1] - iv[0]), iv[0] + lb * (iv[1] - iv[0]));
      set_error(msg);
      return fail(MREP_ERR_DEPTH);
    }
    if (collect_levels) {
      mrep_approx::Level L;
      std::vector<double> P(B * 12), la(B), lb(B), mxv(B);
      std::vector<int64_t> orig(B), nchild(B + 1);
      std::vector<int32_t> status(B);
      cudaMemcpy(P.data(), q_P.p + head * 12, B * 12 * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(la.data(), q_la.p + head, B * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(lb.data(), q_lb.p + head, B * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(mxv.data(), b_mx.p, B * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(orig.data(), q_orig.p + head, B * sizeof(int64_t), cudaMemcpyDeviceToHost);
      cudaMemcpy(status.data(), b_status.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost);
      cudaMemcpy(nchild.data(), b_nchild.p, B * sizeof(int64_t), cudaMemcpyDeviceToHost);
      std::vector<double> ivh(2 * norig);
      cudaMemcpy(ivh.data(), oiv, 2 * norig * sizeof(double), cudaMemcpyDeviceToHost);
      L.P = P;
      L.err = mxv;
      L.iv.resize(2 * B);
      L.prefix.push_back(0);
      for (int64_t j = 0; j < B; ++j) {
        double oa = ivh[2 * orig[j]], ob = ivh[2 * orig[j] + 1];
        L.iv[2 * j] = oa + la[j] * (ob - oa);
        L.iv[2 * j + 1] = oa + lb[j] * (ob - oa);
        if (status[j] == 1) {
          L.keys.push_back(j);
          L.prefix.push_back(L.prefix.back() + nchild[j]);
        }
      }
      H->levels.push_back(std::move(L));
    }
    if (nch > 0) {
      // compact the live queue when the children would overflow it
      if (tail + nch > qcap) {
        int64_t live = tail - head;
        int64_t nq = std::max<int64_t>(qcap * 2, live + nch + 1024);
        DBuf<int64_t> o2;
        DBuf<double> la2, lb2, P2;
        DBuf<int32_t> d2;
        if ((rc = o2.reserve(nq, false, st)) || (rc = la2.reserve(nq, false, st)) ||
            (rc = lb2.reserve(nq, false, st)) || (rc = P2.reserve(nq * 12, false, st)) ||
            (rc = d2.reserve(nq, false, st)))
          return fail(rc);
        MREP_CUDA_CHECK(cudaMemcpyAsync(o2.p, q_orig.p + head, live * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
        MREP_CUDA_CHECK(cudaMemcpyAsync(la2.p, q_la.p + head, live * sizeof(double), cudaMemcpyDeviceToDevice, st));
        MREP_CUDA_CHECK(cudaMemcpyAsync(lb2.p, q_lb.p + head, live * sizeof(double), cudaMemcpyDeviceToDevice, st));
        MREP_CUDA_CHECK(cudaMemcpyAsync(P2.p, q_P.p + head * 12, live * 12 * sizeof(double), cudaMemcpyDeviceToDevice, st));
        MREP_CUDA_CHECK(cudaMemcpyAsync(d2.p, q_depth.p + head, live * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        MREP_CUDA_CHECK(cudaStreamSynchronize(st));
        std::swap(q_orig.p, o2.p);
        std::swap(q_orig.n, o2.n);
        std::swap(q_la.p, la2.p);
        std::swap(q_la.n, la2.n);
        std::swap(q_lb.p, lb2.p);
        std::swap(q_lb.n, lb2.n);
        std::swap(q_P.p, P2.p);
        std::swap(q_P.n, P2.n);
        std::swap(q_depth.p, d2.p);
        std::swap(q_depth.n, d2.n);
        tail -= head;
        head = 0;
        qcap = nq;
        bind();
      }
      approx_child_kernel<<<grid_for(nch, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, st>>>(
          A, head, B, child_ofs.p, nch, tail);
      MREP_LAUNCH_CHECK();
    }
    head += B;
    tail += nch;
  }
  // sort outputs by (curve, ta): ta first, then a stable pass on the curve id
  unsigned long long total = 0;
  MREP_CUDA_CHECK(cudaMemcpyAsync(&total, counters.p, sizeof(total), cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  int64_t S = (int64_t)total;
  H->count = S;
  if (S > 0) {
    DBuf<double> key, key2;
    DBuf<int64_t> idx, idx2;
    DBuf<int32_t> ck, ck2;
    if ((rc = key.reserve(S, false, st)) || (rc = key2.reserve(S, false, st)) ||
        (rc = idx.reserve(S, false, st)) || (rc = idx2.reserve(S, false, st)) ||
        (rc = ck.reserve(S, false, st)) || (rc = ck2.reserve(S, false, st)))
      return fail(rc);
    ta_key_kernel<<<grid_for(S, 256), 256, 0, st>>>(oiv2.p, S, key.p);
    iota_kernel<<<grid_for(S, 256), 256, 0, st>>>(idx.p, S);
    size_t tmp = 0;
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, idx2.p, (int)S, 0, 64, st));
    void* t = nullptr;
    MREP_CUDA_CHECK(cudaMallocAsync(&t, tmp + 1, st));
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(t, tmp, key.p, key2.p, idx.p, idx2.p, (int)S, 0, 64, st));
    MREP_CUDA_CHECK(cudaFreeAsync(t, st));
    curve_key_kernel<<<grid_for(S, 256), 256, 0, st>>>(ocur.p, idx2.p, S, ck.p);
    tmp = 0;
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ck.p, ck2.p, idx2.p, idx.p, (int)S, 0, 32, st));
    MREP_CUDA_CHECK(cudaMallocAsync(&t, tmp + 1, st));
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(t, tmp, ck.p, ck2.p, idx2.p, idx.p, (int)S, 0, 32, st));
    MREP_CUDA_CHECK(cudaFreeAsync(t, st));
    if ((rc = H->P.reserve(S * 4 * d, false, st)) || (rc = H->iv.reserve(S * 2, false, st)) ||
        (rc = H->err.reserve(S, false, st)) || (rc = H->curve.reserve(S, false, st)))
      return fail(rc);
    gather_out_kernel<<<grid_for(S, 128), 128, 0, st>>>(idx.p, S, oP.p, oiv2.p, oerr.p, ocur.p, d,
                                                        H->P.p, H->iv.p, H->err.p, H->curve.p);
    MREP_LAUNCH_CHECK();
    MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  *out = H;
  return MREP_OK;
}

MREP_API int64_t mrep_approx_count(const mrep_approx* h) { return h ? h->count : -1; }

MREP_API int mrep_approx_fetch(const mrep_approx* h, double* pts, double* iv, double* err,
                               int32_t* curve, void* stream) {
  if (!h) return MREP_ERR_ARG;
  if (h->count == 0) return MREP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t S = h->count;
  if (pts) MREP_CUDA_CHECK(cudaMemcpyAsync(pts, h->P.p, S * 4 * h->d * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (iv) MREP_CUDA_CHECK(cudaMemcpyAsync(iv, h->iv.p, S * 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (err) MREP_CUDA_CHECK(cudaMemcpyAsync(err, h->err.p, S * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (curve) MREP_CUDA_CHECK(cudaMemcpyAsync(curve, h->curve.p, S * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return MREP_OK;
}

MREP_API int mrep_approx_num_levels(const mrep_approx* h) {
  return h ? (int)h->levels.size() : -1;
}

MREP_API int mrep_approx_level_sizes(const mrep_approx* h, int lvl, int64_t* nrec, int64_t* nfail) {
  if (!h || lvl < 0 || lvl >= (int)h->levels.size()) return MREP_ERR_ARG;
  *nrec = (int64_t)h->levels[lvl].err.size();
  *nfail = (int64_t)h->levels[lvl].keys.size();
  return MREP_OK;
}

MREP_API int mrep_approx_level_fetch(const mrep_approx* h, int lvl, double* P_host, double* iv_host,
                                     double* err_host, int64_t* prefix_host, int64_t* keys_host) {
  if (!h || lvl < 0 || lvl >= (int)h->levels.size()) return MREP_ERR_ARG;
  const auto& L = h->levels[lvl];
  int64_t B = (int64_t)L.err.size();
  int d = h->d;
  for (int64_t j = 0; j < B; ++j)
    for (int r = 0; r < 4; ++r)
      for (int k = 0; k < d; ++k) P_host[(j * 4 + r) * d + k] = L.P[j * 12 + r * 3 + k];
  std::memcpy(iv_host, L.iv.data(), L.iv.size() * sizeof(double));
  std::memcpy(err_host, L.err.data(), L.err.size() * sizeof(double));
  std::memcpy(prefix_host, L.prefix.data(), L.prefix.size() * sizeof(int64_t));
  if (!L.keys.empty()) std::memcpy(keys_host, L.keys.data(), L.keys.size() * sizeof(int64_t));
  return MREP_OK;
}

MREP_API void mrep_approx_free(mrep_approx* h) { delete h; }

MREP_API int mrep_span_basis(const double* knots, int p, int q, double center, double* A,
                             void* stream) {
  if (p < 1 || p > 31) {
    set_error("mrep_span_basis: degree in [1,31]");
    return MREP_ERR_ARG;
  }
  int rc = ensure_pascal();
  if (rc) return rc;
  span_basis_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(knots, p, q, center, A);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_reduce_g1(const double* Q, int p, int d, int64_t n, double* R, double* delta,
                            double* l2, void* stream) {
  if (p < 4 || p > 31 || (d != 2 && d != 3)) {
    set_error("mrep_reduce_g1: degree in [4,31], d in {2,3}");
    return MREP_ERR_ARG;
  }
  int rc = ensure_pascal();
  if (rc) return rc;
  if (n <= 0) return MREP_OK;
  reduce_g1_kernel<<<grid_for(n, 64), 64, 0, (cudaStream_t)stream>>>(Q, p, d, n, R, delta, l2);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_max_error(const double* P, double pa, double pb, const double* Q, int p, int d,
                            double oa, double ob, int samples, double* mx, uint32_t* mask,
                            void* stream) {
  if (p < 1 || p > 31 || (d != 2 && d != 3) || samples < 1) {
    set_error("mrep_max_error: bad arguments");
    return MREP_ERR_ARG;
  }
  int rc = ensure_pascal();
  if (rc) return rc;
  max_error_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(P, pa, pb, Q, p, d, oa, ob, samples, mx,
                                                       mask);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_elevate(const double* P, int p, int d, int target, double* out, void* stream) {
  if (p < 0 || target < p || target > 32 || (d != 2 && d != 3)) {
    set_error("mrep_elevate: need p <= target <= 32");
    return MREP_ERR_ARG;
  }
  elevate_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(P, p, d, target, out);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

MREP_API int mrep_split_cubic(const double* P, int d, double z, int snap, double aa, double ab,
                              const double* Q, int p, double oa, double ob, double* L, double* R,
                              void* stream) {
  if ((d != 2 && d != 3) || (snap && (p < 1 || p > 31))) {
    set_error("mrep_split_cubic: bad arguments");
    return MREP_ERR_ARG;
  }
  int rc = ensure_pascal();
  if (rc) return rc;
  split_cubic_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(P, d, z, snap, aa, ab, Q, p, oa, ob, L, R);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}


}  // extern "C"
