// mrep_prep_math.cuh -- scalar helpers for the per-curve preprocessing
// kernels (decomposition, approximation, curve evaluation).
#pragma once
#include <cstdint>

namespace mrep {

constexpr int PASCAL_ROWS = 64;
// Pascal triangle built by repeated double additions exactly like the
// reference's PASCAL table (basis.py:17-22); uploaded once per process.
// (Defined here: only mrep_prep.cu includes this header.)
__device__ double g_pascal[PASCAL_ROWS * PASCAL_ROWS];

__device__ __forceinline__ double binom(int n, int k) {
  return (k < 0 || k > n) ? 0.0 : __ldg(&g_pascal[n * PASCAL_ROWS + k]);
}

// double-double product (a_h + a_l) * (b_h + b_l), renormalised
__device__ __forceinline__ void dd_mul(double& ah, double& al, double bh, double bl) {
  double p = ah * bh;
  double e = fma(ah, bh, -p);
  e += ah * bl;
  e += al * bh;
  double h = p + e;
  double l = e - (h - p);
  ah = h;
  al = l;
}

// x**k for an integer k >= 0, correctly rounded (double-double binary
// powering, one final rounding).  numpy's power on integer exponents 1 and 2
// is exact-by-construction (positive / square), and libm / SVML pow are
// correctly rounded in all but rare cases, so this reproduces the reference's
// `u**j` and `h**k` in practice bit for bit.
__device__ __forceinline__ double powi_cr(double x, int k) {
  if (k == 0) return 1.0;
  if (k == 1) return x;
  if (k == 2) return x * x;
  double rh = 1.0, rl = 0.0, bh = x, bl = 0.0;
  while (k) {
    if (k & 1) dd_mul(rh, rl, bh, bl);
    k >>= 1;
    if (k) dd_mul(bh, bl, bh, bl);
  }
  return rh + rl;
}

// Bernstein basis value as bernstein_design builds it (basis.py:192-196):
// (C(n,j) * u**j) * (1-u)**(n-j)
__device__ __forceinline__ double bern(int n, int j, double u) {
  return binom(n, j) * powi_cr(u, j) * powi_cr(1.0 - u, n - j);
}

}  // namespace mrep
