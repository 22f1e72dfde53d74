// mrep_math.cuh -- per-(query, cubic) scalar arithmetic of the M-rep projection,
// written for sm_100a FP64 CUDA cores.
//
// Every routine restates one numba kernel of the reference
// (/root/reference/pkg/src/splinemat/_kernels.py) with the SAME operation
// order, so with FMA contraction disabled (-fmad=false) the only source of
// bit differences against the reference is the device libm (acos, cos, cbrt:
// CUDA's are 1-2 ulp, glibc's ~0.5 ulp).  Everything lives in registers:
// fixed-size arrays are fully unrolled, the convex-hull stacks are 3-bit index
// words, and root lists are fixed slots with validity flags instead of
// appended arrays (no local-memory traffic).
#pragma once
#include <cstdint>

namespace mrep {

// ------------------------------------------------------------------ helpers
template <int N>
struct Vec {
  double v[N];
};

__device__ __forceinline__ double sel6(const double (&b)[6], int i) {
  // b[i] for a runtime i in [0, 5] without dynamic register indexing
  double r = b[0];
  r = (i == 1) ? b[1] : r;
  r = (i == 2) ? b[2] : r;
  r = (i == 3) ? b[3] : r;
  r = (i == 4) ? b[4] : r;
  r = (i == 5) ? b[5] : r;
  return r;
}

// xs[i] = i / 5 (_kernels.py:249-251), the correctly rounded quotients:
// i * 0.2 rounds to them for every i in [0, 5] except 3 (3 * 0.2 is a tie
// that rounds up to 0.6000000000000001), so one multiply and one select
// replace a five-way select chain
__device__ __forceinline__ double xs5(int i) {
  const double r = (double)i * 0.2;
  return i == 3 ? 0.6 : r;
}

// numba lowers np.cbrt to sign(x)*pow(|x|, 1/3) (numba/np/npyfuncs.py); on the
// device cbrt() is the faster, 1-ulp approximation of the same value.
__device__ __forceinline__ double np_cbrt(double x) { return cbrt(x); }

// numba's static integer power: x**3 = x*(x*x), x**4 = (x*x)*(x*x)
__device__ __forceinline__ double pow3(double x) { return x * (x * x); }
__device__ __forceinline__ double pow4(double x) {
  double a = x * x;
  return a * a;
}

// ------------------------------------------------------- polynomial roots
// _kernels.py:21-31
__device__ __forceinline__ double polish_root(double c0, double c1, double c2, double c3, double c4,
                                              double x) {
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    double f = c0 + x * (c1 + x * (c2 + x * (c3 + x * c4)));
    double df = c1 + x * (2.0 * c2 + x * (3.0 * c3 + x * 4.0 * c4));
    if (df != 0.0) {
      double step = f / df;
      if (fabs(step) < 0.5) x -= step;
    }
  }
  return x;
}

// _kernels.py:34-55; returns count (0..2), roots in r0, r1 (append order)
__device__ __forceinline__ int quad_roots(double c0, double c1, double c2, double& r0, double& r1) {
  if (c2 == 0.0) {
    if (c1 != 0.0) {
      r0 = -c0 / c1;
      return 1;
    }
    return 0;
  }
  double disc = c1 * c1 - 4.0 * c2 * c0;
  if (disc < 0.0) return 0;
  double sq = sqrt(disc);
  double qq = (c1 >= 0.0) ? -0.5 * (c1 + sq) : -0.5 * (c1 - sq);
  r0 = qq / c2;
  if (qq != 0.0) {
    r1 = c0 / qq;
    return 2;
  }
  return 1;
}

// _kernels.py:58-88; up to 3 roots in append order.  Not inlined: it is
// called from two sites (degenerate cubic, Ferrari resolvent) and carries
// acos / cos / cbrt, the largest instruction sequences of the solve.
struct Cubic3 {
  double r0, r1, r2;
  int n;
};

__device__ __noinline__ Cubic3 cubic_roots3(double c0, double c1, double c2, double c3) {
  Cubic3 o{0.0, 0.0, 0.0, 0};
  if (c3 == 0.0) {
    o.n = quad_roots(c0, c1, c2, o.r0, o.r1);
    return o;
  }
  double b = c2 / c3, c = c1 / c3, d = c0 / c3;
  double p = c - b * b / 3.0;
  double q = 2.0 * pow3(b) / 27.0 - b * c / 3.0 + d;
  double off = -b / 3.0;
  double disc = -4.0 * pow3(p) - 27.0 * q * q;
  if (disc >= 0.0 && p < 0.0) {
    double m = 2.0 * sqrt(-p / 3.0);
    double arg = 3.0 * q / (p * m);
    if (arg > 1.0) arg = 1.0;
    else if (arg < -1.0) arg = -1.0;
    double th = acos(arg) / 3.0;
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      double r = m * cos(th - 2.0943951023931953 * (double)k) + off;
      o.r0 = o.r1;  // shift in: after 3 steps r0, r1, r2 = roots k = 0, 1, 2
      o.r1 = o.r2;
      o.r2 = r;
    }
    o.n = 3;
    return o;
  }
  double rr = q * q / 4.0 + pow3(p) / 27.0;
  double srt = sqrt((0.0 > rr) ? 0.0 : rr);  // Python max(rr, 0.0)
  double u = -q / 2.0 + srt;
  double v = -q / 2.0 - srt;
  o.r0 = np_cbrt(u) + np_cbrt(v) + off;
  o.n = 1;
  return o;
}

// The largest real root of the resolvent cubic, as the reference computes it
// (_kernels.py:141-145: every root of _cubic_roots, then the strict max).
// In the three-real-roots branch th = acos(.)/3 lies in [0, pi/3], so
// cos(th) >= 1/2 >= cos(th - 2pi/3) and cos(th - 4pi/3) <= -1/2: with m > 0
// the k = 2 root is below the k = 0 root by m (1 - 2 eps) and can only equal
// it when both round to `off` -- it never changes the maximum, and its
// cosine is skipped.  Same operations otherwise, so the same bits.
__device__ __noinline__ bool resolvent_max_root(double c0, double c1, double c2, double c3,
                                               double& mmax) {
  // c3 = 8 here (never zero)
  double b = c2 / c3, c = c1 / c3, d = c0 / c3;
  double p = c - b * b / 3.0;
  double q = 2.0 * pow3(b) / 27.0 - b * c / 3.0 + d;
  double off = -b / 3.0;
  double disc = -4.0 * pow3(p) - 27.0 * q * q;
  if (disc >= 0.0 && p < 0.0) {
    double m = 2.0 * sqrt(-p / 3.0);
    double arg = 3.0 * q / (p * m);
    if (arg > 1.0) arg = 1.0;
    else if (arg < -1.0) arg = -1.0;
    double th = acos(arg) / 3.0;
    const double r0 = m * cos(th - 2.0943951023931953 * 0.0) + off;
    const double r1 = m * cos(th - 2.0943951023931953 * 1.0) + off;
    mmax = r1 > r0 ? r1 : r0;
    return true;
  }
  double rr = q * q / 4.0 + pow3(p) / 27.0;
  double srt = sqrt((0.0 > rr) ? 0.0 : rr);  // Python max(rr, 0.0)
  double u = -q / 2.0 + srt;
  double v = -q / 2.0 - srt;
  mmax = np_cbrt(u) + np_cbrt(v) + off;
  return true;
}

// Root set of E' on [0,1]: up to 4 sorted slots, `valid` bitmask (bit i = slot i).
struct Roots4 {
  double r[4];
  int count;  // number of valid roots (they occupy slots 0..count-1, ascending)
};

// stable compare-exchange: swap only when strictly out of order
__device__ __forceinline__ void cex(double& a, double& b) {
  if (a > b) {
    double t = a;
    a = b;
    b = t;
  }
}

// _kernels.py:91-176 (Ferrari with the degeneracy cascade, polish, filter,
// sort, dedup).  Candidate slots keep the reference's append order; invalid
// slots hold +inf so a stable 4-element odd-even transposition sort reproduces
// the reference's compaction followed by insertion sort.
// Candidate slots for the quartic: values are shifted in at the END in the
// reference's append order (slot 3 newest); the stable sort afterwards only
// needs the relative order, which shifting preserves.
struct Slots4 {
  double v0, v1, v2, v3;
};

__device__ __forceinline__ void push4(Slots4& S, double x) {
  S.v0 = S.v1;
  S.v1 = S.v2;
  S.v2 = S.v3;
  S.v3 = x;
}

__device__ __forceinline__ Roots4 quartic_roots_01(const double c[5]) {
  Roots4 out;
  out.count = 0;
  out.r[0] = out.r[1] = out.r[2] = out.r[3] = 0.0;
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double a = fabs(c[i]);
    if (a > scale) scale = a;
  }
  if (scale == 0.0) return out;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  double eps = 1e-12 * scale;
  Slots4 S{INF, INF, INF, INF};
  if (fabs(c[4]) <= eps) {
    double a0 = 0.0, a1 = 0.0;
    int n = 0;
    Cubic3 cr{0.0, 0.0, 0.0, 0};
    if (fabs(c[3]) <= eps) {
      n = quad_roots(c[0], c[1], c[2], a0, a1);
      cr.r0 = a0;
      cr.r1 = a1;
      cr.n = n;
    } else {
      cr = cubic_roots3(c[0], c[1], c[2], c[3]);
    }
    if (cr.n > 0) push4(S, cr.r0);
    if (cr.n > 1) push4(S, cr.r1);
    if (cr.n > 2) push4(S, cr.r2);
  } else {
    double b3 = c[3] / c[4], b2 = c[2] / c[4], b1 = c[1] / c[4], b0 = c[0] / c[4];
    double p = b2 - 3.0 * b3 * b3 / 8.0;
    double q = b1 - b3 * b2 / 2.0 + pow3(b3) / 8.0;
    double r = b0 - b3 * b1 / 4.0 + b3 * b3 * b2 / 16.0 - 3.0 * pow4(b3) / 256.0;
    double off = -b3 / 4.0;
    double qscale = fabs(p) > 1.0 ? fabs(p) : 1.0;
    if (fabs(r) > qscale) qscale = fabs(r);
    if (fabs(q) <= 1e-14 * qscale) {
      // biquadratic in y^2: each nonnegative z gives +sqrt(z)+off, -sqrt(z)+off
      double z0 = 0.0, z1 = 0.0;
      int zn = quad_roots(r, p, 1.0, z0, z1);
#pragma unroll 1
      for (int i = 0; i < zn; ++i) {
        double z = (i == 0) ? z0 : z1;
        if (z >= 0.0) {
          double sq = sqrt(z);
          push4(S, sq + off);
          push4(S, -sq + off);
        }
      }
    } else {
      // resolvent cubic 8m^3 + 8p m^2 + (2p^2 - 8r) m - q^2 = 0
      double m = 0.0;
      const bool have = resolvent_max_root(-q * q, 2.0 * p * p - 8.0 * r, 8.0 * p, 8.0, m);
      if (have && m > 0.0) {
        double s = sqrt(2.0 * m);
#pragma unroll 1
        for (int j = 0; j < 2; ++j) {
          double cc0 = (j == 0) ? p / 2.0 + m - q / (2.0 * s) : p / 2.0 + m + q / (2.0 * s);
          double x0 = 0.0, x1 = 0.0;
          int nj = quad_roots(cc0, (j == 0) ? s : -s, 1.0, x0, x1);
          if (nj > 0) push4(S, x0 + off);
          if (nj > 1) push4(S, x1 + off);
        }
      }
    }
  }
  // polish, residual filter, clamp (_kernels.py:150-161); rolled: slot v0 is
  // processed, then the ring rotates, so after 4 steps the order is restored
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    double x = S.v0;
    if (x != INF) {
      x = polish_root(c[0], c[1], c[2], c[3], c[4], x);
      double f = c[0] + x * (c[1] + x * (c[2] + x * (c[3] + x * c[4])));
      if (fabs(f) <= 1e-9 * scale && -1e-12 <= x && x <= 1.0 + 1e-12) {
        if (x < 0.0) x = 0.0;
        else if (x > 1.0) x = 1.0;
      } else {
        x = INF;
      }
    }
    push4(S, x);  // rotate: v0 leaves the front, re-enters at the back
  }
  double cand[4] = {S.v0, S.v1, S.v2, S.v3};
  // stable sort (odd-even transposition) == compaction + insertion sort
  cex(cand[0], cand[1]);
  cex(cand[2], cand[3]);
  cex(cand[1], cand[2]);
  cex(cand[0], cand[1]);
  cex(cand[2], cand[3]);
  cex(cand[1], cand[2]);
  // dedup within 1e-10 against the last kept root (_kernels.py:170-175)
  double last = 0.0;
  int m = 0;
  double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double x = cand[i];
    if (x != INF && (m == 0 || x - last > 1e-10)) {
      o0 = (m == 0) ? x : o0;
      o1 = (m == 1) ? x : o1;
      o2 = (m == 2) ? x : o2;
      o3 = (m == 3) ? x : o3;
      last = x;
      ++m;
    }
  }
  out.r[0] = o0;
  out.r[1] = o1;
  out.r[2] = o2;
  out.r[3] = o3;
  out.count = m;
  return out;
}

// -------------------------------------------------- Bernstein ordinate ops
// _kernels.py:202-226, n = 5, all in registers
__device__ __forceinline__ void restrict_ordinates(const double (&b)[6], double lo, double hi,
                                                   double (&o)[6]) {
  double cur[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) cur[i] = b[i];
  if (lo > 0.0) {
    double tmp[6], right[6];
    right[5] = cur[5];
#pragma unroll
    for (int i = 0; i < 6; ++i) tmp[i] = cur[i];
#pragma unroll
    for (int k = 1; k <= 5; ++k) {
#pragma unroll
      for (int i = 0; i < 6 - k; ++i) tmp[i] = (1.0 - lo) * tmp[i] + lo * tmp[i + 1];
      right[5 - k] = tmp[5 - k];
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) cur[i] = right[i];
    hi = (hi - lo) / (1.0 - lo);
  }
  if (hi < 1.0) {
    double tmp[6], left[6];
    left[0] = cur[0];
#pragma unroll
    for (int i = 0; i < 6; ++i) tmp[i] = cur[i];
#pragma unroll
    for (int k = 1; k <= 5; ++k) {
#pragma unroll
      for (int i = 0; i < 6 - k; ++i) tmp[i] = (1.0 - hi) * tmp[i] + hi * tmp[i + 1];
      left[k] = tmp[0];
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) cur[i] = left[i];
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) o[i] = cur[i];
}

// _kernels.py:229-236
__device__ __forceinline__ double eval_ordinates(const double (&b)[6], double u) {
  double tmp[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) tmp[i] = b[i];
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int i = 0; i < 5 - k; ++i) tmp[i] = (1.0 - u) * tmp[i] + u * tmp[i + 1];
  return tmp[0];
}

#ifndef MREP_HULL_CARRY
#define MREP_HULL_CARRY 1
#endif
#ifndef MREP_HULL_MASK
#define MREP_HULL_MASK 1
#endif

// one chain edge (x0, y0) -> (x1, y1) of _kernels.py:285-297: its crossing of
// y = 0 (a zero end point, or the interpolated root), folded into [z1, z2]
__device__ __forceinline__ void hull_edge(double x0, double y0, double x1, double y1, double& z1,
                                          double& z2) {
  double z;
  bool hit = true;
  if (y0 == 0.0) z = x0;
  else if (y1 == 0.0) z = x1;
  else if ((y0 < 0.0 && 0.0 < y1) || (y1 < 0.0 && 0.0 < y0))
    z = x0 + (x1 - x0) * (-y0) / (y1 - y0);
  else {
    z = 0.0;
    hit = false;
  }
  if (hit) {
    if (z < z1) z1 = z;
    if (z > z2) z2 = z;
  }
}

// _kernels.py:239-303.  Monotone chains over (i/5, b_i); the stacks hold point
// indices, 3 bits per entry, so the chains stay in registers.
__device__ __forceinline__ bool hull_cross(const double (&b)[6], double& z1o, double& z2o) {
  uint32_t lo_st = 0, hi_st = 0;
  uint32_t lo_m = 0, hi_m = 0;  // chain members as bit sets (x-ordered: bit i = point i)
  int nl = 0, nh = 0;
  // the top two points of each chain are kept as values (a = top, c = the
  // one below); a pop fetches only the new second point.  Same tests on the
  // same operands as the reference, so the same chains.
  double lax = 0.0, lay = 0.0, lcx = 0.0, lcy = 0.0;
  double hax = 0.0, hay = 0.0, hcx = 0.0, hcy = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {  // unrolled: the new point is b[i] at x = i/5
    const double x = xs5(i), y = b[i];
    while (nl > 1) {
      if (((lax - lcx) * (y - lcy) - (x - lcx) * (lay - lcy)) <= 0.0) {
        lo_m &= ~(1u << ((lo_st >> (3 * (nl - 1))) & 7));
        --nl;
        lax = lcx;
        lay = lcy;
        if (nl > 1) {
          const int c = (lo_st >> (3 * (nl - 2))) & 7;
          lcx = xs5(c);
          lcy = sel6(b, c);
        }
      } else {
        break;
      }
    }
    lo_st = (lo_st & ~(7u << (3 * nl))) | ((uint32_t)i << (3 * nl));
    lo_m |= 1u << i;
    ++nl;
    lcx = lax;
    lcy = lay;
    lax = x;
    lay = y;
    while (nh > 1) {
      if (((hax - hcx) * (y - hcy) - (x - hcx) * (hay - hcy)) >= 0.0) {
        hi_m &= ~(1u << ((hi_st >> (3 * (nh - 1))) & 7));
        --nh;
        hax = hcx;
        hay = hcy;
        if (nh > 1) {
          const int c = (hi_st >> (3 * (nh - 2))) & 7;
          hcx = xs5(c);
          hcy = sel6(b, c);
        }
      } else {
        break;
      }
    }
    hi_st = (hi_st & ~(7u << (3 * nh))) | ((uint32_t)i << (3 * nh));
    hi_m |= 1u << i;
    ++nh;
    hcx = hax;
    hcy = hay;
    hax = x;
    hay = y;
  }
  double z1 = 2.0, z2 = -1.0;
#if MREP_HULL_MASK
  // the chains' edges walked with compile-time point indices: each chain runs
  // from point 0 to point 5 through its member bits, so an edge's end points
  // are registers (no stack decode, no select chain); the edges and their
  // operands are the reference's, and min / max do not depend on the order
#pragma unroll
  for (int chain = 0; chain < 2; ++chain) {
    const uint32_t mk = chain == 0 ? lo_m : hi_m;
    double px = 0.0, py = b[0];
#pragma unroll
    for (int i = 1; i < 6; ++i) {
      if ((mk >> i) & 1u) {
        hull_edge(px, py, xs5(i), b[i], z1, z2);
        px = xs5(i);
        py = b[i];
      }
    }
    // the last chain vertex is always point 5 (x = 1)
    if (b[5] == 0.0) {
      if (1.0 < z1) z1 = 1.0;
      if (1.0 > z2) z2 = 1.0;
    }
  }
#else
#pragma unroll 1
  for (int chain = 0; chain < 2; ++chain) {
    uint32_t st = chain == 0 ? lo_st : hi_st;
    int m = chain == 0 ? nl : nh;
#if MREP_HULL_CARRY
    // the chain starts at point 0; each edge's end is the next edge's start
    double x1 = 0.0, y1 = b[0];
    for (int i = 0; i < m - 1; ++i) {
      const int ib = (st >> (3 * (i + 1))) & 7;
      const double x0 = x1, y0 = y1;
      x1 = xs5(ib);
      y1 = sel6(b, ib);
#else
    for (int i = 0; i < m - 1; ++i) {
      int ia = (st >> (3 * i)) & 7, ib = (st >> (3 * (i + 1))) & 7;
      double x0 = xs5(ia), x1 = xs5(ib);
      double y0 = sel6(b, ia), y1 = sel6(b, ib);
#endif
      double z;
      bool hit = true;
      if (y0 == 0.0) z = x0;
      else if (y1 == 0.0) z = x1;
      else if ((y0 < 0.0 && 0.0 < y1) || (y1 < 0.0 && 0.0 < y0))
        z = x0 + (x1 - x0) * (-y0) / (y1 - y0);
      else {
        z = 0.0;
        hit = false;
      }
      if (hit) {
        if (z < z1) z1 = z;
        if (z > z2) z2 = z;
      }
    }
    // the last chain vertex is always point 5 (x = 1)
    if (m > 0 && b[5] == 0.0) {
      if (1.0 < z1) z1 = 1.0;
      if (1.0 > z2) z2 = 1.0;
    }
  }
#endif
  if (z2 < z1) {
    z1o = 0.0;
    z2o = 0.0;
    return false;
  }
  z1o = z1;
  z2o = z2;
  return true;
}

struct ClipOut {
  double root;
  double w3;  // widths[2] if max_iter > 2 else widths[max_iter - 1]
  double wf;  // widths[max_iter - 1]
  int used;
  bool ok;
};

// _kernels.py:306-341.  The widths array is tracked only at the two indices
// the batch kernel reads (i3 and max_iter-1), with the reference's fill rules.
// clip_root as an init + one-iteration step, so a solver can interleave
// many survivors per lane (wave_clip refills a lane when its survivor is
// done); clip_root below is exactly init + steps until finished.
struct ClipState {
  double cur[6];
  double lo, hi;
  int it;
  ClipOut r;
};

__device__ __forceinline__ void clip_init(ClipState& S, const double (&b)[6]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) S.cur[i] = b[i];
  S.lo = 0.0;
  S.hi = 1.0;
  S.it = 0;
  S.r.used = 0;
  S.r.w3 = 0.0;
  S.r.wf = 0.0;
  S.r.ok = false;
  S.r.root = 0.0;
}

// one iteration of _kernels.py:305-341; true when S.r is final
__device__ __forceinline__ bool clip_step(ClipState& S, double tol, int max_iter) {
  const int i3 = max_iter > 2 ? 2 : max_iter - 1;
  const int ilast = max_iter - 1;
  const int it = S.it;
  ClipOut& r = S.r;
  if (it >= max_iter) {
    r.ok = true;
    r.root = 0.5 * (S.lo + S.hi);
    return true;
  }
  double z1, z2;
  bool found = hull_cross(S.cur, z1, z2);
  if (!found) {
    // widths[k] = hi - lo for k >= it
    if (it <= i3) r.w3 = S.hi - S.lo;
    r.wf = S.hi - S.lo;
    r.ok = false;
    r.used = it;
    r.root = 0.5 * (S.lo + S.hi);
    return true;
  }
  r.used = it + 1;
  double nlo = S.lo + z1 * (S.hi - S.lo);
  double nhi = S.lo + z2 * (S.hi - S.lo);
  if (z2 - z1 < 1e-15) {
    if (it <= i3) r.w3 = 0.0;
    r.wf = 0.0;
    r.ok = true;
    r.root = nlo;
    return true;
  }
  restrict_ordinates(S.cur, z1, z2, S.cur);
  S.lo = nlo;
  S.hi = nhi;
  double w = S.hi - S.lo;
  if (it == i3) r.w3 = w;
  if (it == ilast) r.wf = w;
  if (w <= tol) {
    // widths[k] = w for k > it
    if (it < i3) r.w3 = w;
    if (it < ilast) r.wf = w;
    r.ok = true;
    r.root = 0.5 * (S.lo + S.hi);
    return true;
  }
  S.it = it + 1;
  if (S.it >= max_iter) {
    r.ok = true;
    r.root = 0.5 * (S.lo + S.hi);
    return true;
  }
  return false;
}

__device__ __forceinline__ ClipOut clip_root(const double (&b)[6], double tol, int max_iter) {
  ClipState S;
  clip_init(S, b);
#pragma unroll 1
  while (!clip_step(S, tol, max_iter)) {
  }
  return S.r;
}

// The reference's _T5 (power -> degree-5 Bernstein, basis.py:76-92):
// T[i][j] = C(i,j) / C(5,j); b = T e (_kernels.py:360-366, zero terms skipped)
__device__ __forceinline__ void rebase5(const double (&e)[6], double (&bo)[6]) {
  const double t10 = 1.0 / 1.0, t11 = 1.0 / 5.0;
  const double t20 = 1.0 / 1.0, t21 = 2.0 / 5.0, t22 = 1.0 / 10.0;
  const double t30 = 1.0 / 1.0, t31 = 3.0 / 5.0, t32 = 3.0 / 10.0, t33 = 1.0 / 10.0;
  const double t40 = 1.0 / 1.0, t41 = 4.0 / 5.0, t42 = 6.0 / 10.0, t43 = 4.0 / 10.0,
               t44 = 1.0 / 5.0;
  const double t50 = 1.0, t51 = 5.0 / 5.0, t52 = 10.0 / 10.0, t53 = 10.0 / 10.0, t54 = 5.0 / 5.0,
               t55 = 1.0;
  double acc;
  acc = 0.0;
  acc += 1.0 * e[0];
  bo[0] = acc;
  acc = 0.0;
  acc += t10 * e[0];
  acc += t11 * e[1];
  bo[1] = acc;
  acc = 0.0;
  acc += t20 * e[0];
  acc += t21 * e[1];
  acc += t22 * e[2];
  bo[2] = acc;
  acc = 0.0;
  acc += t30 * e[0];
  acc += t31 * e[1];
  acc += t32 * e[2];
  acc += t33 * e[3];
  bo[3] = acc;
  acc = 0.0;
  acc += t40 * e[0];
  acc += t41 * e[1];
  acc += t42 * e[2];
  acc += t43 * e[3];
  acc += t44 * e[4];
  bo[4] = acc;
  acc = 0.0;
  acc += t50 * e[0];
  acc += t51 * e[1];
  acc += t52 * e[2];
  acc += t53 * e[3];
  acc += t54 * e[4];
  acc += t55 * e[5];
  bo[5] = acc;
}

// _kernels.py:179-199 with the query-independent w_k = B3 P precomputed per
// segment (same expression, hoisted): w[k][dim]
template <int D>
__device__ __forceinline__ void distance_poly_w(const double (&w)[4][D], const double (&q)[D],
                                                double (&e)[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) e[k] = 0.0;
#pragma unroll
  for (int dim = 0; dim < D; ++dim) {
    double w0 = w[0][dim], w1 = w[1][dim], w2 = w[2][dim], w3 = w[3][dim];
    w0 -= q[dim];
    double d0 = w1, d1 = 2.0 * w2, d2 = 3.0 * w3;
    e[0] += 2.0 * w0 * d0;
    e[1] += 2.0 * (w0 * d1 + w1 * d0);
    e[2] += 2.0 * (w0 * d2 + w1 * d1 + w2 * d0);
    e[3] += 2.0 * (w1 * d2 + w2 * d1 + w3 * d0);
    e[4] += 2.0 * (w2 * d2 + w3 * d1);
    e[5] += 2.0 * w3 * d2;
  }
}

// _kernels.py:186-189: power coefficients of one coordinate of a cubic
__device__ __forceinline__ void cubic_power_coeffs(double p0, double p1, double p2, double p3,
                                                   double& w0, double& w1, double& w2,
                                                   double& w3) {
  w0 = 1.0 * p0 + 0.0 * p1 + 0.0 * p2 + 0.0 * p3;
  w1 = -3.0 * p0 + 3.0 * p1 + 0.0 * p2 + 0.0 * p3;
  w2 = 3.0 * p0 + -6.0 * p1 + 3.0 * p2 + 0.0 * p3;
  w3 = -1.0 * p0 + 3.0 * p1 + -3.0 * p2 + 1.0 * p3;
}

// _kernels.py:344-357
__device__ __forceinline__ double decasteljau1(double b0, double b1, double b2, double b3,
                                               double u) {
  b0 = (1.0 - u) * b0 + u * b1;
  b1 = (1.0 - u) * b1 + u * b2;
  b2 = (1.0 - u) * b2 + u * b3;
  b0 = (1.0 - u) * b0 + u * b1;
  b1 = (1.0 - u) * b1 + u * b2;
  return (1.0 - u) * b0 + u * b1;
}

}  // namespace mrep
