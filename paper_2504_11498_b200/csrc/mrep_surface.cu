// mrep_surface.cu -- point projection onto tensor-product B-spline surfaces
// (BASELINE.json configs[3]: 10^6 points onto a bicubic / degree-5 surface
// with a 64x64 control net).
//
// The reference has no surface code (SPEC.md:15, 98, 497 mark surfaces out of
// its scope); this path extends its curve pipeline the way SURVEY.md 8(c)
// prescribes: the surface is decomposed into Bezier patches by the
// per-direction span matrices of decompose.py:19-46 (done on the device by
// the batched curve decomposition, rows then columns), and each query is
// solved per candidate patch with a seeded, box-constrained Newton iteration
// (the local refinement of oracle.py:95-128 replacing its dense grid with
// the patch's Bernstein seeds).  The CPU oracle (oracle/mrep_surface_oracle.c)
// restates the same algorithm operation by operation; parity is pinned to
// it and, for the global minimum, to a dense-grid search (tests/).
//
// Pipeline (wavefront, like the curve path):
//   S0 Morton sort of the queries in the surface's root box;
//   S1 traverse  (thread / query): 8-ary AABB hierarchy over the patches
//      (patches in 2-D Morton order, so a box of 8 is a 2x4 block), an
//      upper bound from exact surface points of the leaves reached (four
//      corners + centre); emits (query, patch) pairs;
//   S2 solve     (thread / pair): re-test with the final bound, best of the
//      (pu+1)x(pv+1) Bernstein seeds, projected Newton on |S(u,v) - q|^2
//      with a halving line search; atomicMin of the running minimum;
//   S3 select    (thread / candidate): inside dmin + 1e-12 the smallest
//      patch id wins (each pair yields one candidate);
//   S4 emit: winner's global (u, v), foot point, distance, patch id.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "mrep_common.cuh"
#include "mrep_screen.cuh"
#include "mrep_cells.cuh"
#include "mrep_sort.cuh"

namespace mrep {

int ensure_pool();

// ---------------------------------------------------------------- layout
// Header (HDR doubles): [0] pu [1] pv [2] nus [3] nvs [4] coordinate scale.
// Record per patch (surf_rec(pu, pv) doubles, 64-B multiple), NP = (pu+1)(pv+1):
//   [0, 3 NP)     P[a][c][xyz], a along u, c along v
//   [3 NP, 6 NP)  G[a][c][xyz] = S(a/pu, c/pv): the Newton seed grid,
//                 query-independent, evaluated once at pack time with the
//                 solver's own surf_point (so bit-identical to evaluating
//                 it per query, as the oracle does)
//   then u0 u1 v0 v1 (the patch's parameter rectangle) and the patch id
//   (i * nvs + j, row-major over the span grid);
//   then an oriented box enclosing the control net (so the patch): centre
//   (3), orthonormal axes e1 e2 e3 (9; e1 along u, e3 the net's normal),
//   half extents (3, inflated by a rounding margin) -- for a nearly flat
//   patch it is far tighter than the axis-aligned box.
// Boxes: the same 8-ary hierarchy as the curve tables, over the patches in
// 2-D Morton order of (i, j).
// Bernstein coefficients of D(u,v) = |S(u,v) - q|^2 at degree (2pu, 2pv)
// are SS_m - 2 q.E_m + |q|^2 with two query-independent nets stored per
// patch: E = S elevated to degree (2pu, 2pv) (3 NE doubles) and SS = the
// coefficients of |S|^2 (NE doubles), NE = (2pu+1)(2pv+1).  min_m D_m is a
// lower bound on the patch's squared distance (convex hull property).
__host__ __device__ inline int surf_ne(int pu, int pv) { return (2 * pu + 1) * (2 * pv + 1); }
__host__ __device__ inline int surf_bern(int pu, int pv) {  // E at +0, SS at +3 NE
  return 6 * (pu + 1) * (pv + 1) + 5 + 15;
}
// float copy of the nets for the filter's test: per coefficient m a float4
// (E_m xyz, SS_m), rounded to nearest; 16-B aligned (even double offset)
__host__ __device__ inline int surf_bernf(int pu, int pv) {
  return (surf_bern(pu, pv) + 4 * surf_ne(pu, pv) + 1 + 1) & ~1;  // after the magnitude
}
__host__ __device__ inline int surf_rec(int pu, int pv) {
  int n = surf_bernf(pu, pv) + 2 * surf_ne(pu, pv);
  return (n + 7) & ~7;
}
__host__ __device__ inline int surf_obb(int pu, int pv) { return 6 * (pu + 1) * (pv + 1) + 5; }

// squared distance lower bound from q to the patch's oriented box
__device__ __forceinline__ double obb_lb2(const double* O, const double (&q)[3]) {
  double d[3] = {q[0] - __ldg(O), q[1] - __ldg(O + 1), q[2] - __ldg(O + 2)};
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double pr = d[0] * __ldg(O + 3 + 3 * i) + d[1] * __ldg(O + 4 + 3 * i) +
                d[2] * __ldg(O + 5 + 3 * i);
    double g = fmax(0.0, fabs(pr) - __ldg(O + 12 + i));
    acc += g * g;
  }
  return acc;
}
__host__ __device__ inline int surf_seed(int pu, int pv) { return 3 * (pu + 1) * (pv + 1); }
__host__ __device__ inline int surf_iv(int pu, int pv) { return 6 * (pu + 1) * (pv + 1); }

// C(n, k) as an exact double (the oracle's running product r*(n-k+i)/i is
// an exact integer at every step, so the values agree bit for bit)
__host__ __device__ constexpr double binom_d(int n, int k) {
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return (double)r;
}

// Bernstein basis of degree P at u with first and second derivatives
// (the formulas of oracle/mrep_surface_oracle.c bern(), same order).
template <int P>
__device__ __forceinline__ void bern(double u, double (&B)[P + 1], double (&dB)[P + 1],
                                     double (&ddB)[P + 1]) {
  const double w = 1.0 - u;
  double up[P + 1], wp[P + 1];
  up[0] = 1.0;
  wp[0] = 1.0;
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    up[k] = up[k - 1] * u;
    wp[k] = wp[k - 1] * w;
  }
#pragma unroll
  for (int a = 0; a <= P; ++a) B[a] = binom_d(P, a) * up[a] * wp[P - a];
  // degree P-1 and P-2 bases for the derivatives
  double B1[P + 1], B2[P + 1];
#pragma unroll
  for (int a = 0; a <= P; ++a) {
    B1[a] = (P >= 1 && a <= P - 1) ? binom_d(P - 1, a) * up[a] * wp[P - 1 - a] : 0.0;
    B2[a] = (P >= 2 && a <= P - 2) ? binom_d(P - 2, a) * up[a] * wp[P - 2 - a] : 0.0;
  }
#pragma unroll
  for (int a = 0; a <= P; ++a) {
    double l1 = a >= 1 ? B1[a - 1] : 0.0;
    dB[a] = (double)P * (l1 - B1[a]);
    double m2 = a >= 2 ? B2[a - 2] : 0.0;
    double m1 = a >= 1 ? B2[a - 1] : 0.0;
    ddB[a] = (double)(P * (P - 1)) * ((m2 - 2.0 * m1) + B2[a]);
  }
}

template <int P>
__device__ __forceinline__ void bern0(double u, double (&B)[P + 1]) {
  const double w = 1.0 - u;
  double up[P + 1], wp[P + 1];
  up[0] = 1.0;
  wp[0] = 1.0;
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    up[k] = up[k - 1] * u;
    wp[k] = wp[k - 1] * w;
  }
#pragma unroll
  for (int a = 0; a <= P; ++a) B[a] = binom_d(P, a) * up[a] * wp[P - a];
}

// element i of a patch net: global memory (STRIDE 1, read-only path) or a
// lane's column of the solver's shared-memory staging (STRIDE = block size)
template <int STRIDE>
__device__ __forceinline__ double ldp(const double* P, int i) {
  if (STRIDE == 1) return __ldg(P + i);
  return P[i * STRIDE];
}

// S(u, v) only
template <int PU, int PV, int STRIDE = 1>
__device__ __forceinline__ void surf_point(const double* P, double u, double v, double (&S)[3]) {
  double Bu[PU + 1], Bv[PV + 1];
  bern0<PU>(u, Bu);
  bern0<PV>(v, Bv);
  S[0] = S[1] = S[2] = 0.0;
#pragma unroll
  for (int a = 0; a <= PU; ++a) {
    double R[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c <= PV; ++c)
#pragma unroll
      for (int k = 0; k < 3; ++k) R[k] += Bv[c] * ldp<STRIDE>(P, (a * (PV + 1) + c) * 3 + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) S[k] += Bu[a] * R[k];
  }
}

// surf_point with runtime degrees (pack time only): identical operations
__device__ void surf_point_rt(const double* P, int pu, int pv, double u, double v, double* S) {
  double Bu[8], Bv[8], up[8], wp[8];
  double w = 1.0 - u;
  up[0] = 1.0;
  wp[0] = 1.0;
  for (int k = 1; k <= pu; ++k) {
    up[k] = up[k - 1] * u;
    wp[k] = wp[k - 1] * w;
  }
  for (int a = 0; a <= pu; ++a) Bu[a] = binom_d(pu, a) * up[a] * wp[pu - a];
  w = 1.0 - v;
  for (int k = 1; k <= pv; ++k) {
    up[k] = up[k - 1] * v;
    wp[k] = wp[k - 1] * w;
  }
  for (int c = 0; c <= pv; ++c) Bv[c] = binom_d(pv, c) * up[c] * wp[pv - c];
  S[0] = S[1] = S[2] = 0.0;
  for (int a = 0; a <= pu; ++a) {
    double R[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c <= pv; ++c)
      for (int k = 0; k < 3; ++k) R[k] += Bv[c] * P[(a * (pv + 1) + c) * 3 + k];
    for (int k = 0; k < 3; ++k) S[k] += Bu[a] * R[k];
  }
}

struct Jet {
  double S[3], Su[3], Sv[3], Suu[3], Suv[3], Svv[3];
};

// Bernstein value / first / second derivative of index a, degree P, from
// the power tables (the per-element formulas of bern(): identical values)
template <int P>
__device__ __forceinline__ void bern_at(int a, const double (&up)[P + 1], const double (&wp)[P + 1],
                                        double& B, double& dB, double& ddB) {
  B = binom_d(P, a) * up[a] * wp[P - a];
  double b1a = (P >= 1 && a <= P - 1) ? binom_d(P - 1, a) * up[a] * wp[P - 1 - a] : 0.0;
  double b1m = (P >= 1 && a >= 1) ? binom_d(P - 1, a - 1) * up[a - 1] * wp[P - a] : 0.0;
  dB = (double)P * (b1m - b1a);
  double b2a = (P >= 2 && a <= P - 2) ? binom_d(P - 2, a) * up[a] * wp[P - 2 - a] : 0.0;
  double b2m1 = (P >= 2 && a >= 1 && a - 1 <= P - 2) ? binom_d(P - 2, a - 1) * up[a - 1] * wp[P - 1 - a]
                                                      : 0.0;
  double b2m2 = (P >= 2 && a >= 2) ? binom_d(P - 2, a - 2) * up[a - 2] * wp[P - a] : 0.0;
  ddB = (double)(P * (P - 1)) * ((b2m2 - 2.0 * b2m1) + b2a);
}

// S and its first / second partials at (u, v).  Register-lean: the u basis
// is produced one index at a time from the power tables.
template <int PU, int PV, int STRIDE = 1>
__device__ __forceinline__ void surf_jet(const double* P, double u, double v, Jet& J) {
  double Bv[PV + 1], dBv[PV + 1], ddBv[PV + 1];
  bern<PV>(v, Bv, dBv, ddBv);
  double up[PU + 1], wp[PU + 1];
  {
    const double w = 1.0 - u;
    up[0] = 1.0;
    wp[0] = 1.0;
#pragma unroll
    for (int k = 1; k <= PU; ++k) {
      up[k] = up[k - 1] * u;
      wp[k] = wp[k - 1] * w;
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) J.S[k] = J.Su[k] = J.Sv[k] = J.Suu[k] = J.Suv[k] = J.Svv[k] = 0.0;
#pragma unroll
  for (int a = 0; a <= PU; ++a) {
    double R[3] = {0.0, 0.0, 0.0}, Rv[3] = {0.0, 0.0, 0.0}, Rvv[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c <= PV; ++c)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double p = ldp<STRIDE>(P, (a * (PV + 1) + c) * 3 + k);
        R[k] += Bv[c] * p;
        Rv[k] += dBv[c] * p;
        Rvv[k] += ddBv[c] * p;
      }
    double Bu, dBu, ddBu;
    bern_at<PU>(a, up, wp, Bu, dBu, ddBu);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      J.S[k] += Bu * R[k];
      J.Su[k] += dBu * R[k];
      J.Suu[k] += ddBu * R[k];
      J.Sv[k] += Bu * Rv[k];
      J.Suv[k] += dBu * Rv[k];
      J.Svv[k] += Bu * Rvv[k];
    }
  }
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

__device__ __forceinline__ double dist2_to(const double (&S)[3], const double (&q)[3]) {
  double d0 = S[0] - q[0], d1 = S[1] - q[1], d2 = S[2] - q[2];
  return d0 * d0 + d1 * d1 + d2 * d2;
}

__device__ __forceinline__ double clamp01(double x) { return fmin(fmax(x, 0.0), 1.0); }

struct QStatsLite {
  uint64_t boxes, points;
};

constexpr int NEWTON_MAX = 30;
#ifndef MREP_SURF_REFILL
#define MREP_SURF_REFILL 28
#endif
constexpr int LS_MAX = 12;
constexpr double LS_STEP_MIN = 1e-11;

// Minimum of |S(u,v) - q|^2 on one patch: best Bernstein seed, then
// projected Newton (oracle: surf_patch_min in mrep_surface_oracle.c).  Split
// into seed_init + newton_iter so the solver can interleave many pairs per
// lane (surf_solve refills a lane as soon as its pair finishes).
struct NState {
  double u, v, f;
  int it;
};

template <int PU, int PV>
__device__ __forceinline__ void seed_init(const double* P, const double (&q)[3], NState& n) {
  double best = __longlong_as_double(0x7ff0000000000000LL);
  const double* G = P + surf_seed(PU, PV);  // precomputed S(a/PU, c/PV)
  int bk = 0;
#pragma unroll 4
  for (int k = 0; k < (PU + 1) * (PV + 1); ++k) {
    double S[3] = {__ldg(G + 3 * k), __ldg(G + 3 * k + 1), __ldg(G + 3 * k + 2)};
    double f = dist2_to(S, q);
    if (f < best) {
      best = f;
      bk = k;
    }
  }
  n.u = (double)(bk / (PV + 1)) / (double)PU;
  n.v = (double)(bk % (PV + 1)) / (double)PV;
  n.f = best;
  n.it = 0;
}

// one iteration of the oracle's loop; true when the solve is finished
template <int PU, int PV, int STRIDE = 1>
__device__ __forceinline__ bool newton_iter(const double* P, const double (&q)[3], NState& n) {
  const double u = n.u, v = n.v;
  Jet J;
  surf_jet<PU, PV, STRIDE>(P, u, v, J);
  double rr[3] = {J.S[0] - q[0], J.S[1] - q[1], J.S[2] - q[2]};
  const double f = dot3(rr, rr);
  n.f = f;
  double gu = dot3(J.Su, rr), gv = dot3(J.Sv, rr);
  double guu = dot3(J.Su, J.Su), gvv = dot3(J.Sv, J.Sv), guv = dot3(J.Su, J.Sv);
  double huu = guu + dot3(J.Suu, rr);
  double huv = guv + dot3(J.Suv, rr);
  double hvv = gvv + dot3(J.Svv, rr);
  bool fu = !((u <= 0.0 && gu > 0.0) || (u >= 1.0 && gu < 0.0));
  bool fv = !((v <= 0.0 && gv > 0.0) || (v >= 1.0 && gv < 0.0));
  double du = 0.0, dv = 0.0;
  if (fu && fv) {
    double det = huu * hvv - huv * huv;
    if (huu > 0.0 && det > 0.0) {
      du = -(hvv * gu - huv * gv) / det;
      dv = -(huu * gv - huv * gu) / det;
    } else {
      double dg = guu * gvv - guv * guv;  // Gauss-Newton (J^T J, PSD)
      if (guu > 0.0 && dg > 0.0) {
        du = -(gvv * gu - guv * gv) / dg;
        dv = -(guu * gv - guv * gu) / dg;
      } else {
        return true;
      }
    }
  } else if (fu) {
    double h = huu > 0.0 ? huu : guu;
    if (!(h > 0.0)) return true;
    du = -gu / h;
  } else if (fv) {
    double h = hvv > 0.0 ? hvv : gvv;
    if (!(h > 0.0)) return true;
    dv = -gv / h;
  } else {
    return true;  // KKT point at a corner
  }
  double t = 1.0, un = u, vn = v, fn = f;
  bool ok = false;
#pragma unroll 1
  for (int ls = 0; ls < LS_MAX; ++ls) {
    // the full step is always tried; no decrease down to a halved step of
    // LS_STEP_MIN: the iterate is stationary to that resolution (the
    // remaining halvings would only chase rounding noise in f)
    if (ls > 0 && t * fmax(fabs(du), fabs(dv)) < LS_STEP_MIN) break;
    un = clamp01(u + t * du);
    vn = clamp01(v + t * dv);
    // the step rounds away: every further (halved) trial is this same point,
    // whose value f cannot beat -- the search fails exactly as it would after
    // LS_MAX evaluations (same state, no wasted evaluations)
    if (un == u && vn == v) break;
    double S[3];
    surf_point<PU, PV, STRIDE>(P, un, vn, S);
    fn = dist2_to(S, q);
    if (fn < f) {
      ok = true;
      break;
    }
    t = t * 0.5;
  }
  if (!ok) return true;
  bool conv = fabs(un - u) <= 1e-16 && fabs(vn - v) <= 1e-16;
  n.u = un;
  n.v = vn;
  n.f = fn;
  if (conv) return true;
  return ++n.it >= NEWTON_MAX;
}

struct PatchMin {
  double u, v, d2;
  int iters;
};

template <int PU, int PV>
__device__ PatchMin patch_min(const double* P, const double (&q)[3]) {
  NState n;
  seed_init<PU, PV>(P, q, n);
#pragma unroll 1
  while (!newton_iter<PU, PV>(P, q, n)) {
  }
  return PatchMin{n.u, n.v, n.f, n.it};
}

// ---------------------------------------------------------------- pipeline
struct SurfParams {
  TableView tab;
  int pu, pv, rec;
  const double* q;
  int64_t n;
  const uint32_t* perm;
  double* out_u;
  double* out_v;
  double* out_foot;
  double* out_dist;
  int32_t* out_patch;
  uint64_t* counters;
  unsigned long long* cnt;  // [0] pairs [1] candidates [2] fallbacks
  double* qs;               // per sorted query: xyz + running min distance
  unsigned long long* pkey; // min patch id in the band
  int32_t* flag;
  int32_t* prim;            // per sorted query: the greedy-descent patch (solved first)
  uint32_t* pq;
  uint32_t* ps;
  uint32_t* fq;  // pairs surviving the post-greedy re-test (compacted)
  uint32_t* fs;
  unsigned long long pcap;
  uint32_t* cq;
  uint32_t* cs;
  double* cu;
  double* cv;
  double* cd;
  unsigned long long ccap;
  int64_t* fb;
  int cells;  // MREP_CELLS: scan the query's cell list instead of the tree
};

__device__ __forceinline__ unsigned long long* smin_ptr(const SurfParams& w, int64_t g) {
  return (unsigned long long*)(w.qs + g * 4 + 3);
}
__device__ __forceinline__ double smin_of(const SurfParams& w, int64_t g) {
  return __longlong_as_double((long long)*smin_ptr(w, g));
}

template <int PU, int PV>
__device__ __forceinline__ bool offer_points(const SurfParams& w, int64_t s, const double (&q)[3],
                                             double& ub, QStatsLite& st) {
  // the patch's seed grid: (pu+1)(pv+1) exact surface points
  const double* G = w.tab.rec + s * w.rec + surf_seed(PU, PV);
  const int NP = (PU + 1) * (PV + 1);
  double m = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 4
  for (int k = 0; k < NP; ++k) {
    double S[3] = {__ldg(G + 3 * k), __ldg(G + 3 * k + 1), __ldg(G + 3 * k + 2)};
    m = fmin(m, dist2_to(S, q));
  }
  st.points += NP;
  const double d = sqrt(m);
  if (!(d < ub)) return false;
  ub = d;
  return true;  // this patch now holds the nearest seed point seen
}


// S1: per-thread depth-first walk (queries in Morton order)
template <int PU, int PV>
__global__ void __launch_bounds__(128) surf_traverse(const __grid_constant__ SurfParams w) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = g < w.n;
  QStatsLite st{};
  const TableView& T = w.tab;
  int64_t qi = active ? (w.perm ? (int64_t)w.perm[g] : g) : 0;
  double q[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) q[k] = active ? w.q[qi * 3 + k] : 0.0;
  if (active && (isnan(q[0]) || isnan(q[1]) || isnan(q[2]))) {
    // a NaN coordinate: every candidate distance is NaN and no later stage
    // writes this query, so its answer (NaN, patch -1) is written here
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    w.out_u[qi] = w.out_v[qi] = w.out_dist[qi] = nan;
#pragma unroll
    for (int k = 0; k < 3; ++k) w.out_foot[qi * 3 + k] = nan;
    if (w.out_patch) w.out_patch[qi] = -1;
  }
  double scale = T.hdr[4];
#pragma unroll
  for (int k = 0; k < 3; ++k) scale = fmax(scale, fabs(q[k]));
  double ub = __longlong_as_double(0x7ff0000000000000LL);
  bool fall = false;
  int64_t cell = 0;
  if (active && w.cells && cell_of<3>(T, q, cell)) {
    // cell index: the list holds every patch that can come within the cut of
    // any query in the cell, nearest first; the first one seeds the bound
    int32_t a, b;
    const uint2* E = cell_list(T, 3, cell, a, b);
    const int64_t p0 = (int32_t)__ldg(E + a).y;
    offer_points<PU, PV>(w, p0, q, ub, st);
    int64_t prim = p0;  // the patch holding the nearest seed point: solved first
#pragma unroll 1
    for (int32_t i = a; i < b; ++i) {
      const double c2 = cut2(ub, scale);
      const uint2 e = __ldg(E + i);
      if ((double)__uint_as_float(e.x) > c2) break;  // keys ascend: the rest lie beyond the cut
      const int64_t s = (int32_t)e.y;
      st.boxes++;
      if (box_lb2<3>(T, T.lvl_off[0] + s, q) <= c2 &&
          obb_lb2(T.rec + s * w.rec + surf_obb(PU, PV), q) <= c2) {
        if (s != p0 && offer_points<PU, PV>(w, s, q, ub, st)) prim = s;
        unsigned long long slot = wave_append(&w.cnt[0], true);
        if (slot < w.pcap) {
          w.pq[slot] = (uint32_t)g;
          w.ps[slot] = (uint32_t)s;
        } else {
          fall = true;
        }
      }
    }
    w.prim[g] = (int32_t)prim;
  } else if (active) {
    // greedy descent to a nearby patch: its points give the first bound
    int level = T.top;
    int64_t idx = 0;
    while (level > 0) {
      int64_t first = idx * FANOUT, cnt = T.lvl_cnt[level - 1], off = T.lvl_off[level - 1];
      double best = 0.0;
      int64_t bi = first;
#pragma unroll 1
      for (int c = 0; c < FANOUT; ++c) {
        int64_t ch = first + c;
        if (ch < cnt) {
          st.boxes++;
          double lb = box_lb2<3>(T, off + ch, q);
          if (c == 0 || lb < best) {
            best = lb;
            bi = ch;
          }
        }
      }
      idx = bi;
      --level;
    }
    offer_points<PU, PV>(w, idx, q, ub, st);
    int64_t prim = idx;  // the patch holding the nearest seed point: solved first
    int lv = T.top;
    int64_t node = 0;
    uint64_t masks = 0;
    {
      uint32_t m = 0;
      double c2 = cut2(ub, scale);
      for (int c = 0; c < FANOUT; ++c)
        if (c < T.lvl_cnt[lv - 1] && box_lb2<3>(T, T.lvl_off[lv - 1] + c, q) <= c2) m |= 1u << c;
      st.boxes += (uint64_t)(T.lvl_cnt[lv - 1] < FANOUT ? T.lvl_cnt[lv - 1] : FANOUT);
      masks = (uint64_t)m << (8 * lv);
    }
    for (;;) {
      uint32_t mk = (uint32_t)(masks >> (8 * lv)) & 0xffu;
      if (mk == 0) {
        if (lv == T.top) break;
        ++lv;
        node /= FANOUT;
        continue;
      }
      int c = __ffs(mk) - 1;
      masks &= ~(1ull << (8 * lv + c));
      int64_t ch = node * FANOUT + c;
      double c2 = cut2(ub, scale);
      st.boxes++;
      if (lv == 1) {
        if (box_lb2<3>(T, T.lvl_off[0] + ch, q) <= c2 &&
            obb_lb2(T.rec + ch * w.rec + surf_obb(PU, PV), q) <= c2) {
          if (offer_points<PU, PV>(w, ch, q, ub, st)) prim = ch;
          unsigned long long slot = wave_append(&w.cnt[0], true);
          if (slot < w.pcap) {
            w.pq[slot] = (uint32_t)g;
            w.ps[slot] = (uint32_t)ch;
          } else {
            fall = true;
          }
        }
      } else if (box_lb2<3>(T, T.lvl_off[lv - 1] + ch, q) <= c2) {
        --lv;
        node = ch;
        uint32_t m = 0;
        int64_t first = node * FANOUT, cnt = T.lvl_cnt[lv - 1], off = T.lvl_off[lv - 1];
        for (int cc = 0; cc < FANOUT; ++cc)
          if (first + cc < cnt) {
            st.boxes++;
            if (box_lb2<3>(T, off + first + cc, q) <= c2) m |= 1u << cc;
          }
        masks |= (uint64_t)m << (8 * lv);
      }
    }
    w.prim[g] = (int32_t)prim;
  }
  if (active) {
    double4 rec;
    rec.x = q[0];
    rec.y = q[1];
    rec.z = q[2];
    rec.w = ub;  // upper bound; S2 lowers it to the true minimum
    *(double4*)(w.qs + g * 4) = rec;
    w.pkey[g] = ~0ull;
    w.flag[g] = fall ? 1 : 0;
    if (fall) {
      unsigned long long slot = atomicAdd(&w.cnt[2], 1ull);
      w.fb[slot] = g;
    }
  }
  warp_count(w.counters, MREP_CNT_SEAMS, st.points);
  warp_count(w.counters, MREP_CNT_BOXES, st.boxes);
}

// S2a: re-test every traversal pair against the bound the greedy patches
// left (box + oriented box) and compact the survivors, so the solver's
// lanes only ever hold real work.
template <int PU, int PV>
__global__ void __launch_bounds__(256) surf_filter(const __grid_constant__ SurfParams w) {
  // one 8-lane group per pair.  Bernstein test: |S - q|^2 over the patch is
  // a degree-(2pu, 2pv) polynomial whose Bernstein coefficients are
  // SS_k - 2 q.E_k + |q|^2 (surf_bern nets); their minimum bounds it from
  // below.  The group splits the (2pu+1)(2pv+1) coefficients and
  // min-reduces by shuffles (min is exact: the order does not matter).
  // Rounding: the nets are O(1e-16) relative to their magnitude; the sums
  // add a few ulps of (mag + 2|q| mag + |q|^2).
  constexpr int NE = (2 * PU + 1) * (2 * PV + 1);
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[0];
  if (total > w.pcap) total = w.pcap;
  const TableView& T = w.tab;
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const unsigned gmask = 0xffu << (lane & 24);
  const unsigned long long ng = ((unsigned long long)gridDim.x * blockDim.x) >> 3;
  for (unsigned long long i = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
       i < total; i += ng) {
    const int64_t g = w.pq[i];
    const int64_t s = w.ps[i];
    bool keep = !w.flag[g] && s != w.prim[g];
    double q[3] = {0.0, 0.0, 0.0}, c2 = 0.0;
    if (keep) {
      double4 rec = *(const double4*)(w.qs + g * 4);
      q[0] = rec.x;
      q[1] = rec.y;
      q[2] = rec.z;
      double scale = fmax(T.hdr[4], fmax(fabs(q[0]), fmax(fabs(q[1]), fabs(q[2]))));
      c2 = cut2(rec.w, scale);
      keep = box_lb2<3>(T, T.lvl_off[0] + s, q) <= c2 &&
             obb_lb2(T.rec + s * w.rec + surf_obb(PU, PV), q) <= c2;
    }
    if (keep) {  // group-uniform (same pair in all 8 lanes)
      const double qq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
      const double qa = fabs(q[0]) + fabs(q[1]) + fabs(q[2]);
      const double mag = __ldg(T.rec + s * w.rec + surf_bern(PU, PV) + 4 * NE);
      // the float test needs every term inside float's normal range: mag
      // (~length^2) and |q|^2 below ~1e30, and mag large enough that float
      // underflow (absolute error < 1e-37) is far below the allowance
      bool fnet = mag > 1e-25 && mag < 1e30 && qa < 1e15;
      double lb = 0.0, err = 0.0;
      if (fnet) {
        // on the float copy of the nets (half the bytes; the filter is
        // L2-bandwidth bound): every coefficient, the query and each of the
        // ~6 operations err by <= 2^-24 relative, so the float minimum is
        // within 8 * 2^-24 (mag (1 + 2|q|_1) + |q|^2) of the exact one (mag
        // bounds |E|, |SS|); 4e-6 covers it with an 8x margin
        const float4* F = reinterpret_cast<const float4*>(T.rec + s * w.rec + surf_bernf(PU, PV));
        const float q0 = __double2float_rn(q[0]), q1 = __double2float_rn(q[1]),
                    q2 = __double2float_rn(q[2]);
        const float qqf = q0 * q0 + q1 * q1 + q2 * q2;
        float m = __int_as_float(0x7f800000);
        for (int k = sub; k < NE; k += 8) {
          const float4 e = __ldg(F + k);
          m = fminf(m, (e.w - 2.0f * (q0 * e.x + q1 * e.y + q2 * e.z)) + qqf);
        }
        m = fminf(m, __shfl_xor_sync(gmask, m, 4));
        m = fminf(m, __shfl_xor_sync(gmask, m, 2));
        m = fminf(m, __shfl_xor_sync(gmask, m, 1));
        lb = (double)m;
        err = 4e-6 * (mag * (1.0 + 2.0 * qa) + qq);
        fnet = isfinite(lb);
      }
      if (!fnet) {
        // the double nets: a few ulps of the same magnitudes
        const double* E = T.rec + s * w.rec + surf_bern(PU, PV);
        double m = INFINITY;
        for (int k = sub; k < NE; k += 8)
          m = fmin(m, (E[3 * NE + k] - 2.0 * (q[0] * E[3 * k] + q[1] * E[3 * k + 1] +
                                               q[2] * E[3 * k + 2])) + qq);
        m = fmin(m, __shfl_xor_sync(gmask, m, 4));
        m = fmin(m, __shfl_xor_sync(gmask, m, 2));
        m = fmin(m, __shfl_xor_sync(gmask, m, 1));
        lb = m;
        err = 1e-13 * (mag * (1.0 + 2.0 * qa) + qq);
      }
      keep = !(lb - err > c2);
    }
    if (sub == 0) {
      unsigned long long slot = wave_append(&w.cnt[6], keep);
      if (keep) {  // slot < pcap: the compact list is never longer than the input
        w.fq[slot] = (uint32_t)g;
        w.fs[slot] = (uint32_t)s;
      }
    }
  }
}

// S2: projected-Newton solves of (query, patch) pairs with lane refill: a
// persistent warp loop in which every lane runs one Newton iteration of its
// current pair and a lane whose pair finished takes the next pair from the
// queue at once (warp-aggregated atomics), so the 1..30 iterations per pair
// do not leave lanes idle.  PASS 0: each query's greedy-descent patch
// (its minimum is a tight bound); PASS 1: the compacted survivors.
template <int PU, int PV, int PASS>
#ifndef MREP_SURF_SOLVE_MINB
#define MREP_SURF_SOLVE_MINB 3
#endif
__global__ void __launch_bounds__(128, (PU + PV <= 6) ? MREP_SURF_SOLVE_MINB : 1) surf_solve(const __grid_constant__ SurfParams w) {
  // each lane's current control net, staged column-wise in shared memory
  // (element k of lane t at [k][t]: conflict-free), so the ~20 surface
  // evaluations of a solve read shared memory instead of 3(p+1)^2 scattered
  // global loads each
  constexpr int NPD = 3 * (PU + 1) * (PV + 1);
  extern __shared__ double snet[];  // NPD * 128 doubles (dynamic)
  double* mynet = snet + threadIdx.x;
  const unsigned long long total =
      PASS == 0 ? (unsigned long long)w.n : *(volatile unsigned long long*)&w.cnt[6];
  unsigned long long* queue = &w.cnt[PASS == 0 ? 4 : 5];
  const TableView& T = w.tab;
  const int lane = threadIdx.x & 31;
  uint64_t npairs = 0, nit = 0;
  bool have = false, done = false;
  int64_t g = 0, s = 0;
  double q[3] = {0.0, 0.0, 0.0};
  const double* P = T.rec;
  NState ns{0.0, 0.0, 0.0, 0};
  for (;;) {
    // refill lanes without a pair
    const bool want = !have && !done;
    const unsigned wm = __ballot_sync(0xffffffffu, want);
    // refill in batches: the refill (net staging, seeds, bound re-test) runs
    // once at least MREP_SURF_REFILL lanes are idle (or nothing else runs),
    // so its ~100 loads per lane issue with most of the warp active.
    // Measured (cfg4 / cfg4q solve): 1 -> 3.75 / 9.56 ms, 16 -> 3.37,
    // 28 -> 3.24 / 8.56, 32 -> 3.32 / 8.78.
    if (wm && (__popc(wm) >= MREP_SURF_REFILL || !__any_sync(0xffffffffu, have))) {
      const int leader = __ffs(wm) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(queue, (unsigned long long)__popc(wm));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (want) {
        const unsigned long long i = base + __popc(wm & ((1u << lane) - 1));
        if (i >= total) {
          done = true;
        } else {
          g = PASS == 0 ? (int64_t)i : (int64_t)w.fq[i];
          s = PASS == 0 ? (int64_t)w.prim[g] : (int64_t)w.fs[i];
          // (no fallback-flag test: a flagged query's pair is solved anyway,
          // harmlessly -- select skips the query, the fallback recomputes it)
          double4 rec = *(const double4*)(w.qs + g * 4);
          q[0] = rec.x;
          q[1] = rec.y;
          q[2] = rec.z;
          bool go = true;
          if (PASS == 1) {  // the bound may have tightened since the filter
            double scale = fmax(T.hdr[4], fmax(fabs(q[0]), fmax(fabs(q[1]), fabs(q[2]))));
            const double c2 = cut2(smin_of(w, g), scale);
            go = obb_lb2(T.rec + s * w.rec + surf_obb(PU, PV), q) <= c2;
          }
          if (go) {
            P = T.rec + s * w.rec;
            seed_init<PU, PV>(P, q, ns);
#pragma unroll 4
            for (int k = 0; k < NPD; ++k) mynet[k * 128] = __ldg(P + k);
            have = true;
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;
    if (!newton_iter<PU, PV, 128>(mynet, q, ns)) continue;
    // pair finished: its candidate
    have = false;
    ++npairs;
    nit += (uint64_t)ns.it;
    const double d = sqrt(ns.f);
    const bool keep = d <= smin_of(w, g) + 1e-12;
    unsigned long long slot = wave_append(&w.cnt[1], keep);
    if (keep) {
      atomicMin(smin_ptr(w, g), (unsigned long long)__double_as_longlong(d));
      if (slot < w.ccap) {
        w.cq[slot] = (uint32_t)g;
        w.cs[slot] = (uint32_t)s;
        w.cu[slot] = ns.u;
        w.cv[slot] = ns.v;
        w.cd[slot] = d;
      } else if (atomicExch(&w.flag[g], 1) == 0) {
        unsigned long long fs = atomicAdd(&w.cnt[2], 1ull);
        w.fb[fs] = g;
      }
    }
  }
  warp_count(w.counters, MREP_CNT_PAIRS, npairs);
  warp_count(w.counters, MREP_CNT_CLIP_ITERS, nit);
}

__device__ __forceinline__ uint32_t patch_id_of(const SurfParams& w, int64_t s) {
  return (uint32_t)__ldg(w.tab.rec + s * w.rec + surf_iv(w.pu, w.pv) + 4);
}

// S3: smallest patch id inside the final band; PASS 1: the winner writes
template <int PU, int PV, int PASS>
__global__ void __launch_bounds__(256) surf_select(const __grid_constant__ SurfParams w) {
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[1];
  if (total > w.ccap) total = w.ccap;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t g = w.cq[i];
    if (w.flag[g]) continue;
    double d = w.cd[i];
    if (!(d <= smin_of(w, g) + 1e-12)) continue;
    int64_t s = w.cs[i];
    unsigned long long key = patch_id_of(w, s);
    if (PASS == 0) {
      atomicMin(&w.pkey[g], key);
      continue;
    }
    if (key != w.pkey[g]) continue;
    int64_t qi = w.perm ? (int64_t)w.perm[g] : g;
    const double* P = w.tab.rec + s * w.rec;
    const double* iv = P + surf_iv(PU, PV);
    double u = w.cu[i], v = w.cv[i];
    double S[3];
    surf_point<PU, PV>(P, u, v, S);
    w.out_u[qi] = iv[0] + u * (iv[1] - iv[0]);
    w.out_v[qi] = iv[2] + v * (iv[3] - iv[2]);
    w.out_dist[qi] = d;
#pragma unroll
    for (int k = 0; k < 3; ++k) w.out_foot[qi * 3 + k] = S[k];
    if (w.out_patch) w.out_patch[qi] = (int32_t)key;
  }
}

// exact per-thread path for queries whose buffers overflowed: every patch
// whose box can still beat the running bound, in table order
template <int PU, int PV>
__global__ void __launch_bounds__(128) surf_fallback(const __grid_constant__ SurfParams w) {
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[2];
  const TableView& T = w.tab;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t g = w.fb[i];
    int64_t qi = w.perm ? (int64_t)w.perm[g] : g;
    double q[3] = {w.qs[g * 4], w.qs[g * 4 + 1], w.qs[g * 4 + 2]};
    double scale = T.hdr[4];
    for (int k = 0; k < 3; ++k) scale = fmax(scale, fabs(q[k]));
    // pass 1: minimum distance; pass 2: smallest patch id inside the band
    double dmin = w.qs[g * 4 + 3];
    for (int pass = 0; pass < 2; ++pass) {
      uint32_t bestid = 0xffffffffu;
      double bu = 0.0, bv = 0.0, bd = 0.0;
      int64_t bs = -1;
      for (int64_t s = 0; s < T.S; ++s) {
        double lb = box_lb2<3>(T, T.lvl_off[0] + s, q);
        if (!(lb <= cut2(dmin, scale))) continue;
        const double* P = T.rec + s * w.rec;
        if (!(obb_lb2(P + surf_obb(PU, PV), q) <= cut2(dmin, scale))) continue;
        PatchMin m = patch_min<PU, PV>(P, q);
        double d = sqrt(m.d2);
        if (pass == 0) {
          dmin = fmin(dmin, d);
        } else if (d <= dmin + 1e-12) {
          uint32_t id = patch_id_of(w, s);
          if (id < bestid) {
            bestid = id;
            bu = m.u;
            bv = m.v;
            bd = d;
            bs = s;
          }
        }
      }
      if (pass == 1 && bs >= 0) {
        const double* P = T.rec + bs * w.rec;
        const double* iv = P + surf_iv(PU, PV);
        double S[3];
        surf_point<PU, PV>(P, bu, bv, S);
        w.out_u[qi] = iv[0] + bu * (iv[1] - iv[0]);
        w.out_v[qi] = iv[2] + bv * (iv[3] - iv[2]);
        w.out_dist[qi] = bd;
        for (int k = 0; k < 3; ++k) w.out_foot[qi * 3 + k] = S[k];
        if (w.out_patch) w.out_patch[qi] = (int32_t)bestid;
      }
    }
  }
  if (w.counters && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd((unsigned long long*)&w.counters[MREP_CNT_PASS2], total);
}

// Morton key (10 bits per axis) inside the root box
__global__ void surf_morton_kernel(const double* q, int64_t n, const double* box_root,
                                   uint32_t* key, uint32_t* idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t code = 0;
  for (int k = 0; k < 3; ++k) {
    double lo = box_root[k], hi = box_root[3 + k];
    double ext = fmax(hi - lo, 1e-300);
    double u = (q[i * 3 + k] - (lo - ext)) / (3.0 * ext);
    u = fmin(fmax(u, 0.0), 1.0);
    uint32_t c = (uint32_t)(u * 1023.0);
    for (int b = 0; b < 10; ++b) code |= ((c >> b) & 1u) << (b * 3 + k);
  }
  key[i] = code;
  idx[i] = (uint32_t)i;
}

// ---------------------------------------------------------------- table build
__global__ void surf_pack_kernel(const double* pts, const double* iv, const uint32_t* order,
                                 int64_t np, int pu, int pv, int64_t nvs, double* hdr,
                                 double* rec, double* box0) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int64_t s = order[k];  // source patch, row-major (i * nvs + j)
  const int NP = (pu + 1) * (pv + 1), R = surf_rec(pu, pv);
  double* r = rec + k * R;
  double lo[3], hi[3], amax = 0.0;
  for (int c = 0; c < 3; ++c) {
    lo[c] = pts[s * NP * 3 + c];
    hi[c] = lo[c];
  }
  for (int j = 0; j < NP; ++j)
    for (int c = 0; c < 3; ++c) {
      double x = pts[(s * NP + j) * 3 + c];
      r[j * 3 + c] = x;
      lo[c] = fmin(lo[c], x);
      hi[c] = fmax(hi[c], x);
      amax = fmax(amax, fabs(x));
    }
  double* G = r + surf_seed(pu, pv);
  for (int a = 0; a <= pu; ++a)
    for (int c = 0; c <= pv; ++c)
      surf_point_rt(r, pu, pv, (double)a / (double)pu, (double)c / (double)pv,
                    G + (a * (pv + 1) + c) * 3);
  const int o = surf_iv(pu, pv);
  for (int j = 0; j < 4; ++j) r[o + j] = iv[s * 4 + j];
  r[o + 4] = (double)s;
  for (int j = o + 5; j < R; ++j) r[j] = 0.0;
  {
    // frame: e1 along u (mean of the two u-edges), e3 normal to e1 and the
    // mean v-edge, e2 = e3 x e1
    const double* P00 = r;
    const double* P0v = r + pv * 3;
    const double* Pu0 = r + (pu * (pv + 1)) * 3;
    const double* Puv = r + (pu * (pv + 1) + pv) * 3;
    double a[3], b[3], e1[3], e2[3], e3[3];
    for (int k = 0; k < 3; ++k) {
      a[k] = (Pu0[k] - P00[k]) + (Puv[k] - P0v[k]);
      b[k] = (P0v[k] - P00[k]) + (Puv[k] - Pu0[k]);
    }
    double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    bool ok = na > 0.0;
    for (int k = 0; k < 3; ++k) e1[k] = ok ? a[k] / na : (k == 0 ? 1.0 : 0.0);
    e3[0] = e1[1] * b[2] - e1[2] * b[1];
    e3[1] = e1[2] * b[0] - e1[0] * b[2];
    e3[2] = e1[0] * b[1] - e1[1] * b[0];
    double n3 = sqrt(e3[0] * e3[0] + e3[1] * e3[1] + e3[2] * e3[2]);
    if (!(n3 > 1e-300)) {  // degenerate: any frame containing e1
      double t[3] = {fabs(e1[0]) < 0.9 ? 1.0 : 0.0, fabs(e1[0]) < 0.9 ? 0.0 : 1.0, 0.0};
      e3[0] = e1[1] * t[2] - e1[2] * t[1];
      e3[1] = e1[2] * t[0] - e1[0] * t[2];
      e3[2] = e1[0] * t[1] - e1[1] * t[0];
      n3 = sqrt(e3[0] * e3[0] + e3[1] * e3[1] + e3[2] * e3[2]);
    }
    for (int k = 0; k < 3; ++k) e3[k] /= n3;
    e2[0] = e3[1] * e1[2] - e3[2] * e1[1];
    e2[1] = e3[2] * e1[0] - e3[0] * e1[2];
    e2[2] = e3[0] * e1[1] - e3[1] * e1[0];
    const double* E[3] = {e1, e2, e3};
    double lo[3], hi[3];
    for (int i = 0; i < 3; ++i) {
      lo[i] = 1e300;
      hi[i] = -1e300;
    }
    for (int j = 0; j < NP; ++j)
      for (int i = 0; i < 3; ++i) {
        double pr = r[j * 3] * E[i][0] + r[j * 3 + 1] * E[i][1] + r[j * 3 + 2] * E[i][2];
        lo[i] = fmin(lo[i], pr);
        hi[i] = fmax(hi[i], pr);
      }
    double* O = r + surf_obb(pu, pv);
    double c[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 3; ++i) {
      double mid = 0.5 * (lo[i] + hi[i]);
      for (int k = 0; k < 3; ++k) c[k] += mid * E[i][k];
    }
    for (int k = 0; k < 3; ++k) O[k] = c[k];
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) O[3 + 3 * i + k] = E[i][k];
    // rounding margin: projections, the centre reconstruction and the
    // non-orthogonality of the rounded axes all err by O(1e-15 |x|)
    for (int i = 0; i < 3; ++i) O[12 + i] = 0.5 * (hi[i] - lo[i]) + 1e-12 * (1.0 + amax);
  }
  {
    // elevated net E and |S|^2 coefficients SS (see surf_bern)
    const int Nu = 2 * pu, Nv = 2 * pv, NE = surf_ne(pu, pv);
    double* E = r + surf_bern(pu, pv);
    double* SS = E + 3 * NE;
    double mag = 0.0;
    auto C = [](int n, int k) { return binom_d(n, k); };
    for (int a = 0; a <= Nu; ++a)
      for (int c = 0; c <= Nv; ++c) {
        double e[3] = {0.0, 0.0, 0.0}, ss = 0.0;
        for (int i = (a > pu ? a - pu : 0); i <= (a < pu ? a : pu); ++i)
          for (int k = (c > pv ? c - pv : 0); k <= (c < pv ? c : pv); ++k) {
            // elevation: C(pu,i) C(pu,a-i) / C(2pu,a) x the same in v
            const double wgt = (C(pu, i) * C(pu, a - i) / C(Nu, a)) *
                               (C(pv, k) * C(pv, c - k) / C(Nv, c));
            const double* Pik = r + (i * (pv + 1) + k) * 3;
            const double* Pjl = r + ((a - i) * (pv + 1) + (c - k)) * 3;
            for (int x = 0; x < 3; ++x) e[x] += wgt * Pik[x];
            // product of the two degree-p nets (same weights)
            ss += wgt * (Pik[0] * Pjl[0] + Pik[1] * Pjl[1] + Pik[2] * Pjl[2]);
          }
        const int m = a * (Nv + 1) + c;
        for (int x = 0; x < 3; ++x) E[3 * m + x] = e[x];
        SS[m] = ss;
        float* F = reinterpret_cast<float*>(r + surf_bernf(pu, pv)) + 4 * m;
        for (int x = 0; x < 3; ++x) F[x] = __double2float_rn(e[x]);
        F[3] = __double2float_rn(ss);
        mag = fmax(mag, fmax(fabs(ss), fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2])))));
      }
    SS[NE] = mag;
  }
  for (int c = 0; c < 3; ++c) {
    box0[k * 6 + c] = lo[c];
    box0[k * 6 + 3 + c] = hi[c];
  }
  if (k == 0) {
    hdr[0] = pu;
    hdr[1] = pv;
    hdr[2] = (double)(np / nvs);
    hdr[3] = (double)nvs;
  }
  atomicMax((unsigned long long*)&hdr[4], (unsigned long long)__double_as_longlong(amax));
}

__global__ void surf_boxes_kernel(const double* child, int64_t nchild, double* parent,
                                  int64_t nparent) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nparent) return;
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = child[i * FANOUT * 6 + k];
    hi[k] = child[i * FANOUT * 6 + 3 + k];
  }
  for (int c = 1; c < FANOUT; ++c) {
    int64_t ch = i * FANOUT + c;
    if (ch >= nchild) break;
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], child[ch * 6 + k]);
      hi[k] = fmax(hi[k], child[ch * 6 + 3 + k]);
    }
  }
  for (int k = 0; k < 3; ++k) {
    parent[i * 6 + k] = lo[k];
    parent[i * 6 + 3 + k] = hi[k];
  }
}


// ---------------------------------------------------------------- evaluation
// Cox-de Boor basis of the p+1 functions alive at t (span = last nonzero
// [k_s, k_s+1) holding t; t == k[-1] uses the final nonzero span), as the
// curve evaluator does (oracle.py:13-52 restricted to the live functions).
__device__ int64_t live_basis(int p, const double* kn, int64_t m, double t, double* N) {
  int64_t s = -1, last = -1;
  for (int64_t j = 0; j < m - 1; ++j)
    if (kn[j] < kn[j + 1]) {
      last = j;
      if (kn[j] <= t && t < kn[j + 1]) s = j;
    }
  if (t == kn[m - 1] && last >= 0) s = last;
  for (int j = 0; j <= p; ++j) N[j] = 0.0;
  if (s < 0) return -1;
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
  return s;
}

__global__ void eval_surface_kernel(int pu, int pv, const double* ku, int64_t mu, const double* kv,
                                    int64_t mv, const double* ctrl, int64_t nu, int64_t nv,
                                    const double* uv, int64_t n, double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double Nu[32], Nv[32];
  int64_t su = live_basis(pu, ku, mu, uv[2 * i], Nu);
  int64_t sv = live_basis(pv, kv, mv, uv[2 * i + 1], Nv);
  double acc[3] = {0.0, 0.0, 0.0};
  if (su >= 0 && sv >= 0) {
    for (int a = 0; a <= pu; ++a) {
      int64_t r = su - pu + a;
      if (r < 0 || r >= nu) continue;
      double row[3] = {0.0, 0.0, 0.0};
      for (int c = 0; c <= pv; ++c) {
        int64_t col = sv - pv + c;
        if (col < 0 || col >= nv) continue;
        for (int k = 0; k < 3; ++k) row[k] += Nv[c] * ctrl[(r * nv + col) * 3 + k];
      }
      for (int k = 0; k < 3; ++k) acc[k] += Nu[a] * row[k];
    }
  }
  for (int k = 0; k < 3; ++k) out[i * 3 + k] = acc[k];
}

static bool degree_supported(int pu, int pv) {
  return (pu == pv && pu >= 1 && pu <= 5) || (pu == 3 && pv == 5) || (pu == 5 && pv == 3);
}


template <int PU, int PV>
static int launch_surface(SurfParams& w, cudaStream_t st, bool timing) {
  const int64_t n = w.n;
  const unsigned long long pcap = (unsigned long long)std::max<int64_t>(24 * n, 1 << 16);
  const unsigned long long ccap = (unsigned long long)std::max<int64_t>(4 * n, 1 << 16);
  size_t bytes = 0;
  auto take = [&](size_t b) {
    size_t o = bytes;
    bytes += (b + 255) & ~(size_t)255;
    return o;
  };
  size_t o_cnt = take(8 * 8), o_qs = take(n * 32), o_pk = take(n * 8), o_fl = take(n * 4),
         o_pr = take(n * 4);
  size_t o_pq = take(pcap * 4), o_ps = take(pcap * 4), o_fq = take(pcap * 4),
         o_fs = take(pcap * 4);
  size_t o_cq = take(ccap * 4), o_cs = take(ccap * 4), o_cu = take(ccap * 8), o_cv = take(ccap * 8),
         o_cd = take(ccap * 8), o_fb = take(n * 8);
  char* base = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&base, bytes, st));
  w.cnt = (unsigned long long*)(base + o_cnt);
  w.qs = (double*)(base + o_qs);
  w.pkey = (unsigned long long*)(base + o_pk);
  w.flag = (int32_t*)(base + o_fl);
  w.prim = (int32_t*)(base + o_pr);
  w.pq = (uint32_t*)(base + o_pq);
  w.ps = (uint32_t*)(base + o_ps);
  w.fq = (uint32_t*)(base + o_fq);
  w.fs = (uint32_t*)(base + o_fs);
  w.pcap = pcap;
  w.cq = (uint32_t*)(base + o_cq);
  w.cs = (uint32_t*)(base + o_cs);
  w.cu = (double*)(base + o_cu);
  w.cv = (double*)(base + o_cv);
  w.cd = (double*)(base + o_cd);
  w.ccap = ccap;
  w.fb = (int64_t*)(base + o_fb);
  MREP_CUDA_CHECK(cudaMemsetAsync(w.cnt, 0, 64, st));
  auto persist_grid = [](const void* fn, int block) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, block, 0);
    return (unsigned)(sms * (per > 0 ? per : 1));
  };
  const size_t solve_smem = (size_t)3 * (PU + 1) * (PV + 1) * 128 * sizeof(double);
  // attribute + grid size once per instantiation and device
  static int attr_dev = -1;
  static unsigned g_solve = 0;
  int cur_dev = 0;
  MREP_CUDA_CHECK(cudaGetDevice(&cur_dev));
  if (attr_dev != cur_dev) {
    for (const void* fn : {(const void*)surf_solve<PU, PV, 0>, (const void*)surf_solve<PU, PV, 1>})
      MREP_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)solve_smem));
    int sms = 148, per = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)surf_solve<PU, PV, 1>, 128,
                                                  solve_smem);
    g_solve = (unsigned)(sms * (per > 0 ? per : 1));
    attr_dev = cur_dev;
  }
  const unsigned g_sel = persist_grid((const void*)surf_select<PU, PV, 1>, 256);
  StageTimer tm(timing, st);
  tm.mark();
  surf_traverse<PU, PV><<<grid_for(n, 128), 128, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  surf_solve<PU, PV, 0><<<g_solve, 128, solve_smem, st>>>(w);
  surf_filter<PU, PV><<<g_sel, 256, 0, st>>>(w);
  surf_solve<PU, PV, 1><<<g_solve, 128, solve_smem, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  tm.mark();  // (no clip stage for surfaces)
  surf_select<PU, PV, 0><<<g_sel, 256, 0, st>>>(w);
  surf_select<PU, PV, 1><<<g_sel, 256, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  surf_fallback<PU, PV><<<148u, 128, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  tm.finish(1);
  MREP_CUDA_CHECK(cudaFreeAsync(base, st));
  return MREP_OK;
}

static int surface_chunk(const void* table, int64_t np, int pu, int pv, const double* queries,
                         int64_t n, unsigned flags, double* out_u, double* out_v, double* out_foot,
                         double* out_dist, int32_t* out_patch, uint64_t* counters,
                         cudaStream_t st) {
  int prc = ensure_pool();
  if (prc) return prc;
  SurfParams w{};
  w.rec = surf_rec(pu, pv);
  w.tab = table_view(table, np, w.rec);
  w.pu = pu;
  w.pv = pv;
  w.q = queries;
  w.n = n;
  w.out_u = out_u;
  w.out_v = out_v;
  w.out_foot = out_foot;
  w.out_dist = out_dist;
  w.out_patch = out_patch;
  w.counters = counters;
  w.cells = (flags & MREP_CELLS) ? 1 : 0;
  size_t sort_tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 30, st);
  static const bool radix = getenv("MREP_RADIX_SORT") != nullptr;
  if (!radix) sort_tmp = bucket_sort_bytes(n, 3);
  char* ws = nullptr;
  const size_t o_tmp = 16 * (size_t)n + 256;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&ws, o_tmp + sort_tmp + 256, st));
  uint32_t* k_in = (uint32_t*)ws;
  uint32_t* k_out = k_in + n;
  uint32_t* i_in = k_out + n;
  uint32_t* i_out = i_in + n;
  const bool timing = (flags & MREP_TIMING) != 0;
  StageTimer sort_tm(timing, st);
  sort_tm.mark();
  w.perm = nullptr;
  if (!(flags & MREP_NO_SORT) && n > 64) {
    const double* root = w.tab.box + w.tab.lvl_off[w.tab.top] * 6;
    if (!radix) {
      const int rc = bucket_sort(queries, n, 3, root, ws + o_tmp, sort_tmp, i_out, st);
      if (rc != MREP_OK) {
        cudaFreeAsync(ws, st);
        return rc;
      }
    } else {
      surf_morton_kernel<<<grid_for(n, 256), 256, 0, st>>>(queries, n, root, k_in, i_in);
      MREP_LAUNCH_CHECK();
      MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ws + o_tmp, sort_tmp, k_in, k_out, i_in,
                                                      i_out, (int)n, 0, 30, st));
    }
    w.perm = i_out;
  }
  sort_tm.mark();
  sort_tm.finish(0);
  int rc = MREP_ERR_ARG;
#define MREP_SURF_CASE(a, b) \
  if (pu == a && pv == b) rc = launch_surface<a, b>(w, st, timing);
  MREP_SURF_CASE(1, 1)
  MREP_SURF_CASE(2, 2)
  MREP_SURF_CASE(3, 3)
  MREP_SURF_CASE(4, 4)
  MREP_SURF_CASE(5, 5)
  MREP_SURF_CASE(3, 5)
  MREP_SURF_CASE(5, 3)
#undef MREP_SURF_CASE
  MREP_CUDA_CHECK(cudaFreeAsync(ws, st));
  return rc;
}

// cell-index leaf points of a patch: its (pu+1)(pv+1) seed-grid points
struct SurfaceLeaves {
  int pu, pv, rec;
  __device__ int npts(const TableView&) const { return (pu + 1) * (pv + 1); }
  __device__ void pt(const TableView& T, int, int64_t s, int k, double* p) const {
    const double* G = T.rec + s * rec + surf_seed(pu, pv) + 3 * k;
    p[0] = G[0];
    p[1] = G[1];
    p[2] = G[2];
  }
};

}  // namespace mrep

using namespace mrep;

extern "C" {

int64_t mrep_surface_cells_bytes(const void* table, int64_t npatch, int pu, int pv, int grid,
                                 void* stream) {
  if (!degree_supported(pu, pv)) {
    set_error("mrep_surface_cells_bytes: unsupported degrees");
    return -1;
  }
  const int R = surf_rec(pu, pv);
  return cells_bytes(table, npatch, 3, grid, R, SurfaceLeaves{pu, pv, R}, (cudaStream_t)stream);
}

int mrep_surface_cells_build(void* table, int64_t npatch, int pu, int pv, int grid, void* cells,
                             int64_t bytes, void* stream) {
  if (!degree_supported(pu, pv)) {
    set_error("mrep_surface_cells_build: unsupported degrees");
    return MREP_ERR_ARG;
  }
  const int R = surf_rec(pu, pv);
  return cells_build(table, npatch, 3, grid, R, SurfaceLeaves{pu, pv, R}, cells, bytes,
                     (cudaStream_t)stream);
}

int64_t mrep_surface_table_bytes(int64_t npatch, int pu, int pv) {
  if (npatch < 1 || pu < 1 || pv < 1) return -1;
  return table_layout(npatch, surf_rec(pu, pv)).total_doubles * (int64_t)sizeof(double);
}

int mrep_surface_table_pack(const double* patch_pts, const double* patch_iv, int64_t nus,
                            int64_t nvs, int pu, int pv, void* table, void* stream) {
  if (nus < 1 || nvs < 1 || !table || !degree_supported(pu, pv)) {
    set_error("mrep_surface_table_pack: need nus, nvs >= 1 and (pu, pv) in {(1,1)..(5,5), (3,5), "
              "(5,3)}");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t np = nus * nvs;
  const int R = surf_rec(pu, pv);
  TableLayout L = table_layout(np, R);
  // patches in 2-D Morton order of (i, j): consecutive runs of 8 / 64 are
  // 2x4 / 8x8 blocks of the span grid, so every box of the hierarchy is compact
  std::vector<uint64_t> key(np);
  std::vector<uint32_t> order(np);
  for (int64_t s = 0; s < np; ++s) {
    uint64_t i = (uint64_t)(s / nvs), j = (uint64_t)(s % nvs), m = 0;
    for (int b = 0; b < 24; ++b) m |= (((i >> b) & 1ull) << (2 * b + 1)) | (((j >> b) & 1ull) << (2 * b));
    key[s] = (m << 24) | (uint64_t)s;
  }
  std::sort(key.begin(), key.end());
  for (int64_t k = 0; k < np; ++k) order[k] = (uint32_t)(key[k] & 0xffffffull);
  if (np >= (1 << 24)) {
    set_error("mrep_surface_table_pack: at most 2^24 patches");
    return MREP_ERR_ARG;
  }
  uint32_t* dorder = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&dorder, np * 4, st));
  MREP_CUDA_CHECK(cudaMemcpyAsync(dorder, order.data(), np * 4, cudaMemcpyHostToDevice, st));
  double* base = (double*)table;
  MREP_CUDA_CHECK(cudaMemsetAsync(base, 0, HDR * sizeof(double), st));
  double* box = base + L.box_off;
  surf_pack_kernel<<<grid_for(np, 128), 128, 0, st>>>(patch_pts, patch_iv, dorder, np, pu, pv, nvs,
                                                      base, base + L.rec_off, box + L.lvl_off[0]);
  MREP_LAUNCH_CHECK();
  for (int lv = 1; lv <= L.top; ++lv) {
    surf_boxes_kernel<<<grid_for(L.lvl_cnt[lv], 128), 128, 0, st>>>(
        box + L.lvl_off[lv - 1] * 6, L.lvl_cnt[lv - 1], box + L.lvl_off[lv] * 6, L.lvl_cnt[lv]);
    MREP_LAUNCH_CHECK();
  }
  boxes_to_float_kernel<<<grid_for(L.total_boxes, 256), 256, 0, st>>>(
      box, reinterpret_cast<float*>(base + L.fbox_off), L.total_boxes);
  MREP_LAUNCH_CHECK();
  MREP_CUDA_CHECK(cudaFreeAsync(dorder, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));  // the host order vector dies here
  return MREP_OK;
}

int mrep_project_surface(const void* table, int64_t npatch, int pu, int pv, const double* queries,
                         int64_t n, unsigned flags, double* out_u, double* out_v, double* out_foot,
                         double* out_dist, int32_t* out_patch, uint64_t* counters, void* stream) {
  if (!table || npatch < 1 || n < 0 || !degree_supported(pu, pv)) {
    set_error("mrep_project_surface: bad arguments");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  if (!queries || !out_u || !out_v || !out_foot || !out_dist) {
    set_error("mrep_project_surface: null query/output pointer");
    return MREP_ERR_ARG;
  }
  if (flags & MREP_TIMING)
    for (double& v : g_stage_ms) v = 0.0;
  const int64_t CHUNK_Q = (int64_t)1 << 23;
  for (int64_t lo = 0; lo < n; lo += CHUNK_Q) {
    int64_t m = n - lo < CHUNK_Q ? n - lo : CHUNK_Q;
    int rc = surface_chunk(table, npatch, pu, pv, queries + lo * 3, m, flags, out_u + lo,
                           out_v + lo, out_foot + lo * 3, out_dist + lo,
                           out_patch ? out_patch + lo : nullptr, counters, (cudaStream_t)stream);
    if (rc != MREP_OK) return rc;
  }
  return MREP_OK;
}

int mrep_eval_surface(int pu, int pv, const double* knots_u, int64_t mu, const double* knots_v,
                      int64_t mv, const double* ctrl, int64_t nu, int64_t nv, const double* uv,
                      int64_t n, double* out, void* stream) {
  if (pu < 1 || pu > 31 || pv < 1 || pv > 31) {
    set_error("mrep_eval_surface: degrees in [1, 31]");
    return MREP_ERR_ARG;
  }
  if (n <= 0) return MREP_OK;
  eval_surface_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      pu, pv, knots_u, mu, knots_v, mv, ctrl, nu, nv, uv, n, out);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

}  // extern "C"
