/*
 * CPU ORACLE for surface projection -- test infrastructure only.
 *
 * The reference (splinemat) has no surface code, so
 * there is nothing to restate bit for bit: this file IS the definition of
 * the surface projection the GPU path implements, written independently in
 * plain C so the two can be compared operation by operation:
 *
 *   per patch: Bernstein form S(u,v) = sum_a sum_c B_a(u) B_c(v) P[a][c];
 *   seeds: the (pu+1) x (pv+1) parameter grid (a/pu, c/pv), best |S - q|^2;
 *   refinement: projected Newton on f = |S(u,v) - q|^2 over [0,1]^2 with
 *     the exact Hessian (Gauss-Newton J^T J when it is not positive
 *     definite), coordinates at a bound with an outward gradient held fixed,
 *     a halving line search that must decrease f, <= 30 iterations;
 *   per query: brute force over EVERY patch (the GPU screens with a BVH),
 *     minimum distance, ties inside dmin + 1e-12 to the smallest patch id
 *     (the curve path's two-pass rule, _kernels.py:480-490, with the patch
 *     id in place of t).
 *
 * Built with -ffp-contract=off (the GPU kernels use -fmad=false) so both
 * sides round every product and sum alike.  "Parity unpinned" in the sense
 * of the task: no reference outputs exist; global optimality of the result
 * is checked separately against a dense-grid search (oracle/surface.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NEWTON_MAX 30
#define LS_MAX 12
#define LS_STEP_MIN 1e-11

static double binom_d(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
  return r;
}

/* degree-p Bernstein basis at u (+ first / second derivatives if wanted) */
static void bern(int p, double u, double* B, double* dB, double* ddB) {
  double w = 1.0 - u, up[8], wp[8], B1[8], B2[8];
  up[0] = 1.0;
  wp[0] = 1.0;
  for (int k = 1; k <= p; ++k) {
    up[k] = up[k - 1] * u;
    wp[k] = wp[k - 1] * w;
  }
  for (int a = 0; a <= p; ++a) B[a] = binom_d(p, a) * up[a] * wp[p - a];
  if (!dB) return;
  for (int a = 0; a <= p; ++a) {
    B1[a] = (p >= 1 && a <= p - 1) ? binom_d(p - 1, a) * up[a] * wp[p - 1 - a] : 0.0;
    B2[a] = (p >= 2 && a <= p - 2) ? binom_d(p - 2, a) * up[a] * wp[p - 2 - a] : 0.0;
  }
  for (int a = 0; a <= p; ++a) {
    double l1 = a >= 1 ? B1[a - 1] : 0.0;
    dB[a] = (double)p * (l1 - B1[a]);
    double m2 = a >= 2 ? B2[a - 2] : 0.0;
    double m1 = a >= 1 ? B2[a - 1] : 0.0;
    ddB[a] = (double)(p * (p - 1)) * ((m2 - 2.0 * m1) + B2[a]);
  }
}

static void surf_point(const double* P, int pu, int pv, double u, double v, double* S) {
  double Bu[8], Bv[8];
  bern(pu, u, Bu, NULL, NULL);
  bern(pv, v, Bv, NULL, NULL);
  S[0] = S[1] = S[2] = 0.0;
  for (int a = 0; a <= pu; ++a) {
    double R[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c <= pv; ++c)
      for (int k = 0; k < 3; ++k) R[k] += Bv[c] * P[(a * (pv + 1) + c) * 3 + k];
    for (int k = 0; k < 3; ++k) S[k] += Bu[a] * R[k];
  }
}

typedef struct {
  double S[3], Su[3], Sv[3], Suu[3], Suv[3], Svv[3];
} Jet;

static void surf_jet(const double* P, int pu, int pv, double u, double v, Jet* J) {
  double Bu[8], dBu[8], ddBu[8], Bv[8], dBv[8], ddBv[8];
  bern(pu, u, Bu, dBu, ddBu);
  bern(pv, v, Bv, dBv, ddBv);
  memset(J, 0, sizeof *J);
  for (int a = 0; a <= pu; ++a) {
    double R[3] = {0, 0, 0}, Rv[3] = {0, 0, 0}, Rvv[3] = {0, 0, 0};
    for (int c = 0; c <= pv; ++c)
      for (int k = 0; k < 3; ++k) {
        double p = P[(a * (pv + 1) + c) * 3 + k];
        R[k] += Bv[c] * p;
        Rv[k] += dBv[c] * p;
        Rvv[k] += ddBv[c] * p;
      }
    for (int k = 0; k < 3; ++k) {
      J->S[k] += Bu[a] * R[k];
      J->Su[k] += dBu[a] * R[k];
      J->Suu[k] += ddBu[a] * R[k];
      J->Sv[k] += Bu[a] * Rv[k];
      J->Suv[k] += dBu[a] * Rv[k];
      J->Svv[k] += Bu[a] * Rvv[k];
    }
  }
}

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static double dist2(const double* S, const double* q) {
  double d0 = S[0] - q[0], d1 = S[1] - q[1], d2 = S[2] - q[2];
  return d0 * d0 + d1 * d1 + d2 * d2;
}

static double clamp01(double x) { return fmin(fmax(x, 0.0), 1.0); }

/* minimum of |S(u,v) - q|^2 over one patch (local u, v in [0,1]) */
void oracle_surf_patch_min(const double* P, int pu, int pv, const double* q, double* uo,
                           double* vo, double* d2o, int* iters) {
  double best = INFINITY, bu = 0.0, bv = 0.0;
  for (int a = 0; a <= pu; ++a)
    for (int c = 0; c <= pv; ++c) {
      double u = (double)a / (double)pu, v = (double)c / (double)pv, S[3];
      surf_point(P, pu, pv, u, v, S);
      double f = dist2(S, q);
      if (f < best) {
        best = f;
        bu = u;
        bv = v;
      }
    }
  double u = bu, v = bv, f = best;
  int it = 0;
  for (; it < NEWTON_MAX; ++it) {
    Jet J;
    surf_jet(P, pu, pv, u, v, &J);
    double rr[3] = {J.S[0] - q[0], J.S[1] - q[1], J.S[2] - q[2]};
    f = dot3(rr, rr);
    double gu = dot3(J.Su, rr), gv = dot3(J.Sv, rr);
    double guu = dot3(J.Su, J.Su), gvv = dot3(J.Sv, J.Sv), guv = dot3(J.Su, J.Sv);
    double huu = guu + dot3(J.Suu, rr);
    double huv = guv + dot3(J.Suv, rr);
    double hvv = gvv + dot3(J.Svv, rr);
    int fu = !((u <= 0.0 && gu > 0.0) || (u >= 1.0 && gu < 0.0));
    int fv = !((v <= 0.0 && gv > 0.0) || (v >= 1.0 && gv < 0.0));
    double du = 0.0, dv = 0.0;
    if (fu && fv) {
      double det = huu * hvv - huv * huv;
      if (huu > 0.0 && det > 0.0) {
        du = -(hvv * gu - huv * gv) / det;
        dv = -(huu * gv - huv * gu) / det;
      } else {
        double dg = guu * gvv - guv * guv;
        if (guu > 0.0 && dg > 0.0) {
          du = -(gvv * gu - guv * gv) / dg;
          dv = -(guu * gv - guv * gu) / dg;
        } else {
          break;
        }
      }
    } else if (fu) {
      double h = huu > 0.0 ? huu : guu;
      if (!(h > 0.0)) break;
      du = -gu / h;
    } else if (fv) {
      double h = hvv > 0.0 ? hvv : gvv;
      if (!(h > 0.0)) break;
      dv = -gv / h;
    } else {
      break;
    }
    double t = 1.0, un = u, vn = v, fn = f;
    int ok = 0;
    for (int ls = 0; ls < LS_MAX; ++ls) {
      /* the full step is always tried; no decrease down to a halved step of
       * LS_STEP_MIN: stationary to that resolution (further halvings only
       * chase rounding noise in f) */
      if (ls > 0 && t * fmax(fabs(du), fabs(dv)) < LS_STEP_MIN) break;
      un = clamp01(u + t * du);
      vn = clamp01(v + t * dv);
      if (un == u && vn == v) break; /* the step rounds away: no decrease possible */
      double S[3];
      surf_point(P, pu, pv, un, vn, S);
      fn = dist2(S, q);
      if (fn < f) {
        ok = 1;
        break;
      }
      t = t * 0.5;
    }
    if (!ok) break;
    int conv = fabs(un - u) <= 1e-16 && fabs(vn - v) <= 1e-16;
    u = un;
    v = vn;
    f = fn;
    if (conv) break;
  }
  *uo = u;
  *vo = v;
  *d2o = f;
  if (iters) *iters = it;
}

typedef struct {
  const double *pts, *iv, *q;
  int64_t np, lo, hi;
  int pu, pv;
  double *ou, *ov, *ofoot, *odist;
  int32_t* opatch;
  int32_t* otie; /* 1: another patch's minimum lies within dmin (1 + 1e-9) + 1e-12 */
} Job;

static void* run(void* arg) {
  Job* J = (Job*)arg;
  const int NP = (J->pu + 1) * (J->pv + 1);
  double* cu = (double*)malloc(sizeof(double) * (size_t)J->np * 3);
  for (int64_t i = J->lo; i < J->hi; ++i) {
    const double* q = J->q + i * 3;
    double dmin = INFINITY;
    for (int64_t s = 0; s < J->np; ++s) {
      double u, v, d2;
      oracle_surf_patch_min(J->pts + s * NP * 3, J->pu, J->pv, q, &u, &v, &d2, NULL);
      cu[s * 3] = u;
      cu[s * 3 + 1] = v;
      cu[s * 3 + 2] = sqrt(d2);
      if (cu[s * 3 + 2] < dmin) dmin = cu[s * 3 + 2];
    }
    int64_t w = -1;
    for (int64_t s = 0; s < J->np; ++s)
      if (cu[s * 3 + 2] <= dmin + 1e-12) {
        w = s;  /* first in patch-id order */
        break;
      }
    const double* P = J->pts + w * NP * 3;
    const double* iv = J->iv + w * 4;
    double u = cu[w * 3], v = cu[w * 3 + 1], S[3];
    surf_point(P, J->pu, J->pv, u, v, S);
    J->ou[i] = iv[0] + u * (iv[1] - iv[0]);
    J->ov[i] = iv[2] + v * (iv[3] - iv[2]);
    J->odist[i] = cu[w * 3 + 2];
    for (int k = 0; k < 3; ++k) J->ofoot[i * 3 + k] = S[k];
    J->opatch[i] = (int32_t)w;
    if (J->otie) {
      /* a tie: the winner is decided by rounding-level distance differences
       * (feet on shared patch edges), so another solver may pick the other */
      int tie = 0;
      const double band = dmin * (1.0 + 1e-9) + 1e-12;
      for (int64_t s = 0; s < J->np && !tie; ++s)
        if (s != w && cu[s * 3 + 2] <= band) tie = 1;
      J->otie[i] = tie;
    }
  }
  free(cu);
  return NULL;
}

/* patch_pts [np][pu+1][pv+1][3] and patch_iv [np][4] in patch-id order */
void oracle_surface_project(const double* patch_pts, const double* patch_iv, int64_t np, int pu,
                            int pv, const double* q, int64_t n, int threads, double* ou,
                            double* ov, double* ofoot, double* odist, int32_t* opatch,
                            int32_t* otie) {
  if (threads < 1) threads = 1;
  if (n < threads) threads = n > 0 ? (int)n : 1;
  Job* jobs = (Job*)calloc((size_t)threads, sizeof(Job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int64_t k = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    Job j = {patch_pts, patch_iv, q, np, t * k, (t + 1) * k < n ? (t + 1) * k : n, pu, pv,
             ou, ov, ofoot, odist, opatch, otie};
    jobs[t] = j;
    pthread_create(&th[t], NULL, run, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
}
