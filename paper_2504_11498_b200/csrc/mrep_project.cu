// mrep_project.cu -- batch point projection onto one prepared curve (sm_100a).
//
// Replaces the reference's fused per-query loop _kernels._project_block
// (/root/reference/pkg/src/splinemat/_kernels.py:369-502) as driven by
// project_prepared (project.py:245-289).
//
// Mapping: one query per thread; the per-(query, cubic) solve is the
// register-resident routine chain of mrep_math.cuh on the FP64 pipe.
// Two modes share the candidate generator:
//   dense  (reference semantics): every seam and every cubic, with the six
//          per-query stats columns and the soundness minimum;
//   screen (MREP_SCREEN): an 8-ary AABB hierarchy over the cubics prunes
//          every cubic whose box lower bound exceeds the running best
//          candidate distance + the 1e-12 tie band (+ a rounding margin), so
//          the winner -- and t, foot, dist, segment -- is the one dense mode
//          finds; only the candidate count differs (documented in DESIGN.md).
// Reduction: the reference's two-pass "min distance, then min t inside
// dmin + 1e-12" (_kernels.py:480-490) is made streaming and order-free with a
// 4-slot tie-band buffer keyed by each candidate's position in the
// reference's candidate order; if more than 4 candidates share the band, the
// query is re-run in an exact second pass with the final dmin.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "mrep_common.cuh"
#include "mrep_math.cuh"
#include "mrep_screen.cuh"
#include "mrep_cells.cuh"
#include "mrep_sort.cuh"

namespace mrep {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

thread_local double g_stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};

// Keep stream-ordered allocations cached in the device's default pool: the
// projection workspace is re-requested on every call, and releasing it at each
// synchronisation would re-map hundreds of MB per call.
static std::mutex g_pool_mu;
static int g_pool_dev_mask = 0;
int ensure_pool() {
  int dev = 0;
  MREP_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 31 && (g_pool_dev_mask & (1 << dev))) return MREP_OK;
  cudaMemPool_t pool;
  MREP_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~0ull;
  MREP_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  if (dev < 31) g_pool_dev_mask |= 1 << dev;
  return MREP_OK;
}

constexpr uint64_t SURV_BIT = 1ull << 62;
constexpr int BAND_K = 4;
constexpr int LIST_CAP = 32;
constexpr int BLOCK = 128;
// resident blocks per SM the wave kernels are compiled for (register caps:
// 65536 / (128 x minb) per thread; measured on cfg2: 0.865 vs 0.958 ms for
// the uncapped 80-96 registers, despite small spills)
#ifndef MREP_TRAV_MINB
#define MREP_TRAV_MINB 6
#endif
#ifndef MREP_GROUP_MINB
#define MREP_GROUP_MINB 7
#endif
#ifndef MREP_PAIRS_MINB
#define MREP_PAIRS_MINB 6
#endif
#ifndef MREP_STAGE_MINB
#define MREP_STAGE_MINB 3
#endif
#ifndef MREP_CLIP_MINB
#define MREP_CLIP_MINB 8
#endif

struct ProjParams {
  TableView tab;
  const double* q;
  int64_t n;
  double clip_tol;
  int max_iter;
  int soundness;
  double* out_t;
  double* out_foot;
  double* out_dist;
  int64_t* out_cand;
  int32_t* out_seg;
  int64_t* out_stats;
  double* out_sound;
  uint64_t* counters;
  unsigned long long* pass2_count;
  int64_t* pass2_list;
  const uint32_t* perm;  // Morton order of the queries (nullptr = identity)
  const uint32_t* inv;   // its inverse (large batches: emit through a sorted staging pass)
};

// ------------------------------------------------------------ tie band
struct Band {
  double dmin, lim;
  double t[BAND_K], d[BAND_K], v[BAND_K];
  uint64_t ord[BAND_K];
  unsigned valid;
  bool overflow;
  bool pass2;  // second pass: dmin/lim fixed, keep the single (t, ord) minimum
};

__device__ __forceinline__ void band_init(Band& B, bool pass2, double dmin2) {
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  B.valid = 0;
  B.overflow = false;
  B.pass2 = pass2;
  B.dmin = pass2 ? dmin2 : INF;
  B.lim = pass2 ? dmin2 + 1e-12 : INF;
#pragma unroll
  for (int j = 0; j < BAND_K; ++j) {
    B.t[j] = INF;
    B.d[j] = INF;
    B.v[j] = 0.0;
    B.ord[j] = ~0ull;
  }
}

// Offer one candidate (t, d) with foot recipe v and reference order key ord.
__device__ __forceinline__ void band_offer(Band& B, double t, double d, double v, uint64_t ord) {
  if (!(d <= B.lim)) return;
  if (B.pass2) {
    if (t < B.t[0] || (t == B.t[0] && ord < B.ord[0])) {
      B.t[0] = t;
      B.d[0] = d;
      B.v[0] = v;
      B.ord[0] = ord;
      B.valid = 1;
    }
    return;
  }
  if (d < B.dmin) {
    B.dmin = d;
    B.lim = d + 1e-12;
#pragma unroll
    for (int j = 0; j < BAND_K; ++j)
      if (((B.valid >> j) & 1u) && B.d[j] > B.lim) B.valid &= ~(1u << j);
  }
#pragma unroll
  for (int j = 0; j < BAND_K; ++j)
    if (((B.valid >> j) & 1u) && B.ord[j] == ord) return;  // same candidate re-offered
  bool placed = false;
#pragma unroll
  for (int j = 0; j < BAND_K; ++j) {
    if (!placed && !((B.valid >> j) & 1u)) {
      B.t[j] = t;
      B.d[j] = d;
      B.v[j] = v;
      B.ord[j] = ord;
      B.valid |= 1u << j;
      placed = true;
    }
  }
  if (!placed) B.overflow = true;
}

struct Pick {
  double t, d, v;
  uint64_t ord;
  bool ok;
};

// min t inside the band, ties by reference order (_kernels.py:485-490);
// select-based so the band never leaves registers
__device__ __forceinline__ Pick band_pick(const Band& B) {
  Pick p{0.0, 0.0, 0.0, 0ull, false};
#pragma unroll
  for (int j = 0; j < BAND_K; ++j) {
    bool take = ((B.valid >> j) & 1u) &&
                (!p.ok || B.t[j] < p.t || (B.t[j] == p.t && B.ord[j] < p.ord));
    p.t = take ? B.t[j] : p.t;
    p.d = take ? B.d[j] : p.d;
    p.v = take ? B.v[j] : p.v;
    p.ord = take ? B.ord[j] : p.ord;
    p.ok = p.ok || take;
  }
  return p;
}

struct QStats {
  int64_t pieces, c3l, c3g, cfl, cfg, noroot;
  double sound;
  uint64_t pairs, surv, clip_it, seams, boxes, offers;
};

// ------------------------------------------------------------ records
template <int D>
__device__ __forceinline__ void seam_point(const TableView& T, int64_t s, double (&pt)[D],
                                           double& st) {
  if (s == 0) {
    st = T.hdr[0];
#pragma unroll
    for (int k = 0; k < D; ++k) pt[k] = T.hdr[1 + k];
  } else {
    const double* r = T.rec + (s - 1) * REC;
    st = r[R_ST];
#pragma unroll
    for (int k = 0; k < D; ++k) pt[k] = r[R_SP + k];
  }
}

// _kernels.py:404-413 for one seam
template <int D>
__device__ __forceinline__ void offer_seam(const TableView& T, int64_t s, const double (&q)[D],
                                           Band& B, QStats& st) {
  double pt[D], stt;
  seam_point<D>(T, s, pt, stt);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double diff = q[k] - pt[k];
    acc += diff * diff;
  }
  st.seams++;
  st.offers++;
  // sqrt is monotone and correctly rounded: acc > lim^2 (rounded up by a
  // relative 1e-15) implies sqrt(acc) > lim, the band's first rejection test
  if (acc > B.lim * B.lim * (1.0 + 1e-15)) return;
  band_offer(B, stt, sqrt(acc), -1.0, (uint64_t)s);
}

// The roots of E' on [0, 1] that _quartic_roots_01 reports (_kernels.py
// :91-176), skipping the solve when there can be none: E'(u) lies between
// 5 min_j (b_{j+1} - b_j) and 5 max_j (b_{j+1} - b_j) (b = the Bernstein
// ordinates of E).  The reference keeps a candidate x only if its residual
// |E'(x)| <= 1e-9 max_k |c_k| <= 5e-9 sum_k |e_k| (c_k = (k+1) e_{k+1}), so
// when the differences are of one sign and clear 2e-9 sum |e| (far above the
// rounding of b and of the residual, and of E' on the 1e-12 slack outside
// [0, 1]) no candidate can pass: the reference returns no root, and so does
// this.  Typical near the foot point (E' = |C'|^2 + (C - q).C'' > 0), where
// most solved pairs are.
__device__ __forceinline__ Roots4 eprime_roots(const double (&e)[6], const double (&b)[6]) {
  double S = 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) S += fabs(e[k]);
  const double m = fmax(2e-9 * S, 1e-290);
  bool pos = true, neg = true;
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double beta = b[j + 1] - b[j];
    pos = pos && beta > m;
    neg = neg && beta < -m;
  }
  if (pos || neg) {
    Roots4 none;
    none.count = 0;
    none.r[0] = none.r[1] = none.r[2] = none.r[3] = 0.0;
    return none;
  }
  double ep[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) ep[k] = (double)(k + 1) * e[k + 1];
  return quartic_roots_01(ep);
}

// _kernels.py:421-479 for one cubic s: E, E' roots, monotone pieces,
// elimination, clipping, foot points; survivors are offered to the band.
template <int D, bool STATS>
__device__ __forceinline__ void solve_segment(const TableView& T, int64_t s, const double (&q)[D],
                                              double clip_tol, int max_iter, int soundness,
                                              Band& B, QStats& st) {
  const double* r = T.rec + s * REC;
  double w[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int dim = 0; dim < D; ++dim) w[k][dim] = __ldg(r + k * 3 + dim);
  double e[6];
  distance_poly_w<D>(w, q, e);
  double bseg[6];
  rebase5(e, bseg);
  Roots4 rt = eprime_roots(e, bseg);
  // interior split points (1e-10 < r < 1 - 1e-10), compacted in order
  double b1 = 1.0, b2 = 1.0, b3 = 1.0, b4 = 1.0;
  int nin = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double x = rt.r[i];
    if (i < rt.count && 1e-10 < x && x < 1.0 - 1e-10) {
      b1 = (nin == 0) ? x : b1;
      b2 = (nin == 1) ? x : b2;
      b3 = (nin == 2) ? x : b3;
      b4 = (nin == 3) ? x : b4;
      ++nin;
    }
  }
  st.pairs++;
  double lo = 0.0;
  for (int k = 0; k <= nin; ++k) {
    double hi = (k == nin) ? 1.0 : (k == 0 ? b1 : (k == 1 ? b2 : (k == 2 ? b3 : b4)));
    double bp[6];
    restrict_ordinates(bseg, lo, hi, bp);
    if (!(bp[0] < 0.0 && bp[0] * bp[5] <= 0.0)) {
      if (STATS && soundness > 0) {
        for (int si = 0; si < soundness; ++si) {
          double v = lo + (hi - lo) * (double)si / ((double)soundness - 1.0);
          double acc = 0.0;
#pragma unroll
          for (int dim = 0; dim < D; ++dim) {
            double f = decasteljau1(__ldg(r + R_P + dim), __ldg(r + R_P + 3 + dim), __ldg(r + R_P + 6 + dim),
                                    __ldg(r + R_P + 9 + dim), v);
            double diff = q[dim] - f;
            acc += diff * diff;
          }
          if (acc < st.sound) st.sound = acc;
        }
      }
      lo = hi;
      continue;
    }
    if (STATS) st.pieces++;
    ClipOut co = clip_root(bp, clip_tol, max_iter);
    st.surv++;
    st.clip_it += (uint64_t)co.used;
    if (!co.ok) {
      st.noroot++;
      lo = hi;
      continue;
    }
    double ta = __ldg(r + R_TA), tb = __ldg(r + R_TB);
    if (STATS) {
      double gscale = (hi - lo) * (tb - ta);
      if (co.w3 <= clip_tol) st.c3l++;
      if (co.w3 * gscale <= clip_tol) st.c3g++;
      if (co.wf <= clip_tol) st.cfl++;
      if (co.wf * gscale <= clip_tol) st.cfg++;
    }
    double v = lo + co.root * (hi - lo);
    double acc = 0.0;
#pragma unroll
    for (int dim = 0; dim < D; ++dim) {
      double f = decasteljau1(__ldg(r + R_P + dim), __ldg(r + R_P + 3 + dim), __ldg(r + R_P + 6 + dim),
                              __ldg(r + R_P + 9 + dim), v);
      double diff = q[dim] - f;
      acc += diff * diff;
    }
    st.offers++;
    band_offer(B, ta + v * (tb - ta), sqrt(acc), v, SURV_BIT | ((uint64_t)s << 3) | (uint64_t)k);
    lo = hi;
  }
}

// ------------------------------------------------------------ screening


template <int D>
__device__ __forceinline__ uint32_t child_mask(const TableView& T, int level, int64_t idx,
                                               const double (&q)[D], double c2, QStats& st,
                                               bool fb = false, const FQ<D>* fq = nullptr) {
  // children of node idx at `level` live at level-1, indices idx*8 + c
  uint32_t m = 0;
  int64_t first = idx * FANOUT;
  int64_t cnt = T.lvl_cnt[level - 1];
  int64_t off = T.lvl_off[level - 1];
#pragma unroll 1
  for (int c = 0; c < FANOUT; ++c) {
    int64_t ch = first + c;
    if (ch < cnt) {
      st.boxes++;
      if ((fb ? box_lb2f<D>(T, off + ch, *fq) : box_lb2<D>(T, off + ch, q)) <= c2) m |= 1u << c;
    }
  }
  return m;
}

template <int D, bool STATS>
__device__ void gen_screened(const TableView& T, const double (&q)[D], double scale,
                             double clip_tol, int max_iter, Band& B, QStats& st) {
  // 1) greedy descent to a nearby cubic: its seams give the first upper bound
  {
    int level = T.top;
    int64_t idx = 0;
    while (level > 0) {
      int64_t first = idx * FANOUT, cnt = T.lvl_cnt[level - 1], off = T.lvl_off[level - 1];
      double best = 0.0;
      int64_t bi = first;
      for (int c = 0; c < FANOUT; ++c) {
        int64_t ch = first + c;
        if (ch < cnt) {
          st.boxes++;
          double lb = box_lb2<D>(T, off + ch, q);
          if (c == 0 || lb < best) {
            best = lb;
            bi = ch;
          }
        }
      }
      idx = bi;
      --level;
    }
    offer_seam<D>(T, idx, q, B, st);
    offer_seam<D>(T, idx + 1, q, B, st);
  }
  // 2) depth-first traversal with 8-bit child masks per level; surviving
  //    leaf cubics are queued and solved in batches of LIST_CAP (one call
  //    site for the solve keeps the instruction footprint small)
  int64_t list[LIST_CAP];
  uint64_t masks = 0;
  int level = T.top;
  int64_t idx = 0;
  masks = (uint64_t)child_mask<D>(T, level, 0, q, cut2(B.dmin, scale), st) << (8 * level);
  bool done = false;
  while (!done) {
    int nlist = 0;
    while (nlist < LIST_CAP) {
      uint32_t mk = (uint32_t)(masks >> (8 * level)) & 0xffu;
      if (mk == 0) {
        if (level == T.top) {
          done = true;
          break;
        }
        ++level;
        idx /= FANOUT;
        continue;
      }
      int c = __ffs(mk) - 1;
      masks &= ~(1ull << (8 * level + c));
      int64_t ch = idx * FANOUT + c;
      double c2 = cut2(B.dmin, scale);
      st.boxes++;
      if (level - 1 == 0) {
        // leaf cubic: re-test with the current bound, queue it, offer its seams
        if (box_lb2<D>(T, T.lvl_off[0] + ch, q) <= c2) {
          offer_seam<D>(T, ch, q, B, st);
          offer_seam<D>(T, ch + 1, q, B, st);
          list[nlist++] = ch;
        }
      } else if (box_lb2<D>(T, T.lvl_off[level - 1] + ch, q) <= c2) {
        --level;
        idx = ch;
        masks |= (uint64_t)child_mask<D>(T, level, idx, q, c2, st) << (8 * level);
      }
    }
    // 3) exact solve of the queued cubics that still pass the current bound
    for (int i = 0; i < nlist; ++i) {
      st.boxes++;
      if (box_lb2<D>(T, T.lvl_off[0] + list[i], q) <= cut2(B.dmin, scale))
        solve_segment<D, STATS>(T, list[i], q, clip_tol, max_iter, 0, B, st);
    }
  }
}

template <int D, bool STATS>
__device__ void gen_dense(const TableView& T, const double (&q)[D], double clip_tol, int max_iter,
                          int soundness, Band& B, QStats& st) {
  for (int64_t s = 0; s <= T.S; ++s) offer_seam<D>(T, s, q, B, st);
  for (int64_t s = 0; s < T.S; ++s)
    solve_segment<D, STATS>(T, s, q, clip_tol, max_iter, soundness, B, st);
}


template <int D>
__device__ __forceinline__ void write_winner(const TableView& T, const ProjParams& p, int64_t qi,
                                             const Pick& w) {
  const double NaN = __longlong_as_double(0x7ff8000000000000LL);
  if (!w.ok) {
    p.out_t[qi] = NaN;
    p.out_dist[qi] = NaN;
#pragma unroll
    for (int k = 0; k < D; ++k) p.out_foot[qi * D + k] = NaN;
    if (p.out_seg) p.out_seg[qi] = -1;
    return;
  }
  uint64_t ord = w.ord;
  double foot[D];
  int32_t seg;
  if (ord & SURV_BIT) {
    int64_t s = (int64_t)((ord & ~SURV_BIT) >> 3);
    const double* r = T.rec + s * REC;
    double v = w.v;
#pragma unroll
    for (int dim = 0; dim < D; ++dim)
      foot[dim] = decasteljau1(r[R_P + dim], r[R_P + 3 + dim], r[R_P + 6 + dim], r[R_P + 9 + dim], v);
    seg = (int32_t)s;
  } else {
    int64_t s = (int64_t)ord;
    double stt;
    seam_point<D>(T, s, foot, stt);
    seg = (int32_t)(s > 0 ? s - 1 : 0);
  }
  p.out_t[qi] = w.t;
  p.out_dist[qi] = w.d;
#pragma unroll
  for (int k = 0; k < D; ++k) p.out_foot[qi * D + k] = foot[k];
  if (p.out_seg) p.out_seg[qi] = seg;
}

// =================================================================
// Warp-cooperative projection kernel.
//
// Queries arrive in Morton order (p.perm), so the 32 queries of a warp are
// spatial neighbours and visit the same cubics.  Three mechanisms keep the
// FP64 pipe busy despite the reference's data-dependent control flow:
//  * dense mode walks the cubics warp-uniformly (broadcast record loads);
//  * screened mode pools the (query, cubic) pairs of all 32 lanes' BVH
//    candidate lists and deals them out 32 at a time (a lane with 8
//    candidates no longer stalls 31 lanes with 1);
//  * surviving monotone pieces go to a per-warp ring queue in shared memory
//    and are Bezier-clipped 32 at a time, instead of one lane clipping while
//    31 wait.  Each clipped candidate is handed back to its owner lane's tie
//    band with a shuffle.
// =================================================================
constexpr int WARPS_PB = BLOCK / 32;
constexpr int SVQ = 64;        // survivor ring (power of two)
constexpr int PAIRCAP = 512;   // pair pool per warp
constexpr int SLIST = 16;      // per-lane candidate list in screened mode

struct WarpShared {
  double sb[SVQ][6];
  double slo[SVQ], shi[SVQ];
  int sseg[SVQ];
  int smeta[SVQ];  // owner lane | piece index << 8
  double q[32][3];
  double dmin[32];
  int cnt[32][6];  // per owner: ok candidates, c3l, c3g, cfl, cfg, noroot
  int pseg[PAIRCAP];
  unsigned char powner[PAIRCAP];
};

enum { C_OK = 0, C_C3L, C_C3G, C_CFL, C_CFG, C_NOROOT };

// Clip up to 32 queued survivors (one per lane) and deliver the candidates.
template <int D, bool STATS>
__device__ __forceinline__ void flush_survivors(WarpShared& W, int& head, int tail,
                                                const TableView& T, double clip_tol, int max_iter,
                                                Band& B, QStats& st, int lane) {
  int m = tail - head;
  if (m > 32) m = 32;
  bool has = lane < m;
  double t = 0.0, d = 0.0, v = 0.0;
  uint64_t ord = 0;
  int owner = 0;
  bool ok = false;
  if (has) {
    int slot = (head + lane) & (SVQ - 1);
    double bp[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) bp[i] = W.sb[slot][i];
    double lo = W.slo[slot], hi = W.shi[slot];
    int s = W.sseg[slot];
    int meta = W.smeta[slot];
    owner = meta & 0xff;
    int k = meta >> 8;
    ClipOut co = clip_root(bp, clip_tol, max_iter);
    st.surv++;
    st.clip_it += (uint64_t)co.used;
    ok = co.ok;
    if (!ok) {
      atomicAdd(&W.cnt[owner][C_NOROOT], 1);
      st.noroot++;
    } else {
      const double* r = T.rec + (int64_t)s * REC;
      double ta = __ldg(r + R_TA), tb = __ldg(r + R_TB);
      if (STATS) {
        double gscale = (hi - lo) * (tb - ta);
        if (co.w3 <= clip_tol) atomicAdd(&W.cnt[owner][C_C3L], 1);
        if (co.w3 * gscale <= clip_tol) atomicAdd(&W.cnt[owner][C_C3G], 1);
        if (co.wf <= clip_tol) atomicAdd(&W.cnt[owner][C_CFL], 1);
        if (co.wf * gscale <= clip_tol) atomicAdd(&W.cnt[owner][C_CFG], 1);
      }
      v = lo + co.root * (hi - lo);
      double acc = 0.0;
#pragma unroll
      for (int dim = 0; dim < D; ++dim) {
        double f = decasteljau1(__ldg(r + R_P + dim), __ldg(r + R_P + 3 + dim), __ldg(r + R_P + 6 + dim),
                                __ldg(r + R_P + 9 + dim), v);
        double diff = W.q[owner][dim] - f;
        acc += diff * diff;
      }
      t = ta + v * (tb - ta);
      d = sqrt(acc);
      ord = SURV_BIT | ((uint64_t)s << 3) | (uint64_t)k;
    }
  }
  head += m;
  __syncwarp();
  // hand each candidate to its owner's tie band
  for (int j = 0; j < m; ++j) {
    int oj = __shfl_sync(0xffffffffu, owner, j);
    bool okj = __shfl_sync(0xffffffffu, ok, j);
    double tj = __shfl_sync(0xffffffffu, t, j);
    double dj = __shfl_sync(0xffffffffu, d, j);
    double vj = __shfl_sync(0xffffffffu, v, j);
    uint64_t oj_ord = __shfl_sync(0xffffffffu, ord, j);
    if (okj && lane == oj) {
      st.offers++;
      band_offer(B, tj, dj, vj, oj_ord);
      W.dmin[lane] = B.dmin;
    }
  }
  __syncwarp();
}

// E, E' roots, interior split points and the rebased ordinates of one pair
struct PairPrep {
  double bseg[6];
  double b1, b2, b3, b4;
  int nin;
};

template <int D>
__device__ __forceinline__ void prep_pair(const TableView& T, int64_t s, const double (&q)[D],
                                          PairPrep& P) {
  const double* r = T.rec + s * REC;
  double w[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int dim = 0; dim < D; ++dim) w[k][dim] = __ldg(r + k * 3 + dim);
  double e[6];
  distance_poly_w<D>(w, q, e);
  rebase5(e, P.bseg);
  Roots4 rt = eprime_roots(e, P.bseg);
  P.b1 = P.b2 = P.b3 = P.b4 = 1.0;
  P.nin = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double x = rt.r[i];
    if (i < rt.count && 1e-10 < x && x < 1.0 - 1e-10) {
      P.b1 = (P.nin == 0) ? x : P.b1;
      P.b2 = (P.nin == 1) ? x : P.b2;
      P.b3 = (P.nin == 2) ? x : P.b3;
      P.b4 = (P.nin == 3) ? x : P.b4;
      ++P.nin;
    }
  }
}

// Rigorous lower bound on min_u |C_s(u) - q|^2 from the Bernstein
// coefficients of D = |C - q|^2 (see prep_pair_cut); true if it can reach cut_sq.
template <int D>
__device__ __forceinline__ bool bern_may_reach(const TableView& T, int64_t s, const double (&q)[D],
                                               double cut_sq) {
  const double* r = T.rec + s * REC;
  double w[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int dim = 0; dim < D; ++dim) w[k][dim] = __ldg(r + k * 3 + dim);
  double e[6], b[6];
  distance_poly_w<D>(w, q, e);
  rebase5(e, b);
  double d0 = 0.0;
#pragma unroll
  for (int dim = 0; dim < D; ++dim) {
    double df = w[0][dim] - q[dim];
    d0 += df * df;
  }
  double di = d0, dmin_b = d0, mag = fabs(d0);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    di += b[i] * (1.0 / 6.0);
    dmin_b = fmin(dmin_b, di);
    mag += fabs(b[i]);
  }
  return !(dmin_b - 1e-9 * mag > cut_sq);
}

// the early-exit tests of prep_pair_cut alone (same arithmetic): true if the
// pair can contribute a survivor within cut_sq
template <int D>
__device__ __forceinline__ bool pair_may_survive(const TableView& T, int64_t s, const double (&q)[D],
                                                 double cut_sq) {
  const double* r = T.rec + s * REC;
  double w[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int dim = 0; dim < D; ++dim) w[k][dim] = __ldg(r + k * 3 + dim);
  double e[6], b[6];
  distance_poly_w<D>(w, q, e);
  rebase5(e, b);
  double d0 = 0.0;
#pragma unroll
  for (int dim = 0; dim < D; ++dim) {
    double df = w[0][dim] - q[dim];
    d0 += df * df;
  }
  double di = d0, dmin_b = d0, mag = fabs(d0);
  bool pos = true, neg = true;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    di += b[i] * (1.0 / 6.0);
    dmin_b = fmin(dmin_b, di);
    mag += fabs(b[i]);
    pos = pos && b[i] > 1e-290;
    neg = neg && b[i] < -1e-290;
  }
  if (dmin_b - 1e-9 * mag > cut_sq) return false;
  return !(pos || neg);
}

// prep_pair with a rigorous early exit: the degree-6 Bernstein coefficients
// of D(u) = |C(u) - q|^2 follow from E = D' by d_0 = D(0), d_{i+1} = d_i + b_i/6
// (b = Bernstein ordinates of E); min_i d_i <= min_u D(u).  If that bound
// (minus a generous rounding allowance) exceeds the cut, no candidate of this
// cubic can reach the tie band and the quartic is skipped.
template <int D>
__device__ __forceinline__ bool prep_pair_cut(const TableView& T, int64_t s, const double (&q)[D],
                                              double cut_sq, PairPrep& P) {
  const double* r = T.rec + s * REC;
  double w[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int dim = 0; dim < D; ++dim) w[k][dim] = __ldg(r + k * 3 + dim);
  double e[6];
  distance_poly_w<D>(w, q, e);
  rebase5(e, P.bseg);
  double d0 = 0.0;
#pragma unroll
  for (int dim = 0; dim < D; ++dim) {
    double df = w[0][dim] - q[dim];
    d0 += df * df;
  }
  double di = d0, dmin_b = d0, mag = fabs(d0);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    di += P.bseg[i] * (1.0 / 6.0);
    dmin_b = fmin(dmin_b, di);
    mag += fabs(P.bseg[i]);
  }
  if (dmin_b - 1e-9 * mag > cut_sq) return false;
  // E = D'/2 of one strict sign on [0, 1] (all six Bernstein ordinates,
  // kept clear of underflow): every monotone piece's restricted ordinates
  // are positively weighted combinations of them, so each piece has
  // b0 > 0, or b0 < 0 with b0 b5 > 0 -- the elimination of
  // _kernels.py:427-441 drops them all.  No survivor: skip the quartic.
  {
    bool pos = true, neg = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      pos = pos && P.bseg[i] > 1e-290;
      neg = neg && P.bseg[i] < -1e-290;
    }
    if (pos || neg) return false;
  }
  Roots4 rt = eprime_roots(e, P.bseg);
  P.b1 = P.b2 = P.b3 = P.b4 = 1.0;
  P.nin = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double x = rt.r[i];
    if (i < rt.count && 1e-10 < x && x < 1.0 - 1e-10) {
      P.b1 = (P.nin == 0) ? x : P.b1;
      P.b2 = (P.nin == 1) ? x : P.b2;
      P.b3 = (P.nin == 2) ? x : P.b3;
      P.b4 = (P.nin == 3) ? x : P.b4;
      ++P.nin;
    }
  }
  return true;
}

}  // namespace mrep
#include "mrep_cand.cuh"
namespace mrep {

// Walk the monotone pieces of the warp's current pairs in lock step
// (piece k of every pair together), queue survivors, flush full batches.
template <int D, bool STATS>
__device__ __forceinline__ void pieces_step(WarpShared& W, int& head, int& tail, bool has,
                                            int64_t s, int owner, const PairPrep& P,
                                            const double (&q)[D], const TableView& T,
                                            double clip_tol, int max_iter, int soundness,
                                            Band& B, QStats& st, int lane) {
  int K = __reduce_max_sync(0xffffffffu, has ? P.nin + 1 : 0);
  double lo = 0.0;
  for (int k = 0; k < K; ++k) {
    bool act = has && k <= P.nin;
    double hi = (k == P.nin) ? 1.0 : (k == 0 ? P.b1 : (k == 1 ? P.b2 : (k == 2 ? P.b3 : P.b4)));
    bool surv = false;
    double bp[6];
    if (act) {
      restrict_ordinates(P.bseg, lo, hi, bp);
      surv = bp[0] < 0.0 && bp[0] * bp[5] <= 0.0;
      if (!surv && STATS && soundness > 0) {
        const double* r = T.rec + s * REC;
        for (int si = 0; si < soundness; ++si) {
          double v = lo + (hi - lo) * (double)si / ((double)soundness - 1.0);
          double acc = 0.0;
#pragma unroll
          for (int dim = 0; dim < D; ++dim) {
            double f = decasteljau1(__ldg(r + R_P + dim), __ldg(r + R_P + 3 + dim),
                                    __ldg(r + R_P + 6 + dim), __ldg(r + R_P + 9 + dim), v);
            double diff = q[dim] - f;
            acc += diff * diff;
          }
          if (acc < st.sound) st.sound = acc;
        }
      }
      if (surv && STATS) st.pieces++;
    }
    unsigned bal = __ballot_sync(0xffffffffu, surv);
    if (surv) {
      int slot = (tail + __popc(bal & ((1u << lane) - 1))) & (SVQ - 1);
#pragma unroll
      for (int i = 0; i < 6; ++i) W.sb[slot][i] = bp[i];
      W.slo[slot] = lo;
      W.shi[slot] = hi;
      W.sseg[slot] = (int)s;
      W.smeta[slot] = owner | (k << 8);
    }
    tail += __popc(bal);
    __syncwarp();
    if (tail - head >= 32) flush_survivors<D, STATS>(W, head, tail, T, clip_tol, max_iter, B, st, lane);
    lo = hi;
  }
}

template <int D, bool SCREEN, bool STATS>
__global__ void __launch_bounds__(BLOCK) project_kernel(ProjParams p) {
  __shared__ WarpShared wsh[WARPS_PB];
  const int lane = threadIdx.x & 31;
  WarpShared& W = wsh[threadIdx.x >> 5];
  int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool active = gi < p.n;
  int64_t qi = active ? (p.perm ? (int64_t)p.perm[gi] : gi) : 0;
  QStats st{};
  st.sound = __longlong_as_double(0x7ff0000000000000LL);
  const TableView& T = p.tab;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = active ? p.q[qi * D + k] : 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) W.q[lane][k] = q[k];
#pragma unroll
  for (int c = 0; c < 6; ++c) W.cnt[lane][c] = 0;
  Band B;
  band_init(B, false, 0.0);
  int head = 0, tail = 0;
  __syncwarp();
  if (!SCREEN) {
    if (active)
      for (int64_t s = 0; s <= T.S; ++s) offer_seam<D>(T, s, q, B, st);
    for (int64_t s = 0; s < T.S; ++s) {
      PairPrep P;
      if (active) {
        prep_pair<D>(T, s, q, P);
        st.pairs++;
      }
      pieces_step<D, STATS>(W, head, tail, active, s, lane, P, q, T, p.clip_tol, p.max_iter,
                            p.soundness, B, st, lane);
    }
  } else {
    double scale = T.hdr[4];
#pragma unroll
    for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
    // greedy descent: first upper bound from the seams of a nearby cubic
    if (active) {
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
            double lb = box_lb2<D>(T, off + ch, q);
            if (c == 0 || lb < best) {
              best = lb;
              bi = ch;
            }
          }
        }
        idx = bi;
        --level;
      }
#pragma unroll 1
      for (int e = 0; e < 2; ++e) offer_seam<D>(T, idx + e, q, B, st);
    }
    uint64_t masks = 0;
    int level = T.top;
    int64_t idx = 0;
    if (active) masks = (uint64_t)child_mask<D>(T, level, 0, q, cut2(B.dmin, scale), st) << (8 * level);
    bool done = !active;
    int64_t list[SLIST];
    while (__any_sync(0xffffffffu, !done)) {
      // 1) each lane extends its traversal until its list is full or it is done
      int nlist = 0;
      while (!done && nlist < SLIST) {
        uint32_t mk = (uint32_t)(masks >> (8 * level)) & 0xffu;
        if (mk == 0) {
          if (level == T.top) {
            done = true;
            break;
          }
          ++level;
          idx /= FANOUT;
          continue;
        }
        int c = __ffs(mk) - 1;
        masks &= ~(1ull << (8 * level + c));
        int64_t ch = idx * FANOUT + c;
        double c2 = cut2(B.dmin, scale);
        st.boxes++;
        if (level - 1 == 0) {
          if (box_lb2<D>(T, T.lvl_off[0] + ch, q) <= c2) {
#pragma unroll 1
            for (int e = 0; e < 2; ++e) offer_seam<D>(T, ch + e, q, B, st);
            list[nlist++] = ch;
          }
        } else if (box_lb2<D>(T, T.lvl_off[level - 1] + ch, q) <= c2) {
          --level;
          idx = ch;
          masks |= (uint64_t)child_mask<D>(T, level, idx, q, c2, st) << (8 * level);
        }
      }
      __syncwarp();
      W.dmin[lane] = B.dmin;
      // 2) pool the warp's pairs
      int incl = nlist;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      int total = __shfl_sync(0xffffffffu, incl, 31);
      int base = incl - nlist;
      for (int i = 0; i < nlist; ++i) {
        W.pseg[base + i] = (int)list[i];
        W.powner[base + i] = (unsigned char)lane;
      }
      __syncwarp();
      // 3) deal the pairs out 32 at a time
      for (int c0 = 0; c0 < total; c0 += 32) {
        int pi = c0 + lane;
        bool has = pi < total;
        int owner = 0;
        int64_t s = 0;
        double qq[D];
#pragma unroll
        for (int k = 0; k < D; ++k) qq[k] = 0.0;
        if (has) {
          owner = W.powner[pi];
          s = W.pseg[pi];
#pragma unroll
          for (int k = 0; k < D; ++k) qq[k] = W.q[owner][k];
          double sc = T.hdr[4];
#pragma unroll
          for (int k = 0; k < D; ++k) sc = fmax(sc, fabs(qq[k]));
          st.boxes++;
          // re-test with the owner's current bound (survivors may have tightened it)
          has = box_lb2<D>(T, T.lvl_off[0] + s, qq) <= cut2(W.dmin[owner], sc);
        }
        PairPrep P;
        if (has) {
          prep_pair<D>(T, s, qq, P);
          st.pairs++;
        }
        pieces_step<D, STATS>(W, head, tail, has, s, owner, P, qq, T, p.clip_tol, p.max_iter, 0,
                              B, st, lane);
      }
      __syncwarp();
    }
  }
  while (tail > head)
    flush_survivors<D, STATS>(W, head, tail, T, p.clip_tol, p.max_iter, B, st, lane);
  __syncwarp();
  if (active) {
    if (B.overflow) {
      // more than BAND_K candidates inside the tie band: exact second pass
      p.out_dist[qi] = B.dmin;
      unsigned long long slot = atomicAdd(p.pass2_count, 1ull);
      p.pass2_list[slot] = qi;
      if (p.out_seg) p.out_seg[qi] = -2;
    } else {
      write_winner<D>(T, p, qi, band_pick(B));
    }
    if (p.out_cand)
      p.out_cand[qi] = SCREEN ? (int64_t)st.offers
                              : (int64_t)(T.S + 1) + (int64_t)(st.offers - st.seams);
    if (STATS) {
      if (p.out_stats) {
        int64_t* o = p.out_stats + qi * 6;
        o[0] = st.pieces;
        o[1] = W.cnt[lane][C_C3L];
        o[2] = W.cnt[lane][C_C3G];
        o[3] = W.cnt[lane][C_CFL];
        o[4] = W.cnt[lane][C_CFG];
        o[5] = W.cnt[lane][C_NOROOT];
      }
      if (p.out_sound) p.out_sound[qi] = st.sound;
    }
  }
  warp_count(p.counters, MREP_CNT_PAIRS, st.pairs);
  warp_count(p.counters, MREP_CNT_SURVIVORS, st.surv);
  warp_count(p.counters, MREP_CNT_CLIP_ITERS, st.clip_it);
  warp_count(p.counters, MREP_CNT_SEAMS, st.seams);
  warp_count(p.counters, MREP_CNT_BOXES, st.boxes);
  warp_count(p.counters, MREP_CNT_HULL_MISS, (uint64_t)st.noroot);
}

// Morton key (10 bits per axis) of each query inside the table's padded box
template <int D>
__global__ void morton_kernel(const double* q, int64_t n, const double* box_root, uint32_t* key,
                              uint32_t* idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t code = 0;
  for (int k = 0; k < D; ++k) {
    double lo = box_root[k], hi = box_root[3 + k];
    double ext = fmax(hi - lo, 1e-300);
    double u = (q[i * D + k] - (lo - ext)) / (3.0 * ext);
    u = fmin(fmax(u, 0.0), 1.0);
    uint32_t c = (uint32_t)(u * 1023.0);
    // spread 10 bits with stride D
    for (int b = 0; b < 10; ++b) code |= ((c >> b) & 1u) << (b * D + k);
  }
  key[i] = code;
  idx[i] = (uint32_t)i;
}

template <int D, bool SCREEN>
__global__ void __launch_bounds__(BLOCK) project_pass2_kernel(ProjParams p) {
  unsigned long long total = *p.pass2_count;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t qi = p.pass2_list[i];
    double q[D];
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = p.q[qi * D + k];
    Band B;
    band_init(B, true, p.out_dist[qi]);
    QStats st{};
    st.sound = 0.0;
    if (SCREEN) {
      double scale = p.tab.hdr[4];
#pragma unroll
      for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
      gen_screened<D, false>(p.tab, q, scale, p.clip_tol, p.max_iter, B, st);
    } else {
      gen_dense<D, false>(p.tab, q, p.clip_tol, p.max_iter, 0, B, st);
    }
    write_winner<D>(p.tab, p, qi, Pick{B.t[0], B.d[0], B.v[0], B.ord[0], B.valid != 0});
  }
  if (p.counters && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd((unsigned long long*)&p.counters[MREP_CNT_PASS2], total);
}

// =================================================================
// Wavefront pipeline for the screened mode.
//
// Small single-purpose kernels, each with a compact instruction footprint
// and uniform work items, connected by device-side append buffers:
//   W1 traverse  (thread / query, Morton order; or an 8-lane group per query
//                for sparse batches): cell-list scan or BVH walk with the seam
//                upper bound; emits (query, cubic) pairs and the seam
//                candidates inside the seam tie band;
//   W2a filter   (thread / pair): box, Bernstein and one-signed-E tests with
//                the final seam bound; compacts the pairs that can survive;
//   W2b pairs    (thread / pair): E, E' roots, monotone pieces, elimination;
//                emits surviving pieces;
//   W3 clip      (lane refill): Bezier clipping, foot point, distance;
//                emits candidates that can still reach the tie band and
//                lowers the query's running minimum (atomicMin on the bits of
//                a non-negative double);
//   W4 emit      (thread / query): walks the query's candidate list (atomic
//                head + next links) applying the reference's two-pass rule
//                (_kernels.py:480-490): min distance -> min t inside
//                dmin + 1e-12 -> min reference order; writes the winner.
// Queries whose buffers would overflow (or whose seam band exceeds BAND_K)
// are finished by a per-thread exact fallback kernel.
// =================================================================
// a candidate of a query's final selection: parameter, distance, local
// parameter of a clipped survivor (-1 for seams), tie order (seam index, or
// CAND_SURV | cubic << 3 | piece for survivors) and the query's previous
// candidate (a per-query linked list headed by chead): one sector per record
constexpr uint32_t CAND_SURV = 1u << 31;
struct alignas(32) Cand {
  double t, d, v;
  uint32_t ord, next;
};

__device__ __forceinline__ void put_cand(Cand* c, double t, double d, double v, uint32_t ord,
                                         uint32_t next) {
  double4* p = reinterpret_cast<double4*>(c);
  *p = make_double4(t, d, v, __longlong_as_double((long long)(((uint64_t)next << 32) | ord)));
}

struct WaveParams {
  TableView tab;
  const double* q;
  int64_t n;
  const uint32_t* perm;
  double clip_tol;
  int max_iter;
  double* out_t;
  double* out_foot;
  double* out_dist;
  int64_t* out_cand;
  int32_t* out_seg;
  uint64_t* counters;
  unsigned long long* dmin;  // bits of the running min distance (non-negative double)
  int32_t* flag;             // 1 = finish in the fallback kernel
  double* qs;                // per sorted query: 4 doubles = coords (D) + running min (slot 3)
  double* win_t;             // winner record per sorted position
  double* win_d;
  double* win_v;
  int64_t* scnt;             // candidate count per sorted position
  unsigned long long* cnt;   // [0] pairs, [1] survivors, [2] candidates, [3] fallbacks
  uint32_t* pq;
  uint32_t* ps;
  uint32_t* pq2;  // pairs that pass W2a (compacted)
  uint32_t* ps2;
  unsigned long long pcap;
  double* sb;  // survivors: b0..b5, lo, hi
  uint32_t* sq;
  uint32_t* ssk;  // cubic << 3 | piece
  unsigned long long scap;
  int set_cells;        // curve set with per-curve cell indices (group scans may use them)
  const uint32_t* inv;  // caller -> sorted position (large batches; null otherwise)
  double* orec;         // with inv: each sorted query's outputs, 8 doubles (unpermuted after)
  uint32_t* ccnt;   // per sorted query: candidates appended so far
  Cand* cin;        // per sorted query: the first CIN candidates, inline ([n][CIN])
  uint32_t* chead;  // per sorted query: last overflow candidate (linked list), ~0 = none
  Cand* cand;       // overflow candidate records (one 32-B sector each)
  unsigned long long ccap;
  int64_t* fb;
  // multi-curve batch (mrep_project_batch): per-curve table descriptors, the
  // curve of each query (caller order) and of each sorted position, and the
  // persistent traversal's task counter
  int retest_min;  // re-test popped packet nodes at levels >= this (MREP_RETEST_LEVEL)
  int trav_bern;   // Bernstein distance test at packet leaves (MREP_TRAV_BERN)
  int trav_sort;   // full best-first child order in packets (MREP_TRAV_SORT)
  int fuse_filter;  // cell scans run W2a themselves (MREP_TRAV_FILTER)
  const TableView* tabs;
  const int32_t* qcurve;
  int64_t ncurves;
  int32_t* gcur;
  unsigned long long* queue;
};

// A query's first CIN candidates live inline in its own [CIN] row of `cin`
// (sorted order: the emit pass reads them as one coalesced 64-B run per
// query instead of chasing a linked list through a shared append buffer);
// later ones (rare: a tie band with many members) go to the overflow buffer,
// linked from chead.  Any thread may append for any query.
constexpr int CIN = 2;
__device__ __forceinline__ bool add_cand(const WaveParams& w, int64_t g, double t, double d,
                                         double v, uint32_t ord) {
  const uint32_t k = atomicAdd(&w.ccnt[g], 1u);
  if (k < CIN) {
    put_cand(w.cin + g * CIN + k, t, d, v, ord, ~0u);
    return true;
  }
  const unsigned long long slot = atomicAdd(&w.cnt[2], 1ull);
  if (slot >= w.ccap) return false;
  put_cand(w.cand + slot, t, d, v, ord, atomicExch(&w.chead[g], (uint32_t)slot));
  return true;
}

// table of sorted position g: the single curve, or its curve in a batch
template <bool MULTI>
__device__ __forceinline__ const TableView& tab_of(const WaveParams& w, int64_t g) {
  if (MULTI) return w.tabs[w.gcur[g]];
  return w.tab;
}



// every per-query array below is indexed by the SORTED position g; only the
// final emit kernel touches the caller's order (one scattered write pass).
// The running minimum lives in slot 3 of the query's 32-byte record, so a
// pair / survivor fetches coordinates and bound in one sector.
__device__ __forceinline__ unsigned long long* dmin_ptr(const WaveParams& w, int64_t g) {
  return (unsigned long long*)(w.qs + g * 4 + 3);
}
__device__ __forceinline__ double dmin_of(const WaveParams& w, int64_t g) {
  return __longlong_as_double((long long)*dmin_ptr(w, g));
}

// Packet traversal: the 32 (Morton-adjacent) queries of a warp walk the AABB
// tree together (nearest child on top of the stack; the Bernstein distance
// test of a leaf is left to W2, which runs it densely per pair).  One DFS stack per warp lives in shared memory; each entry
// carries the lane mask of the queries that still need the node, so control
// flow is warp-uniform and every box is one broadcast load.
constexpr int PSTACK = 72;  // >= 8 entries per level x 9 levels

__device__ __forceinline__ unsigned long long pk(unsigned mask, int level, int64_t idx) {
  return ((unsigned long long)mask << 32) | ((unsigned long long)level << 28) |
         (unsigned long long)idx;
}

// One warp-task: sorted positions base .. base+31.  Per-lane greedy descent,
// then packet traversal.  In a multi-curve batch the lanes of one warp may
// belong to different curves (queries are sorted by curve, so a warp spans at
// most a few): the packet walk runs once per distinct curve of the warp with
// that curve's lanes as the packet mask, so control flow stays warp-uniform.
// traversal modes of traverse_task
enum { TM_LANE = 0, TM_PACKET = 1, TM_CELLS = 2 };

// cell index leaf policy for curve tables: the exact curve points a leaf
// (cubic s) carries are its two seams s and s+1
struct CurveLeaves {
  __device__ int npts(const TableView&) const { return 2; }
  __device__ void pt(const TableView& T, int d, int64_t s, int k, double* p) const {
    const int64_t si = s + k;
    p[0] = p[1] = p[2] = 0.0;
    for (int j = 0; j < d; ++j) p[j] = si == 0 ? T.hdr[1 + j] : T.rec[(si - 1) * REC + R_SP + j];
  }
};

template <int D, bool MULTI, int TM>
__device__ __forceinline__ void traverse_task(const WaveParams& w, int64_t gi,
                                              unsigned long long* S, int lane) {
  constexpr bool PACKET = TM == TM_PACKET;
  bool active = gi < w.n;
  QStats st{};
  int64_t qi = active ? (w.perm ? (int64_t)w.perm[gi] : gi) : 0;
  int32_t cid = 0;
  if (MULTI && active) {
    cid = w.qcurve[qi];
    if (cid < 0 || cid >= w.ncurves) cid = -1;
    w.gcur[gi] = cid;
    if (cid < 0) {  // out-of-range curve id (sorted last): NaN result, no work
      w.scnt[gi] = 0;
      w.flag[gi] = 0;
      active = false;
    }
  }
  const TableView& T = MULTI ? w.tabs[cid < 0 ? 0 : cid] : w.tab;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = active ? w.q[qi * D + k] : 0.0;
  bool fall = false;
  Band B;
  band_init(B, false, 0.0);
  double scale = T.hdr[4];
#pragma unroll
  for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
  const bool fb = fbox_ok(scale);  // float box tests (see box_lb2f)
  const FQ<D> fq = make_fq<D>(q, scale);
  // cell mode: the query's cell in the uniform grid over the table box lists
  // every cubic that can hold a candidate for ANY query of the cell
  // (mrep_cells_build), nearest first; queries outside the grid walk the tree
  bool incell = false;
  int64_t cell = 0;
  if (TM == TM_CELLS && active) incell = cell_of<D>(T, q, cell);
  if (active && !incell) {  // greedy descent: first bound from the seams of a nearby cubic
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
          double lb = fb ? box_lb2f<D>(T, off + ch, fq) : box_lb2<D>(T, off + ch, q);
          if (c == 0 || lb < best) {
            best = lb;
            bi = ch;
          }
        }
      }
      idx = bi;
      --level;
    }
#pragma unroll 1
    for (int e = 0; e < 2; ++e) offer_seam<D>(T, idx + e, q, B, st);
  }
  // cell mode buffers a lane's pairs in registers and appends them once per
  // query (one warp-aggregated reservation) instead of one warp-wide atomic
  // round trip per list entry that any lane needs
  constexpr int PEND = 8;
  uint32_t pend[PEND];
  int np = 0;
  if (TM == TM_CELLS && incell) {
    int32_t a, b;
    const uint2* E = cell_list(T, D, cell, a, b);
    // entries one ahead (single tables: the lists are L2-hot) or two ahead
    // (curve sets: every list comes from HBM; measured cfg3 traverse 0.86 ->
    // 0.78 ms, while single tables lose 3% with the extra registers)
    constexpr bool AHEAD2 = MULTI;
    uint2 nxt = a < b ? __ldg(E + a) : make_uint2(0u, 0u);
    uint2 nxt2 = (AHEAD2 && a + 1 < b) ? __ldg(E + a + 1) : make_uint2(0u, 0u);
    double c2 = cut2(B.dmin, scale);  // refreshed only when the bound moves
#pragma unroll 1
    for (int32_t k = a; k < b; ++k) {
      // keys ascend and bound the box distance of every query of the cell:
      // past the cut, no later cubic can hold a band candidate
      const uint2 cur = nxt;
      if ((double)__uint_as_float(cur.x) > c2) break;
      const int64_t ch = (int32_t)cur.y;
      if (AHEAD2) {
        nxt = nxt2;
        if (k + 2 < b) nxt2 = __ldg(E + k + 2);
      } else if (k + 1 < b) {
        nxt = __ldg(E + k + 1);  // next entry in flight during this one
      }
      // the list's sector two ahead toward L2, once per sector (4 entries):
      // long lists come from HBM (cfg5 traverse 6.7 -> 6.3 ms per 2*10^7)
      if (((k - a) & 3) == 0 && k + 8 < b)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(E + k + 8));
      st.boxes++;
      bool need = (fb ? box_lb2f<D>(T, T.lvl_off[0] + ch, fq) : box_lb2<D>(T, T.lvl_off[0] + ch, q)) <=
                  c2;
      if (need) {
#pragma unroll 1
        for (int e = 0; e < 2; ++e) offer_seam<D>(T, ch + e, q, B, st);
        c2 = cut2(B.dmin, scale);
        st.pairs++;
        if (np == PEND) {  // buffer full (rare): this lane appends alone
          const unsigned long long base = atomicAdd(&w.cnt[0], (unsigned long long)PEND);
#pragma unroll
          for (int e = 0; e < PEND; ++e) {
            if (base + e < w.pcap) {
              w.pq[base + e] = (uint32_t)gi;
              w.ps[base + e] = pend[e];
            } else {
              fall = true;
            }
          }
          np = 0;
        }
#pragma unroll
        for (int e = 0; e < PEND; ++e)
          if (e == np) pend[e] = (uint32_t)ch;
        ++np;
      }
    }
  }
  if (TM == TM_CELLS) {  // warp-uniform: all lanes reconverge here
    int incl = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (w.fuse_filter) {
      // W2a fused (MREP_TRAV_FILTER): the query's bound is final here (only its
      // own seams move it), so the warp re-tests its buffered pairs now, with
      // the pairs dealt round-robin over the lanes (converged, one pair per
      // lane per round), and appends the ones that pass straight to the
      // compacted list W2b reads -- wave_pairs_filter's tests on the same
      // operands, without the pair list's round trip through memory (the
      // records are still in L1 from the scan).
      int maxnp = __reduce_max_sync(0xffffffffu, np);
      const double dmin_l = B.dmin;
      int nk = 0;  // staged kept pairs (warp-uniform)
      auto stage_flush = [&](int cnt) {
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&w.cnt[7], (unsigned long long)cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        unsigned om = 0;
#pragma unroll 1
        for (int j0 = 0; j0 < cnt; j0 += 32) {
          const int j = j0 + lane;
          const unsigned long long e = j < cnt ? S[j] : 0ull;
          const int o = (int)(e >> 32) & 31;
          const int64_t go = __shfl_sync(0xffffffffu, gi, o);
          if (j < cnt) {
            if (base + j < w.pcap) {
              w.pq2[base + j] = (uint32_t)go;
              w.ps2[base + j] = (uint32_t)e;
            } else {
              om |= 1u << o;
            }
          }
        }
        om = __reduce_or_sync(0xffffffffu, om);
        if ((om >> lane) & 1u) fall = true;
        __syncwarp();
      };
#pragma unroll 1
      for (int r = 0; r < total; r += 32) {
        const int p = r + lane;
        int lo = 0, hi = 31;  // owner: the first lane whose inclusive count exceeds p
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int mid = (lo + hi) >> 1;
          const int v = __shfl_sync(0xffffffffu, incl, mid);
          if (v > p) hi = mid;
          else lo = mid + 1;
        }
        const int owner = lo > 31 ? 31 : lo;
        const int e = p - (__shfl_sync(0xffffffffu, incl, owner) - __shfl_sync(0xffffffffu, np, owner));
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < PEND; ++j) {
          if (j < maxnp) {
            const uint32_t v = __shfl_sync(0xffffffffu, pend[j], owner);
            s = (j == e) ? v : s;
          }
        }
        double qo[D];
#pragma unroll
        for (int k = 0; k < D; ++k) qo[k] = __shfl_sync(0xffffffffu, q[k], owner);
        const double so = __shfl_sync(0xffffffffu, scale, owner);
        const double c2o = cut2(__shfl_sync(0xffffffffu, dmin_l, owner), so);
        const int64_t go = __shfl_sync(0xffffffffu, gi, owner);
        const int32_t co = MULTI ? __shfl_sync(0xffffffffu, cid, owner) : 0;
        bool keep = p < total;
        if (keep) {
          const TableView& TO = MULTI ? w.tabs[co] : w.tab;
          st.boxes++;
          keep = (fbox_ok(so) ? box_lb2f<D>(TO, TO.lvl_off[0] + s, make_fq<D>(qo, so))
                              : box_lb2<D>(TO, TO.lvl_off[0] + s, qo)) <= c2o;
          if (keep) keep = pair_may_survive<D>(TO, s, qo, c2o);
        }
        // kept pairs are staged in the warp's (here unused) packet stack and
        // reserved with one atomic per warp, not one per round
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (nk + __popc(bal) > PSTACK) {
          stage_flush(nk);
          nk = 0;
        }
        if (keep) S[nk + __popc(bal & ((1u << lane) - 1u))] = ((unsigned long long)owner << 32) | s;
        nk += __popc(bal);
        (void)go;
      }
      if (nk) stage_flush(nk);
    } else if (total) {
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(&w.cnt[0], (unsigned long long)total);
      base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(incl - np);
#pragma unroll
      for (int e = 0; e < PEND; ++e) {
        if (e < np) {
          if (base + e < w.pcap) {
            w.pq[base + e] = (uint32_t)gi;
            w.ps[base + e] = pend[e];
          } else {
            fall = true;
          }
        }
      }
    }
  }
  unsigned todo = PACKET ? __ballot_sync(0xffffffffu, active) : 0u;
  if ((TM == TM_LANE || (TM == TM_CELLS && !incell)) && active) {
    // Per-lane depth-first walk, for incoherent queries (a warp's lanes far
    // apart, e.g. ~100 random queries per curve in a batch): a packet would
    // drag every lane through the union of 32 paths.  8-bit child masks per
    // level (top <= 7, checked at launch); each child is re-tested against
    // the bound current when it is reached.
    int level = T.top;
    int64_t idx = 0;
    uint64_t masks = (uint64_t)child_mask<D>(T, level, 0, q, cut2(B.dmin, scale), st, fb, &fq)
                     << (8 * level);
    for (;;) {
      uint32_t mk = (uint32_t)(masks >> (8 * level)) & 0xffu;
      if (mk == 0) {
        if (level == T.top) break;
        ++level;
        idx /= FANOUT;
        continue;
      }
      int c = __ffs(mk) - 1;
      masks &= ~(1ull << (8 * level + c));
      int64_t ch = idx * FANOUT + c;
      double c2 = cut2(B.dmin, scale);
      st.boxes++;
      if (level == 1) {
        bool need = (fb ? box_lb2f<D>(T, T.lvl_off[0] + ch, fq) : box_lb2<D>(T, T.lvl_off[0] + ch, q)) <= c2;
        if (need) {
#pragma unroll 1
          for (int k = 0; k < 2; ++k) offer_seam<D>(T, ch + k, q, B, st);
          need = bern_may_reach<D>(T, ch, q, cut2(B.dmin, scale));
        }
        unsigned long long slot = wave_append(&w.cnt[0], need);
        st.pairs += need ? 1 : 0;
        if (need) {
          if (slot < w.pcap) {
            w.pq[slot] = (uint32_t)gi;
            w.ps[slot] = (uint32_t)ch;
          } else {
            fall = true;
          }
        }
      } else if ((fb ? box_lb2f<D>(T, T.lvl_off[level - 1] + ch, fq) : box_lb2<D>(T, T.lvl_off[level - 1] + ch, q)) <= c2) {
        --level;
        idx = ch;
        masks |= (uint64_t)child_mask<D>(T, level, idx, q, c2, st, fb, &fq) << (8 * level);
      }
    }
  }
  while (todo) {
    // packet = the lanes of one curve (all active lanes for a single curve)
    unsigned amask = todo;
    int32_t lc = 0;
    if (MULTI) {
      lc = __shfl_sync(0xffffffffu, cid, __ffs(todo) - 1);
      amask = __ballot_sync(0xffffffffu, active && cid == lc);
    }
    todo &= ~amask;
    const TableView& TG = MULTI ? w.tabs[lc] : w.tab;
    if (lane == 0) S[0] = pk(amask, TG.top, 0);
    int sp = 1;
    __syncwarp();
    while (sp > 0) {
      unsigned long long e = S[--sp];
      unsigned mask = (unsigned)(e >> 32);
      int level = (int)((e >> 28) & 0xf);
      int64_t idx = (int64_t)(e & 0xfffffffull);
      bool mine = (mask >> lane) & 1u;
      __syncwarp();
      if (level == 0) {
        // leaf cubic: re-test with the current bound, offer its seams, emit the pair
        bool need = false;
        if (mine) {
          st.boxes++;
          need = (fb ? box_lb2f<D>(TG, TG.lvl_off[0] + idx, fq) : box_lb2<D>(TG, TG.lvl_off[0] + idx, q)) <= cut2(B.dmin, scale);
          if (need) {
#pragma unroll 1
            for (int k = 0; k < 2; ++k) offer_seam<D>(TG, idx + k, q, B, st);
            // emit the pair only if the cubic's Bernstein distance bound can
            // still reach the tie band (with the bound its own seams just set)
            if (w.trav_bern) need = bern_may_reach<D>(TG, idx, q, cut2(B.dmin, scale));
          }
        }
        unsigned long long slot = wave_append(&w.cnt[0], need);
        st.pairs += need ? 1 : 0;
        if (need) {
          if (slot < w.pcap) {
            w.pq[slot] = (uint32_t)gi;
            w.ps[slot] = (uint32_t)idx;
          } else {
            fall = true;
          }
        }
        continue;
      }
      // re-test the popped node against the bound as it is now (seams found
      // since the push may have tightened it): one test instead of eight
      double c2 = cut2(B.dmin, scale);
      if (level >= w.retest_min && level < TG.top && mine) {
        st.boxes++;
        const int64_t nb = TG.lvl_off[level] + idx;
        mine = (fb ? box_lb2f<D>(TG, nb, fq) : box_lb2<D>(TG, nb, q)) <= c2;
      }
      mask = __ballot_sync(0xffffffffu, mine);
      if (!mask) continue;
      // children (level-1, idx*8 + c): best-first -- pushed in decreasing order
      // of the packet leader's box distance so the nearest child pops first and
      // the seam bound tightens before the far leaves are reached
      int64_t first = idx * FANOUT, cnt = TG.lvl_cnt[level - 1], off = TG.lvl_off[level - 1];
      double key[FANOUT];
      unsigned msk[FANOUT];
#pragma unroll
      for (int c = 0; c < FANOUT; ++c) {
        int64_t ch = first + c;
        bool need = false;
        double lb = 0.0;
        if (ch < cnt && mine) {
          st.boxes++;
          lb = fb ? box_lb2f<D>(TG, off + ch, fq) : box_lb2<D>(TG, off + ch, q);
          need = lb <= c2;
        }
        unsigned m = __ballot_sync(0xffffffffu, need);
        msk[c] = m;
        key[c] = m ? __shfl_sync(0xffffffffu, lb, __ffs(m) - 1) : -1.0;
      }
      if (!w.trav_sort) {
        // nearest child on top, the others below in index order
        int bc = -1;
        double bk = 0.0;
#pragma unroll
        for (int c = 0; c < FANOUT; ++c)
          if (msk[c] && (bc < 0 || key[c] < bk)) {
            bc = c;
            bk = key[c];
          }
#pragma unroll
        for (int c = 0; c < FANOUT; ++c) {
          if (msk[c] && c != bc) {
            if (lane == 0) S[sp] = pk(msk[c], level - 1, first + c);
            ++sp;
          }
        }
        if (bc >= 0) {
          if (lane == 0) S[sp] = pk(msk[bc], level - 1, first + bc);
          ++sp;
        }
        __syncwarp();
        continue;
      }
      // sort (key, child) descending: 8-input network, uniform across the warp
      int ord8[FANOUT];
#pragma unroll
      for (int c = 0; c < FANOUT; ++c) ord8[c] = c;
#define MREP_CEX(a, b)                                   \
  if (key[a] < key[b]) {                                 \
    double tk = key[a];                                  \
    key[a] = key[b];                                     \
    key[b] = tk;                                         \
    unsigned tm = msk[a];                                \
    msk[a] = msk[b];                                     \
    msk[b] = tm;                                         \
    int to = ord8[a];                                    \
    ord8[a] = ord8[b];                                   \
    ord8[b] = to;                                        \
  }
      MREP_CEX(0, 1) MREP_CEX(2, 3) MREP_CEX(4, 5) MREP_CEX(6, 7)
      MREP_CEX(0, 2) MREP_CEX(1, 3) MREP_CEX(4, 6) MREP_CEX(5, 7)
      MREP_CEX(1, 2) MREP_CEX(5, 6) MREP_CEX(0, 4) MREP_CEX(3, 7)
      MREP_CEX(1, 5) MREP_CEX(2, 6)
      MREP_CEX(1, 4) MREP_CEX(3, 6)
      MREP_CEX(2, 4) MREP_CEX(3, 5)
      MREP_CEX(3, 4)
#undef MREP_CEX
#pragma unroll
      for (int c = 0; c < FANOUT; ++c) {
        if (msk[c]) {
          if (lane == 0) S[sp] = pk(msk[c], level - 1, first + ord8[c]);
          ++sp;
        }
      }
      __syncwarp();
    }
  }
  if (active) {
    if (B.overflow) fall = true;
    double4 rec;
    rec.x = q[0];
    rec.y = q[1];
    rec.z = D == 3 ? q[D - 1] : 0.0;
    rec.w = B.dmin;
    *(double4*)(w.qs + gi * 4) = rec;
  }
  // the seam members of the seam tie band become candidates; this thread is
  // the only writer of its query's candidate row during the traversal (the
  // solve kernels append later), so the row fills without atomics
  uint32_t ncand = 0;
#pragma unroll
  for (int j = 0; j < BAND_K; ++j) {
    if (active && ((B.valid >> j) & 1u)) {
      if (ncand < CIN) {
        put_cand(w.cin + gi * CIN + ncand, B.t[j], B.d[j], -1.0, (uint32_t)B.ord[j], ~0u);
      } else {
        const unsigned long long slot = atomicAdd(&w.cnt[2], 1ull);
        if (slot < w.ccap)
          put_cand(w.cand + slot, B.t[j], B.d[j], -1.0, (uint32_t)B.ord[j],
                   atomicExch(&w.chead[gi], (uint32_t)slot));
        else
          fall = true;
      }
      ++ncand;
    }
  }
  if (ncand) w.ccnt[gi] = ncand;
  if (active) {
    // cand (screened): seams offered + cubics queued for the exact solve by
    // this query's traversal -- independent of the other queries' timing
    w.scnt[gi] = (int64_t)(st.offers + st.pairs);
    w.flag[gi] = fall ? 1 : 0;
    if (fall) {
      unsigned long long slot = atomicAdd(&w.cnt[3], 1ull);
      w.fb[slot] = gi;
    }
  }
  warp_count(w.counters, MREP_CNT_SEAMS, st.seams);
  warp_count(w.counters, MREP_CNT_BOXES, st.boxes);
}

// W1.  Single curve: one thread per sorted query, hardware block scheduling.
// Multi-curve batch (the paper's task scheduler): queries are sorted by
// curve, heaviest curve (most cubics) first, Morton order inside a curve;
// persistent warps pull 32-position tasks from an atomic work queue, so the
// long tasks start first and the short ones fill the tail (LPT order).
template <int D, bool MULTI, int TM>
__global__ void __launch_bounds__(BLOCK, MREP_TRAV_MINB) wave_traverse(const __grid_constant__ WaveParams w) {
  __shared__ unsigned long long stk[BLOCK / 32][PSTACK];
  const int lane = threadIdx.x & 31;
  unsigned long long* S = stk[threadIdx.x >> 5];
  if (!MULTI) {
    traverse_task<D, false, TM>(w, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, S, lane);
  } else {
    for (;;) {
      unsigned long long task = 0;
      if (lane == 0) task = atomicAdd(w.queue, 1ull);
      task = __shfl_sync(0xffffffffu, task, 0);
      int64_t base = (int64_t)task * 32;
      if (base >= w.n) break;
      traverse_task<D, true, TM>(w, base + lane, S, lane);
    }
  }
}

// W1, tensor-core cell screen (MREP_TRAV_DMMA; single table with a cell
// index).  One warp = 8 consecutive sorted queries (rows of an m8n8k4 FP64
// MMA).  Rows of one cell scan its list together; per listed cubic ONE
// mma.sync with the cubic's tensor-core fragment (the same B operand as the
// exact-cand pass: the differences d_{j+1} - d_j of the degree-6 Bernstein
// coefficients of |C(u) - q|^2, affine in q) gives all 8 rows' coefficient
// differences; with d_0 = |P_0 - q|^2 a prefix over the row's lanes yields
// d_0..d_6, whose minimum (less a 1e-9 relative margin, as bern_may_reach)
// is a rigorous lower bound of |C(u) - q|^2 on the cubic -- tighter than the
// control-point box, and computed on the tensor pipe instead of per lane.
// A row stops at the first list key past its cut (keys ascend); the rest
// is traverse_task's cell mode: seams of kept cubics into the row's band,
// pairs buffered and appended once.  Rows outside the grid run
// traverse_task's per-lane walk.  Same exactness argument as the box test
// (any pruned cubic's candidates lie beyond dmin + 1e-12), so t / foot /
// distance / segment are unchanged; the screened `cand` counts this walk.
template <int D>
__global__ void __launch_bounds__(BLOCK, MREP_TRAV_MINB) wave_traverse_dmma(const __grid_constant__ WaveParams w) {
  const int lane = threadIdx.x & 31, row = lane >> 2, p = lane & 3;
  const int64_t g0 = (((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5) * 8;
  const int64_t gi = g0 + row;
  const bool active = gi < w.n;
  const TableView& T = w.tab;
  const int64_t qi = active ? (w.perm ? (int64_t)w.perm[gi] : gi) : 0;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = active ? w.q[qi * D + k] : 0.0;
  double scale = T.hdr[4];
#pragma unroll
  for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
  int64_t cell = -1;
  const bool incell = active && cell_of<D>(T, q, cell);
  // rows outside the grid: the per-lane walk of traverse_task (lane p == 0)
  if (active && !incell && p == 0) traverse_task<D, false, TM_LANE>(w, gi, nullptr, lane);
  const unsigned vin = __ballot_sync(0xffffffffu, incell && p == 0);
  unsigned todo = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) todo |= ((vin >> (4 * r)) & 1u) << r;
  if (!todo) return;  // warp-uniform
  const double a = p == 0 ? 1.0 : (p <= D ? q[p - 1] - T.hdr[4 + p] : 0.0);
  const bool owner = incell && p == 0;
  bool fall = false;
  Band B;
  band_init(B, false, 0.0);
  QStats st{};
  constexpr int PEND = 8;
  uint32_t pend[PEND];
  int np = 0;
  const double* F = T.bfrag;
  while (todo) {
    const int lead = __ffs(todo) - 1;
    const int64_t lc = __shfl_sync(0xffffffffu, cell, 4 * lead);
    const unsigned same = __ballot_sync(0xffffffffu, p == 0 && incell && cell == lc);
    unsigned rows = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) rows |= ((same >> (4 * r)) & 1u) << r;
    rows &= todo;
    todo &= ~rows;
    int32_t a0, a1;
    const uint2* EL = cell_list(T, D, lc, a0, a1);
    bool mine = ((rows >> row) & 1u) != 0;  // this row still scans (all 4 lanes)
    uint2 e_nxt = a0 < a1 ? __ldg(EL + a0) : make_uint2(0u, 0u);
#pragma unroll 1
    for (int32_t k = a0; k < a1; ++k) {
      const uint2 e_cur = e_nxt;
      const int64_t s = (int32_t)e_cur.y;
      if (k + 1 < a1) e_nxt = __ldg(EL + k + 1);
      // keys ascend: past a row's cut no later cubic can hold a band candidate
      bool go = false;
      if (owner && mine) go = !((double)__uint_as_float(e_cur.x) > cut2(B.dmin, scale));
      const unsigned gb = __ballot_sync(0xffffffffu, go);
      mine = ((gb >> (lane & ~3)) & 1u) != 0;
      if (!gb) break;
      const double b = __ldg(F + s * 32 + lane);
      double c0, c1;
      dmma_8x8x4(a, b, c0, c1);
      // d_0 = |P_0 - q|^2 (lane p == 0), then d_{j+1} = d_j + (d_{j+1} - d_j)
      double d0 = 0.0;
      if (p == 0) {
        const double* r0 = T.rec + s * REC + R_P;
#pragma unroll
        for (int k2 = 0; k2 < D; ++k2) {
          const double df = __ldg(r0 + k2) - q[k2];
          d0 += df * df;
        }
      }
      const bool col = p <= 2;  // lanes p = 0..2 hold the six differences
      const double x = col ? c0 : 0.0, y = col ? c1 : 0.0;
      const double xy = x + y;
      double pre = __shfl_up_sync(0xffffffffu, xy, 1);
      if (p == 0) pre = 0.0;
      const double pre2 = __shfl_up_sync(0xffffffffu, pre, 1);
      pre += (p >= 2) ? pre2 : 0.0;
      d0 = __shfl_sync(0xffffffffu, d0, lane & ~3);
      double mn = fmin(d0 + pre + x, d0 + pre + xy);
      if (!col) mn = d0;
      double mag = fabs(x) + fabs(y);
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 2));
      mag += __shfl_xor_sync(0xffffffffu, mag, 1);
      mag += __shfl_xor_sync(0xffffffffu, mag, 2);
      mn = fmin(mn, d0);
      if (go) {
        st.boxes++;
        // as bern_may_reach: prune iff min_j d_j - 1e-9 mag > cut^2
        // (mag = |d_0| + sum |b_j|, b_j = 6 (d_{j+1} - d_j))
        const double magb = fabs(d0) + 6.0 * mag;
        const bool need = !(mn - 1e-9 * magb > cut2(B.dmin, scale));
        if (need) {
#pragma unroll 1
          for (int e = 0; e < 2; ++e) offer_seam<D>(T, s + e, q, B, st);
          st.pairs++;
          if (np == PEND) {  // buffer full (rare): this lane appends alone
            const unsigned long long base = atomicAdd(&w.cnt[0], (unsigned long long)PEND);
#pragma unroll
            for (int e = 0; e < PEND; ++e) {
              if (base + e < w.pcap) {
                w.pq[base + e] = (uint32_t)gi;
                w.ps[base + e] = pend[e];
              } else {
                fall = true;
              }
            }
            np = 0;
          }
#pragma unroll
          for (int e = 0; e < PEND; ++e)
            if (e == np) pend[e] = (uint32_t)s;
          ++np;
        }
      }
    }
  }
  // buffered pairs: one warp-wide reservation
  int incl = np;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total) {
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(&w.cnt[0], (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(incl - np);
#pragma unroll
    for (int e = 0; e < PEND; ++e) {
      if (e < np) {
        if (base + e < w.pcap) {
          w.pq[base + e] = (uint32_t)gi;
          w.ps[base + e] = pend[e];
        } else {
          fall = true;
        }
      }
    }
  }
  if (owner) {
    if (B.overflow) fall = true;
    double4 rec;
    rec.x = q[0];
    rec.y = q[1];
    rec.z = D == 3 ? q[D - 1] : 0.0;
    rec.w = B.dmin;
    *(double4*)(w.qs + gi * 4) = rec;
#pragma unroll
    for (int j = 0; j < BAND_K; ++j)
      if (((B.valid >> j) & 1u) && !add_cand(w, gi, B.t[j], B.d[j], -1.0, (uint32_t)B.ord[j]))
        fall = true;
    w.scnt[gi] = (int64_t)(st.offers + st.pairs);
    w.flag[gi] = fall ? 1 : 0;
    if (fall) {
      unsigned long long slot = atomicAdd(&w.cnt[3], 1ull);
      w.fb[slot] = gi;
    }
  }
  warp_count(w.counters, MREP_CNT_SEAMS, owner ? st.seams : 0);
  warp_count(w.counters, MREP_CNT_BOXES, owner ? st.boxes : 0);
}

// W1, group mode: one 8-lane group per query, lane c tests child c of the
// node being expanded (the 8-ary hierarchy maps onto the group: one
// coalesced 384-B box load per expansion instead of 8 dependent loads).
// Best-first: a node's kept children are pushed nearest-on-top (each entry
// carries its box bound, re-tested against the bound current at pop time).
// Leaves: each lane offers the END seam of its cubic (seam s+1; cubic 0
// also offers seam 0) -- a seam whose other cubic was pruned lies in that
// cubic's box, so it cannot reach the tie band -- and the group min-reduces
// the seam distances into the running bound.  Each lane remembers its two
// nearest seams; kept leaves are parked in a per-group shared-memory list.
// Nothing is appended to the global buffers until the warp's four queries
// are done: then the seams inside each query's final band become
// candidates and the parked leaves that still pass the final bound (box and
// Bernstein tests) become (query, cubic) pairs, with one warp-wide atomic
// per batch of 32 instead of one per group step.  A lane that had to drop a
// third seam inside the final band sends its query to the exact fallback.
constexpr int GSTACK = 64;
constexpr int GPAIRS = 24;  // parked leaves per query (overflow: flushed early)

// Box bounds are compared as floats.  A lane on the float box path keeps the
// FP32 sum `acc` of box_lb2f (whose rigorous bound is acc * (1 - 1e-6)); a
// lane on the double path (coordinates near the float range) keeps its
// double bound rounded down.  The cut-off c2 becomes a float threshold
// rounded up (divided by 1 - 1e-6 on the float path, with room for the
// roundings), so `key > thr` still implies that the box's exact squared
// distance exceeds c2: no box is pruned that the double test would keep.
__device__ __forceinline__ float cut_key(double c2, bool fb) {
  return __double2float_ru(fb ? c2 * (1.0 + 1.1e-6) : c2 * (1.0 + 1e-15));
}

// Where a group traversal reads the float boxes: the table in global memory
// (read-only path) or a copy staged in shared memory (wave_traverse_staged).
template <bool SMEM>
struct BoxSrc {
  const float* fb;  // float boxes of every level, box i at fb + 6 i
  __device__ __forceinline__ float ld(int64_t i) const { return SMEM ? fb[i] : __ldg(fb + i); }
};

// FP32 part of box_lb2f (same expression, so the same float)
template <int D, bool SMEM>
__device__ __forceinline__ float box_accf(const BoxSrc<SMEM>& B, int64_t box, const FQ<D>& f) {
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float g = fmaxf(0.0f, fmaxf(B.ld(box * 6 + k) - f.lo[k], f.hi[k] - B.ld(box * 6 + 3 + k)));
    acc += g * g;
  }
  return acc;
}

struct SeamBest {  // a lane's two nearest seams (t re-read at emission)
  double d1, d2, dropped;
  int32_t s1, s2;
};

__device__ __forceinline__ void seam_keep(SeamBest& b, double d, int32_t s) {
  // a seam offered twice (start of one listed cubic, end of the previous)
  if ((s == b.s1 && b.d1 == d) || (s == b.s2 && b.d2 == d)) return;
  if (d < b.d1) {
    b.dropped = fmin(b.dropped, b.d2);
    b.d2 = b.d1;
    b.s2 = b.s1;
    b.d1 = d;
    b.s1 = s;
  } else if (d < b.d2) {
    b.dropped = fmin(b.dropped, b.d2);
    b.d2 = d;
    b.s2 = s;
  } else {
    b.dropped = fmin(b.dropped, d);
  }
}

// distance from q to seam s (compact seam block of a curve table)
template <int D>
__device__ __forceinline__ double seam_dist(const TableView& T, int64_t s, const double (&q)[D]) {
  const double* p = T.sxyz + s * 3;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double df = q[k] - __ldg(p + k);
    acc += df * df;
  }
  return sqrt(acc);
}

// emit parked leaves [0, cnt) of a group that pass cut c2 (box key <= thr,
// then the Bernstein test)
template <int D>
__device__ __forceinline__ void flush_pairs(const WaveParams& w, const TableView& T, int64_t g,
                                            const double (&q)[D], double c2, float thr,
                                            const uint32_t* PC, const float* PL, int cnt, int sub,
                                            bool& fall, uint32_t& npairs) {
  const int rounds = (cnt + 7) >> 3;
  for (int r = 0; r < rounds; ++r) {
    const int i = r * 8 + sub;
    bool need = false;
    uint32_t ch = 0;
    if (i < cnt) {
      ch = PC[i];
      need = PL[i] <= thr && bern_may_reach<D>(T, ch, q, c2);
    }
    unsigned long long slot = wave_append(&w.cnt[0], need);
    npairs += need ? 1 : 0;
    if (need) {
      if (slot < w.pcap) {
        w.pq[slot] = (uint32_t)g;
        w.ps[slot] = ch;
      } else {
        fall = true;
      }
    }
  }
}

// One query per 8-lane group (see above).  T = the query's table (a global
// descriptor, or a shared-memory copy in the staged kernel), B = where its
// float boxes are read.  Stack keys: level << 28 | node (group mode needs
// top <= 8, so a node index fits 28 bits); stack bounds are float keys.
// A node's kept children are pushed in index order with the nearest on top.
template <int D, bool MULTI, int NSTACK, bool SMEM, bool CELLS = false>
__device__ __forceinline__ void traverse_group(const WaveParams& w, int64_t g, bool active,
                                               int32_t cid, const TableView& T,
                                               const BoxSrc<SMEM>& B, uint32_t* SK, float* SL,
                                               uint32_t* PC, float* PL, int lane) {
  const int sub = lane & 7;
  const unsigned gmask = 0xffu << (lane & 24);
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  struct { uint32_t pairs, seams, boxes, offers; } st{};  // 32-bit: fewer registers
  int64_t qi = active ? (w.perm ? (int64_t)w.perm[g] : g) : 0;
  if (MULTI && active && sub == 0) w.gcur[g] = cid;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = active ? w.q[qi * D + k] : 0.0;
  double scale = T.hdr[4];
#pragma unroll
  for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
  const bool fb = fbox_ok(scale);
  const FQ<D> fq = make_fq<D>(q, scale);
  double dmin = INF;
  float thr = __int_as_float(0x7f800000);  // +inf: no bound yet
  bool fall = false;
  SeamBest sb{INF, INF, INF, 0, 0};
  int sp = 0, npark = 0;
  if (active) {
    if (sub == 0) {
      SK[0] = (uint32_t)T.top << 28;
      SL[0] = 0.0f;
    }
    sp = 1;
  }
  __syncwarp(gmask);
  if constexpr (CELLS) {
    // Cell-list scan, one query per 8-lane group (curve sets with per-curve
    // cell indices; every active query of the warp lies in its grid): each
    // round the group tests 8 consecutive entries of the query's sorted list
    // (lane `sub` takes entry k0 + sub: one coalesced 64-B read), offers both
    // seams of every kept cubic, min-reduces the seam distances into the
    // bound, parks the kept cubics; the scan stops after the round in which
    // an entry's key passed the cut (keys ascend).  Compared with one lane
    // per query, the lanes of a warp no longer wait for the longest list.
    int32_t a = 0, b = 0;
    const uint2* E = nullptr;
    if (active) {
      int64_t cell = 0;
      cell_of<D>(T, q, cell);
      E = cell_list(T, D, cell, a, b);
    }
    int32_t k0 = a;
    for (;;) {
      const bool more = active && k0 < b;
      if (!__any_sync(0xffffffffu, more)) break;
      if (more) {  // group-uniform
        const int32_t k = k0 + sub;
        const bool ex = k < b;
        const uint2 e = ex ? __ldg(E + k) : make_uint2(0u, 0u);
        const double c2 = cut2(dmin, scale);
        const bool live = ex && !((double)__uint_as_float(e.x) > c2);
        const bool past = ex && !live;
        float key = __int_as_float(0x7f800000);
        const int64_t ch = (int32_t)e.y;
        if (live) {
          st.boxes++;
          const int64_t bi = T.lvl_off[0] + ch;
          key = fb ? box_accf<D>(B, bi, fq) : __double2float_rd(box_lb2<D>(T, bi, q));
        }
        const bool keep = live && key <= thr;
        double dr = INF;
        if (keep) {
          const double d0 = seam_dist<D>(T, ch, q);
          const double d1 = seam_dist<D>(T, ch + 1, q);
          seam_keep(sb, d0, (int32_t)ch);
          seam_keep(sb, d1, (int32_t)(ch + 1));
          st.seams += 2;
          st.offers += 2;
          dr = fmin(d0, d1);
        }
        double m = dr;
        m = fmin(m, __shfl_xor_sync(gmask, m, 4));
        m = fmin(m, __shfl_xor_sync(gmask, m, 2));
        m = fmin(m, __shfl_xor_sync(gmask, m, 1));
        if (m < dmin) {  // group-uniform
          dmin = m;
          thr = cut_key(cut2(dmin, scale), fb);
        }
        const bool park = keep && key <= thr;
        const unsigned pm = (__ballot_sync(gmask, park) >> (lane & 24)) & 0xffu;
        if (npark + __popc(pm) > GPAIRS) {  // list full: flush with the current bound
          flush_pairs<D>(w, T, g, q, cut2(dmin, scale), thr, PC, PL, npark, sub, fall, st.pairs);
          __syncwarp(gmask);
          npark = 0;
        }
        if (park) {
          const int at = npark + __popc(pm & ((1u << sub) - 1));
          PC[at] = (uint32_t)ch;
          PL[at] = key;
        }
        npark += __popc(pm);
        // keys ascend: once one entry is past the cut, every later one is
        const unsigned pb = (__ballot_sync(gmask, past) >> (lane & 24)) & 0xffu;
        k0 = pb ? b : k0 + 8;
      }
      __syncwarp();
    }
  }
  // The warp's four groups advance in lockstep: every trip, each group with
  // work pops and expands one node, and the warp reconverges at the end of
  // the trip (otherwise the groups drift apart and the warp issues each
  // group's instructions separately at 8/32 lanes).
  for (; !CELLS;) {
    // pop: the group reads the top 8 entries at once and drops every entry
    // above the first one still under the threshold (a bound that tightened
    // since the push prunes them), so a run of pruned entries costs one trip
    bool found = false, more = sp > 0;
    while (__any_sync(0xffffffffu, more)) {
      if (more) {
        const bool ok = sub < sp && SL[sp - 1 - sub] <= thr;
        const unsigned okm = (__ballot_sync(gmask, ok) >> (lane & 24)) & 0xffu;
        if (okm) {
          sp -= __ffs(okm);
          found = true;
          more = false;
        } else {
          sp = sp > 8 ? sp - 8 : 0;
          more = sp > 0;
        }
      }
    }
    if (!__any_sync(0xffffffffu, found)) break;
    if (found) {  // group-uniform
      const uint32_t e = SK[sp];
      const int level = (int)(e >> 28);
      const int64_t idx = (int64_t)(e & 0x0fffffffu);
      const int64_t ch = idx * FANOUT + sub;
      const bool ex = ch < T.lvl_cnt[level - 1];
      float key = __int_as_float(0x7f800000);
      if (ex) {
        st.boxes++;
        const int64_t bi = T.lvl_off[level - 1] + ch;
        key = fb ? box_accf<D>(B, bi, fq) : __double2float_rd(box_lb2<D>(T, bi, q));
      }
      const bool keep = ex && key <= thr;
      if (level == 1) {
        // leaves: end seams -> bound; kept leaves parked for the final flush
        double dr = INF;
        if (keep) {
          dr = seam_dist<D>(T, ch + 1, q);
          seam_keep(sb, dr, (int32_t)(ch + 1));
          st.seams++;
          st.offers++;
          if (ch == 0) {
            const double dl = seam_dist<D>(T, 0, q);
            dr = fmin(dr, dl);
            seam_keep(sb, dl, 0);
            st.seams++;
            st.offers++;
          }
        }
        double m = dr;
        m = fmin(m, __shfl_xor_sync(gmask, m, 4));
        m = fmin(m, __shfl_xor_sync(gmask, m, 2));
        m = fmin(m, __shfl_xor_sync(gmask, m, 1));
        if (m < dmin) {  // group-uniform
          dmin = m;
          thr = cut_key(cut2(dmin, scale), fb);
        }
        const bool park = keep && key <= thr;
        const unsigned pm = (__ballot_sync(gmask, park) >> (lane & 24)) & 0xffu;
        if (npark + __popc(pm) > GPAIRS) {  // list full: flush with the current bound
          flush_pairs<D>(w, T, g, q, cut2(dmin, scale), thr, PC, PL, npark, sub, fall, st.pairs);
          __syncwarp(gmask);
          npark = 0;
        }
        if (park) {
          const int at = npark + __popc(pm & ((1u << sub) - 1));
          PC[at] = (uint32_t)ch;
          PL[at] = key;
        }
        npark += __popc(pm);
      } else {
        // push the kept children: index order, the nearest on top
        const unsigned km = (__ballot_sync(gmask, keep) >> (lane & 24)) & 0xffu;
        if (km) {
          const unsigned mk = __reduce_min_sync(
              gmask, keep ? ((__float_as_uint(key) & ~7u) | sub) : 0xffffffffu);
          const int top = (int)(mk & 7u);
          const unsigned rest = km & ~(1u << top);
          if (keep) {
            const int pos = sub == top ? __popc(km) - 1 : __popc(rest & ((1u << sub) - 1));
            SK[sp + pos] = ((uint32_t)(level - 1) << 28) | (uint32_t)ch;
            SL[sp + pos] = key;
          }
          sp += __popc(km);
          if (sp > NSTACK - FANOUT) {  // cannot happen for the depths in use; stay exact anyway
            fall = true;
            sp = 0;
          }
        }
      }
    }
    __syncwarp();
  }
  // ---- the warp's four queries are done: batched appends (warp converged)
  __syncwarp();
  const double c2f = cut2(dmin, scale);
  const double lim = dmin + 1e-12;
  // seams inside the final band become candidates
  if (sb.dropped <= lim) fall = true;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double d = j == 0 ? sb.d1 : sb.d2;
    if (active && d <= lim) {
      double pt[D], ts;
      seam_point<D>(T, j == 0 ? sb.s1 : sb.s2, pt, ts);
      if (!add_cand(w, g, ts, d, -1.0, (uint32_t)(j == 0 ? sb.s1 : sb.s2))) fall = true;
    }
  }
  // parked leaves that still pass the final bound become pairs
  flush_pairs<D>(w, T, g, q, c2f, thr, PC, PL, npark, sub, fall, st.pairs);
  // group totals to the leader lane
  unsigned long long offers = st.offers + st.pairs;
  offers += __shfl_xor_sync(0xffffffffu, offers, 4);
  offers += __shfl_xor_sync(0xffffffffu, offers, 2);
  offers += __shfl_xor_sync(0xffffffffu, offers, 1);
  const unsigned fbal = __ballot_sync(0xffffffffu, fall) & gmask;
  if (active && sub == 0) {
    double4 rec;
    rec.x = q[0];
    rec.y = q[1];
    rec.z = D == 3 ? q[D - 1] : 0.0;
    rec.w = dmin;
    *(double4*)(w.qs + g * 4) = rec;
    w.scnt[g] = (int64_t)offers;
    w.flag[g] = fbal ? 1 : 0;
    if (fbal) {
      unsigned long long slot = atomicAdd(&w.cnt[3], 1ull);
      w.fb[slot] = g;
    }
  }
  warp_count(w.counters, MREP_CNT_SEAMS, st.seams);
  warp_count(w.counters, MREP_CNT_BOXES, st.boxes);
}

// the query's curve in a batch (-1: out-of-range id, sorted last: NaN
// result, no work)
template <bool MULTI>
__device__ __forceinline__ int32_t group_curve(const WaveParams& w, int64_t g, bool& active,
                                               int sub) {
  if (!MULTI || !active) return 0;
  const int64_t qi = w.perm ? (int64_t)w.perm[g] : g;
  int32_t cid = w.qcurve[qi];
  if (cid < 0 || cid >= w.ncurves) {
    if (sub == 0) {
      w.gcur[g] = -1;
      w.scnt[g] = 0;
      w.flag[g] = 0;
    }
    active = false;
    cid = 0;
  }
  return cid;
}

template <int D, bool MULTI>
__global__ void __launch_bounds__(BLOCK, MREP_GROUP_MINB) wave_traverse_group(const __grid_constant__ WaveParams w) {
  __shared__ uint32_t sk[BLOCK / 8][GSTACK];
  __shared__ float sl[BLOCK / 8][GSTACK];
  __shared__ uint32_t pc[BLOCK / 8][GPAIRS];
  __shared__ float pl[BLOCK / 8][GPAIRS];
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 3;
  if (!MULTI) {
    int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    bool act = g < w.n;
    traverse_group<D, false, GSTACK, false>(w, g, act, 0, w.tab, BoxSrc<false>{w.tab.fbox}, sk[grp],
                                            sl[grp], pc[grp], pl[grp], lane);
  } else {
    // persistent warps drain 4-query tasks, heaviest curves first; the next
    // task index is fetched while the current one runs
    unsigned long long task = 0;
    if (lane == 0) task = atomicAdd(w.queue, 1ull);
    task = __shfl_sync(0xffffffffu, task, 0);
    for (;;) {
      int64_t base = (int64_t)task * 4;
      if (base >= w.n) break;
      unsigned long long next = 0;
      if (lane == 0) next = atomicAdd(w.queue, 1ull);
      int64_t g = base + (lane >> 3);
      bool act = g < w.n;
      const int32_t cid = group_curve<true>(w, g, act, lane & 7);
      const TableView& T = w.tabs[cid];
      // curve sets with per-curve cell indices: the group scans the query's
      // cell list when every active query of the warp lies in its grid
      bool scan = false;
      if (w.set_cells) {
        bool in = true;
        if (act) {
          const int64_t qi = w.perm ? (int64_t)w.perm[g] : g;
          double qq[D];
#pragma unroll
          for (int k = 0; k < D; ++k) qq[k] = w.q[qi * D + k];
          int64_t cell = 0;
          in = cell_of<D>(T, qq, cell);
        }
        scan = __all_sync(0xffffffffu, in);
      }
      if (scan)
        traverse_group<D, true, GSTACK, false, true>(w, g, act, cid, T, BoxSrc<false>{T.fbox},
                                                     sk[grp], sl[grp], pc[grp], pl[grp], lane);
      else
        traverse_group<D, true, GSTACK, false>(w, g, act, cid, T, BoxSrc<false>{T.fbox}, sk[grp],
                                               sl[grp], pc[grp], pl[grp], lane);
      task = __shfl_sync(0xffffffffu, next, 0);
    }
  }
}

// ---------------------------------------------------------------------------
// W1, staged group mode for curve batches (the paper's scheduler with
// coalesced segment staging, north-star subsystem 4).  A task is a tile of
// up to STG_TILE sorted queries of ONE curve (queries are sorted by curve
// rank, heaviest curve first; stage_plan_kernel cut the tiles).  A
// persistent CTA takes a task, copies the curve's descriptor and its whole
// float box hierarchy (every level, 24 B per box) into shared memory with
// one TMA bulk copy (cp.async.bulk, completion on an mbarrier), and its
// warps then walk the tree for the tile's queries four at a time (one
// 8-lane group per query, as wave_traverse_group) with every box test an
// LDS instead of a dependent L2/HBM load.  Seams (one contiguous 192-B run
// per leaf expansion) and the Bernstein tests of parked leaves still read
// global memory.  Curves whose boxes exceed the stage buffer run the same
// walk from global memory.  Same arithmetic, same decisions: results
// (including cand) equal wave_traverse_group's bit for bit.
constexpr int STG_THREADS = 256;
constexpr int STG_GROUPS = STG_THREADS / 8;
constexpr int STG_STACK = 40;  // top <= 4 when staged: depth <= 1 + 7 * 4 = 29
constexpr int STG_TILE = 256;

struct StagePlan {
  const uint32_t* order;   // [nc] curve of scheduler rank r
  const uint32_t* qstart;  // [nc + 1] first sorted position of rank r
  const uint32_t* tstart;  // [nc + 1] first task of rank r
  int64_t nc;
  unsigned long long* queue;  // task counter
  int64_t stage_bytes;        // float-box capacity of the stage buffer
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MREP_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MREP_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// counting sort of a batch's queries by curve rank (sparse batches):
// queries per rank, then each query's sorted position = first position of
// its rank + a warp-aggregated cursor (lanes of one rank share one atomic).
// Invalid curve ids take rank nc (sorted after every valid query).
__global__ void rank_count_kernel(const int32_t* qcurve, int64_t n, const uint32_t* rank, int64_t nc,
                                  uint32_t* rcnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = qcurve[i];
  const uint32_t r = (c < 0 || c >= nc) ? (uint32_t)nc : rank[c];
  const unsigned peers = __match_any_sync(__activemask(), r);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&rcnt[r], (unsigned)__popc(peers));
}

__global__ void rank_scatter_kernel(const int32_t* qcurve, int64_t n, const uint32_t* rank,
                                    int64_t nc, const uint32_t* qstart, uint32_t* cursor,
                                    uint32_t* perm, uint32_t* inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = qcurve[i];
  const uint32_t r = (c < 0 || c >= nc) ? (uint32_t)nc : rank[c];
  const unsigned peers = __match_any_sync(__activemask(), r);
  const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(&cursor[r], (unsigned)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  const uint32_t pos = qstart[r] + base + __popc(peers & ((1u << lane) - 1));
  perm[pos] = (uint32_t)i;
  if (inv) inv[i] = pos;  // caller -> sorted position (coalesced)
}

// per-rank query counts -> first sorted position and first task of each
// rank (one block: nc is the number of curves, ~1e4)
__global__ void __launch_bounds__(1024) stage_plan_kernel(const uint32_t* cnt, int64_t nc,
                                                          uint32_t* qstart, uint32_t* tstart) {
  __shared__ uint32_t sq[1024], stt[1024];
  const int t = threadIdx.x;
  const int64_t per = (nc + 1023) / 1024, lo = t * per, hi = lo + per < nc ? lo + per : nc;
  uint32_t aq = 0, at = 0;
  for (int64_t r = lo; r < hi; ++r) {
    aq += cnt[r];
    at += (cnt[r] + STG_TILE - 1) / STG_TILE;
  }
  sq[t] = aq;
  stt[t] = at;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan
    uint32_t vq = t >= o ? sq[t - o] : 0, vt = t >= o ? stt[t - o] : 0;
    __syncthreads();
    sq[t] += vq;
    stt[t] += vt;
    __syncthreads();
  }
  uint32_t bq = sq[t] - aq, bt = stt[t] - at;
  for (int64_t r = lo; r < hi; ++r) {
    qstart[r] = bq;
    tstart[r] = bt;
    bq += cnt[r];
    bt += (cnt[r] + STG_TILE - 1) / STG_TILE;
  }
  if (t == 1023) {
    qstart[nc] = sq[1023];
    tstart[nc] = stt[1023];
  }
}

template <int D>
__global__ void __launch_bounds__(STG_THREADS, MREP_STAGE_MINB) wave_traverse_staged(const __grid_constant__ WaveParams w,
                                                                      const __grid_constant__ StagePlan P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t sk[STG_GROUPS][STG_STACK];
  __shared__ float sl[STG_GROUPS][STG_STACK];
  __shared__ uint32_t pc[STG_GROUPS][GPAIRS];
  __shared__ float pl[STG_GROUPS][GPAIRS];
  __shared__ TableView tv;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int64_t t_lo, t_hi;
  __shared__ int32_t t_cid;
  __shared__ unsigned t_cursor;
  float* fbs = reinterpret_cast<float*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 3;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t ntask = P.tstart[P.nc];
  unsigned phase = 0;
  for (;;) {
    if (tid == 0) {
      const unsigned long long task = atomicAdd(P.queue, 1ull);
      int64_t r = -1;
      if (task < ntask) {  // rank of the task: last r with tstart[r] <= task
        int64_t a = 0, b = P.nc;
        while (b - a > 1) {
          const int64_t m = (a + b) >> 1;
          if (P.tstart[m] <= task) a = m;
          else b = m;
        }
        r = a;
      }
      if (r < 0) {
        t_lo = t_hi = 0;
        t_cid = -1;
      } else {
        const int64_t q0 = P.qstart[r], q1 = P.qstart[r + 1];
        t_lo = q0 + (int64_t)(task - P.tstart[r]) * STG_TILE;
        t_hi = t_lo + STG_TILE < q1 ? t_lo + STG_TILE : q1;
        t_cid = (int32_t)P.order[r];
      }
      t_cursor = 0;
    }
    __syncthreads();
    const int32_t cid = t_cid;
    if (cid < 0) break;
    if (tid < (int)(sizeof(TableView) / 8))  // descriptor -> shared memory
      reinterpret_cast<uint64_t*>(&tv)[tid] = reinterpret_cast<const uint64_t*>(&w.tabs[cid])[tid];
    __syncthreads();
    const int64_t nbox = tv.lvl_off[tv.top] + tv.lvl_cnt[tv.top];
    const unsigned bytes = (unsigned)(((nbox * 24) + 15) & ~(int64_t)15);
    const bool staged = (int64_t)bytes <= P.stage_bytes;
    if (staged) {
      if (tid == 0) {
        // the previous task's generic-proxy reads of the buffer are ordered
        // (__syncthreads) before this async-proxy overwrite
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(fbs, tv.fbox, bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
    }
    const int64_t lo = t_lo, m = t_hi - t_lo;
    for (;;) {  // the warp's next four queries of the tile
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(&t_cursor, 4u);
      base = __shfl_sync(0xffffffffu, base, 0);
      if ((int64_t)base >= m) break;
      const int64_t g = lo + base + (lane >> 3);
      bool act = (int64_t)(base + (lane >> 3)) < m;
      if (staged)
        traverse_group<D, true, STG_STACK, true>(w, g, act, cid, tv, BoxSrc<true>{fbs}, sk[grp],
                                                 sl[grp], pc[grp], pl[grp], lane);
      else
        traverse_group<D, true, STG_STACK, false>(w, g, act, cid, tv, BoxSrc<false>{tv.fbox},
                                                  sk[grp], sl[grp], pc[grp], pl[grp], lane);
    }
    __syncthreads();  // the stage buffer and descriptor are reused by the next task
  }
  // queries with an out-of-range curve id (sorted after every valid one)
  const int64_t nvalid = P.qstart[P.nc];
  for (int64_t g = nvalid + (int64_t)blockIdx.x * STG_THREADS + tid; g < w.n;
       g += (int64_t)gridDim.x * STG_THREADS) {
    w.gcur[g] = -1;
    w.scnt[g] = 0;
    w.flag[g] = 0;
  }
}

// W2a: the cheap tests of every traversal pair (box re-test with the final
// seam bound, Bernstein distance bound, one-signed E) -- about half the pairs
// stop here; the rest are compacted so W2b's quartic + pieces run on
// uniformly hard work (less divergence).
template <int D, bool MULTI>
__global__ void __launch_bounds__(BLOCK) wave_pairs_filter(const __grid_constant__ WaveParams w) {
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[0];
  if (total > w.pcap) total = w.pcap;
  uint64_t nboxes = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t qi = w.pq[i];  // sorted position
    int64_t s = w.ps[i];
    const TableView& T = tab_of<MULTI>(w, qi);
    double4 rec = *(const double4*)(w.qs + qi * 4);
    double q[D];
    q[0] = rec.x;
    q[1] = rec.y;
    if (D == 3) q[D - 1] = rec.z;
    double scale = T.hdr[4];
#pragma unroll
    for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
    const double c2 = cut2(rec.w, scale);  // the query's final seam bound
    ++nboxes;
    bool keep = (fbox_ok(scale) ? box_lb2f<D>(T, T.lvl_off[0] + s, make_fq<D>(q, scale))
                                : box_lb2<D>(T, T.lvl_off[0] + s, q)) <= c2;
    if (keep) keep = pair_may_survive<D>(T, s, q, c2);
    unsigned long long slot = wave_append(&w.cnt[7], keep);
    if (keep) {  // the fused cell-scan pairs share the list: check the capacity
      if (slot < w.pcap) {
        w.pq2[slot] = (uint32_t)qi;
        w.ps2[slot] = (uint32_t)s;
      } else if (atomicExch(&w.flag[qi], 1) == 0) {  // finished by the fallback kernel
        unsigned long long fs = atomicAdd(&w.cnt[3], 1ull);
        w.fb[fs] = qi;
      }
    }
  }
  warp_count(w.counters, MREP_CNT_BOXES, nboxes);
}

// The survivor buffer is split into CLIP_QP partitions: W2b's warps append
// to partition (warp % CLIP_QP) through its own counter and W3 claims from
// each partition through another (every counter on its own 128-B line after
// the 8 pipeline counters).  One counter for all of them was both kernels'
// top stall: every warp's append / refill atomic hit a single L2 address.
#ifndef MREP_CLIP_QP
#define MREP_CLIP_QP 32
#endif
constexpr int CLIP_QP = MREP_CLIP_QP, CLIP_QS = 16;
constexpr int CNT_WORDS = 8 + 2 * CLIP_QP * CLIP_QS;
__device__ __forceinline__ unsigned long long* clip_claims(const WaveParams& w) { return w.cnt + 8; }
__device__ __forceinline__ unsigned long long* surv_appends(const WaveParams& w) {
  return w.cnt + 8 + CLIP_QP * CLIP_QS;
}

// W2b: E' roots, monotone pieces, elimination for the filtered pairs
template <int D, bool MULTI>
__global__ void __launch_bounds__(BLOCK, MREP_PAIRS_MINB) wave_pairs(const __grid_constant__ WaveParams w) {
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[7];
  if (total > w.pcap) total = w.pcap;
  uint64_t npairs = 0;
  const int part = (int)(((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % CLIP_QP);
  unsigned long long* const acnt = surv_appends(w) + part * CLIP_QS;
  const unsigned long long pcap = w.scap / CLIP_QP, pbase = (unsigned long long)part * pcap;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t qi = w.pq2[i];  // sorted position
    int64_t s = w.ps2[i];
    const TableView& T = tab_of<MULTI>(w, qi);
    double4 rec = *(const double4*)(w.qs + qi * 4);
    double q[D];
    q[0] = rec.x;
    q[1] = rec.y;
    if (D == 3) q[D - 1] = rec.z;
    double scale = T.hdr[4];
#pragma unroll
    for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
    const double c2 = cut2(rec.w, scale);  // the query's final seam bound
    PairPrep P;
    if (!prep_pair_cut<D>(T, s, q, c2, P)) continue;  // (W2a already passed it)
    ++npairs;
    double lo = 0.0;
#pragma unroll 1
    for (int k = 0; k <= P.nin; ++k) {
      double hi = (k == P.nin) ? 1.0 : (k == 0 ? P.b1 : (k == 1 ? P.b2 : (k == 2 ? P.b3 : P.b4)));
      double bp[6];
      restrict_ordinates(P.bseg, lo, hi, bp);
      bool surv = bp[0] < 0.0 && bp[0] * bp[5] <= 0.0;
      unsigned long long slot = wave_append(acnt, surv);
      if (surv) {
        if (slot < pcap) {
          slot += pbase;
          double* o = w.sb + slot * 8;
#pragma unroll
          for (int j = 0; j < 6; ++j) o[j] = bp[j];
          o[6] = lo;
          o[7] = hi;
          w.sq[slot] = (uint32_t)qi;
          w.ssk[slot] = (uint32_t)((s << 3) | k);
        } else if (atomicExch(&w.flag[qi], 1) == 0) {  // finished by the fallback kernel
          unsigned long long fs = atomicAdd(&w.cnt[3], 1ull);
          w.fb[fs] = qi;
        }
      }
      lo = hi;
    }
  }
  warp_count(w.counters, MREP_CNT_PAIRS, npairs);
}


// W3 with lane refill: each lane runs one clipping iteration of its current
// survivor per loop trip and takes the next survivor from the queue as soon
// as its own is finished (1..8 iterations per survivor no longer leave
// lanes idle).  Same arithmetic as clip_root (clip_init + clip_step).
template <int D, bool MULTI>
__global__ void __launch_bounds__(BLOCK, MREP_CLIP_MINB) wave_clip(const __grid_constant__ WaveParams w) {
  unsigned long long* qctr = clip_claims(w);           // partition p's claims at qctr[p * CLIP_QS]
  const unsigned long long* actr = surv_appends(w);   // and its survivors at actr[p * CLIP_QS]
  const unsigned long long pcap = w.scap / CLIP_QP;
  auto part_end = [&](int p) {  // survivors stored in partition p
    const unsigned long long c = *(volatile const unsigned long long*)(actr + p * CLIP_QS);
    return c < pcap ? c : pcap;
  };
  const int lane = threadIdx.x & 31;
  uint64_t nsurv = 0, nit = 0, nmiss = 0;
  bool have = false, drained = false;  // drained: warp-uniform, every partition claimed
  int part = (int)(((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % CLIP_QP);
  unsigned long long pend_n = part_end(part);  // warp-uniform
  int64_t qi = 0;
  uint32_t sk = 0;
  double plo = 0.0, phi = 0.0;
  ClipState S;
  for (;;) {
    const bool want = !have && !drained;
    const unsigned wm = __ballot_sync(0xffffffffu, want);
    if (wm) {
      const int leader = __ffs(wm) - 1;
      const unsigned long long lo = (unsigned long long)part * pcap, hi = lo + pend_n;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(qctr + part * CLIP_QS, (unsigned long long)__popc(wm));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (want) {
        const unsigned long long i = lo + base + __popc(wm & ((1u << lane) - 1));
        if (i < hi) {
          // no flag test here: a survivor of a query already handed to the
          // fallback is clipped anyway (harmless: emit skips the query and the
          // fallback recomputes it), which keeps the refill's loads independent
          qi = w.sq[i];
          const double* o = w.sb + i * 8;
          double bp[6];
#pragma unroll
          for (int j = 0; j < 6; ++j) bp[j] = o[j];
          plo = o[6];
          phi = o[7];
          sk = w.ssk[i];
          clip_init(S, bp);
          have = true;
        }
      }
      if (lo + base + __popc(wm) >= hi) {
        // this partition is used up: one load per lane reads the claim
        // counters of all partitions, the warp moves to the first with work
        const int pp = (part + 1 + lane) % CLIP_QP;
        const unsigned long long c = *(volatile unsigned long long*)(qctr + pp * CLIP_QS);
        const unsigned long long e = part_end(pp);
        const bool avail = c < e;
        const unsigned am = __ballot_sync(0xffffffffu, avail);
        if (am) {
          const int src = __ffs(am) - 1;
          part = __shfl_sync(0xffffffffu, pp, src);
          pend_n = __shfl_sync(0xffffffffu, e, src);
        } else {
          drained = true;
        }
      }
    }
    if (drained && __all_sync(0xffffffffu, !have)) break;
    if (!have) continue;
    if (!clip_step(S, w.clip_tol, w.max_iter)) continue;
    have = false;
    const ClipOut& co = S.r;
    ++nsurv;
    nit += (uint64_t)co.used;
    if (!co.ok) {
      ++nmiss;
      continue;
    }
    const TableView& T = tab_of<MULTI>(w, qi);
    const int64_t s = sk >> 3;
    const double* r = T.rec + s * REC;
    double ta = __ldg(r + R_TA), tb = __ldg(r + R_TB);
    double v = plo + co.root * (phi - plo);
    double acc = 0.0;
#pragma unroll
    for (int dim = 0; dim < D; ++dim) {
      double f = decasteljau1(__ldg(r + R_P + dim), __ldg(r + R_P + 3 + dim), __ldg(r + R_P + 6 + dim),
                              __ldg(r + R_P + 9 + dim), v);
      double diff = w.qs[qi * 4 + dim] - f;
      acc += diff * diff;
    }
    double d = sqrt(acc);
    double t = ta + v * (tb - ta);
    double cur = dmin_of(w, qi);
    bool keep = d <= cur + 1e-12;
    if (keep) {
      atomicMin(dmin_ptr(w, qi), (unsigned long long)__double_as_longlong(d));
      if (!add_cand(w, qi, t, d, v, CAND_SURV | (uint32_t)sk) &&
          atomicExch(&w.flag[qi], 1) == 0) {
        unsigned long long fs = atomicAdd(&w.cnt[3], 1ull);
        w.fb[fs] = qi;
      }
    }
  }
  warp_count(w.counters, MREP_CNT_SURVIVORS, nsurv);
  warp_count(w.counters, MREP_CNT_CLIP_ITERS, nit);
  warp_count(w.counters, MREP_CNT_HULL_MISS, nmiss);
}

// W4: selection + emit, one thread per sorted query walking its candidate
// list: the reference's rule (_kernels.py:480-490) -- minimum distance, then
// inside dmin + 1e-12 the smallest t (-0.0 == +0.0), then the smallest
// reference order -- then the winner's foot point (recomputed exactly as the
// reference stores it) and one scattered write of the outputs.
template <int D, bool MULTI>
__global__ void __launch_bounds__(256) wave_emit(const __grid_constant__ WaveParams w) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= w.n) return;
  if (w.flag[g]) return;  // written by the fallback kernel
  const int64_t qi = (w.perm && !w.orec) ? (int64_t)w.perm[g] : g;
  if (w.out_cand && !w.orec) w.out_cand[qi] = w.scnt[g];
  const uint32_t nc = w.ccnt[g];
  const double4* row = reinterpret_cast<const double4*>(w.cin + g * CIN);
  // the running minimum is the smallest candidate distance: the seam that
  // set the traversal's bound is in its band and every survivor that lowered
  // it was appended (an overflow of either sends the query to the fallback),
  // so the row gives it without reading the query's state record
  double4 rr[CIN];
  double dm = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
  for (int k = 0; k < CIN; ++k) {
    rr[k] = (uint32_t)k < nc ? row[k] : make_double4(0.0, dm, 0.0, 0.0);
    dm = fmin(dm, rr[k].y);
  }
  if (nc > (uint32_t)CIN) {
    for (uint32_t c = w.chead[g]; c != ~0u;) {
      const double4 r = *reinterpret_cast<const double4*>(w.cand + c);
      c = (uint32_t)((uint64_t)__double_as_longlong(r.w) >> 32);
      dm = fmin(dm, r.y);
    }
  }
  const double lim = dm + 1e-12;
  unsigned long long bt = ~0ull;
  uint32_t bo = ~0u;
  bool found = false;
  double best_t = 0.0, best_d = 0.0, best_v = 0.0;
  auto consider = [&](const double4 r) {
    if (!(r.y <= lim)) return;
    const unsigned long long tk = tkey_of(r.x);
    const uint32_t ok = (uint32_t)(uint64_t)__double_as_longlong(r.w);
    if (tk < bt || (tk == bt && ok < bo)) {
      bt = tk;
      bo = ok;
      best_t = r.x;
      best_d = r.y;
      best_v = r.z;
      found = true;
    }
  };
#pragma unroll
  for (int k = 0; k < CIN; ++k)
    if ((uint32_t)k < nc) consider(rr[k]);
  if (nc > (uint32_t)CIN) {
    for (uint32_t c = w.chead[g]; c != ~0u;) {
      const double4 r = *reinterpret_cast<const double4*>(w.cand + c);
      c = (uint32_t)((uint64_t)__double_as_longlong(r.w) >> 32);
      consider(r);
    }
  }
  if (!found) {
    const double NaN = __longlong_as_double(0x7ff8000000000000LL);
    if (w.orec) {
      double* o = w.orec + g * 8;
      o[0] = NaN;
      o[1] = NaN;
#pragma unroll
      for (int k = 0; k < 3; ++k) o[2 + k] = NaN;
      o[5] = __longlong_as_double((long long)w.scnt[g]);
      o[6] = __longlong_as_double(-1LL);
      return;
    }
    w.out_t[qi] = NaN;
    w.out_dist[qi] = NaN;
#pragma unroll
    for (int k = 0; k < D; ++k) w.out_foot[qi * D + k] = NaN;
    if (w.out_seg) w.out_seg[qi] = -1;
    return;
  }
  const TableView& T = tab_of<MULTI>(w, g);
  double foot[D];
  int32_t seg;
  if (bo & CAND_SURV) {
    int64_t s = (int64_t)((bo & ~CAND_SURV) >> 3);
    const double* r = T.rec + s * REC;
    double v = best_v;
#pragma unroll
    for (int dim = 0; dim < D; ++dim)
      foot[dim] = decasteljau1(r[R_P + dim], r[R_P + 3 + dim], r[R_P + 6 + dim], r[R_P + 9 + dim], v);
    seg = (int32_t)s;
  } else {
    int64_t s = (int64_t)bo;
    double stt;
    seam_point<D>(T, s, foot, stt);
    seg = (int32_t)(s > 0 ? s - 1 : 0);
  }
  if (w.orec) {
    // sorted-order staging record (two full 32-B sectors per query); the
    // unpermute pass writes the caller-order outputs coalesced
    double4* o = reinterpret_cast<double4*>(w.orec + g * 8);
    o[0] = make_double4(best_t, best_d, foot[0], foot[1]);
    o[1] = make_double4(D == 3 ? foot[D - 1] : 0.0, __longlong_as_double((long long)w.scnt[g]),
                        __longlong_as_double((long long)seg), 0.0);
    return;
  }
  w.out_t[qi] = best_t;
  w.out_dist[qi] = best_d;
#pragma unroll
  for (int k = 0; k < D; ++k) w.out_foot[qi * D + k] = foot[k];
  if (w.out_seg) w.out_seg[qi] = seg;
}

// Large batches: caller-order outputs from the sorted staging records, one
// thread per CALLER index -- every output array written coalesced (the
// scattered 8-B writes of wave_emit would cost partial-sector DRAM
// read-modify-writes once the outputs exceed L2).  Fallback queries were
// written directly by wave_fallback and are skipped.
template <int D>
__global__ void __launch_bounds__(256) wave_unpermute(const __grid_constant__ WaveParams w) {
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= w.n) return;
  const int64_t g = w.inv[qi];
  if (w.flag[g]) return;
  const double4* o = reinterpret_cast<const double4*>(w.orec + g * 8);
  const double4 a = o[0], b = o[1];
  w.out_t[qi] = a.x;
  w.out_dist[qi] = a.y;
  w.out_foot[qi * D] = a.z;
  w.out_foot[qi * D + 1] = a.w;
  if (D == 3) w.out_foot[qi * D + D - 1] = b.x;
  if (w.out_cand) w.out_cand[qi] = (int64_t)__double_as_longlong(b.y);
  if (w.out_seg) w.out_seg[qi] = (int32_t)__double_as_longlong(b.z);
}

// diagnostics: emitted pairs / survivors / candidates into counters[7] (packed 21 bits each)
__global__ void wave_diag(const __grid_constant__ WaveParams w) {
  if (w.counters && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long sv = 0;
    for (int p = 0; p < CLIP_QP; ++p) sv += surv_appends(w)[p * CLIP_QS];
    unsigned long long a = w.cnt[0] >> 10, b = sv >> 10, c = w.cnt[2] >> 10;
    atomicAdd((unsigned long long*)&w.counters[7], (a & 0x1fffff) | ((b & 0x1fffff) << 21) |
                                                       ((c & 0x1fffff) << 42));
  }
}

// exact per-thread path for the rare queries the buffers could not hold
template <int D, bool MULTI>
__global__ void __launch_bounds__(BLOCK) wave_fallback(const __grid_constant__ WaveParams w,
                                                       const __grid_constant__ ProjParams p) {
  unsigned long long total = *(volatile unsigned long long*)&w.cnt[3];
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int64_t g = w.fb[i];
    int64_t qi = w.perm ? (int64_t)w.perm[g] : g;
    const TableView& T = tab_of<MULTI>(w, g);
    double q[D];
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = w.qs[g * 4 + k];
    double scale = T.hdr[4];
#pragma unroll
    for (int k = 0; k < D; ++k) scale = fmax(scale, fabs(q[k]));
    Band B;
    band_init(B, false, 0.0);
    QStats st{};
    gen_screened<D, false>(T, q, scale, w.clip_tol, w.max_iter, B, st);
    if (B.overflow) {
      double dm = B.dmin;
      band_init(B, true, dm);
      gen_screened<D, false>(T, q, scale, w.clip_tol, w.max_iter, B, st);
      write_winner<D>(T, p, qi, Pick{B.t[0], B.d[0], B.v[0], B.ord[0], B.valid != 0});
    } else {
      write_winner<D>(T, p, qi, band_pick(B));
    }
    if (w.out_cand) w.out_cand[qi] = (int64_t)st.offers;
  }
  if (w.counters && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd((unsigned long long*)&w.counters[MREP_CNT_PASS2], total);
}

// ------------------------------------------------------------ table build
__global__ void pack_records_kernel(const double* seg_pts, const double* seg_ta,
                                    const double* seg_tb, const double* seam_t,
                                    const double* seam_pt, int64_t S, int d, double* hdr,
                                    double* rec, double* box0, double* sxyz) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) {
    hdr[0] = seam_t[0];
    for (int k = 0; k < 3; ++k) hdr[1 + k] = sxyz[k] = k < d ? seam_pt[k] : 0.0;
  }
  if (s >= S) return;
  double* r = rec + s * REC;
  double P[4][3];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 3; ++k) P[j][k] = k < d ? seg_pts[(s * 4 + j) * d + k] : 0.0;
  // a separator record (NaN interval) between the curves of a nearest-over-set
  // table: an empty box (never tested in range), seams still real points
  const bool sep = isnan(seg_ta[s]);
  double amax = 0.0;
  for (int k = 0; k < 3; ++k) {
    double w0, w1, w2, w3;
    cubic_power_coeffs(P[0][k], P[1][k], P[2][k], P[3][k], w0, w1, w2, w3);
    r[0 * 3 + k] = w0;
    r[1 * 3 + k] = w1;
    r[2 * 3 + k] = w2;
    r[3 * 3 + k] = w3;
    double lo = P[0][k], hi = P[0][k];
    for (int j = 0; j < 4; ++j) {
      r[R_P + j * 3 + k] = P[j][k];
      lo = fmin(lo, P[j][k]);
      hi = fmax(hi, P[j][k]);
      amax = fmax(amax, fabs(P[j][k]));
    }
    box0[s * 6 + k] = sep ? INFINITY : lo;
    box0[s * 6 + 3 + k] = sep ? -INFINITY : hi;
  }
  r[R_TA] = seg_ta[s];
  r[R_TB] = seg_tb[s];
  r[R_ST] = seam_t[s + 1];
  for (int k = 0; k < 3; ++k)
    r[R_SP + k] = sxyz[(s + 1) * 3 + k] = k < d ? seam_pt[(s + 1) * d + k] : 0.0;
  r[30] = 0.0;
  r[31] = 0.0;
  // header[4]: max |coordinate| (positive doubles order like their bit patterns)
  atomicMax((unsigned long long*)&hdr[4], (unsigned long long)__double_as_longlong(amax));
}

__global__ void reduce_boxes_kernel(const double* child, int64_t nchild, double* parent,
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

// searchsorted(knots, x, 'right') - 1 clipped to [p, m - p - 2]: the span
// index q of core.py:108-112 whose [t_q, t_{q+1}) holds x (the last nonzero
// span for x at the domain end).  Pure comparisons: bit-exact by construction.
__device__ __forceinline__ int32_t knot_span_of(const double* knots, int64_t m, int p, double x) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (knots[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  int64_t s = lo - 1;
  int64_t last = m - p - 2;
  if (s < p) s = p;
  if (s > last) s = last;
  return (int32_t)s;
}

__global__ void knot_span_kernel(const double* knots, int64_t m, int p, const double* t, int64_t n,
                                 int32_t* span) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  span[i] = knot_span_of(knots, m, p, t[i]);
}

// curve-set variant: query i searches the knot vector of curve curve_ids[i]
// (CSR knots[knot_ofs[c] .. knot_ofs[c+1]))
__global__ void knot_span_batch_kernel(const double* knots, const int64_t* knot_ofs,
                                       const int32_t* degree, const int32_t* curve_ids,
                                       const double* t, int64_t n, int32_t* span) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = curve_ids[i];
  int64_t a = knot_ofs[c];
  span[i] = knot_span_of(knots + a, knot_ofs[c + 1] - a, degree[c], t[i]);
}

// ------------------------------------------------------------ any-degree ordinate ops
// The reference's NonParametricBezier ops work for any degree n
// (_kernels.py:200-341 loop over b.shape[0]); the projection only ever
// builds quintics (the fast fixed-size kernels below), so these runtime-n
// versions back the public per-op API for other degrees.  Same operation
// order as the reference (abscissae i / n, de Casteljau restriction).
constexpr int ORD_NMAX = 32;  // ordinates per polynomial (degree <= 31)

__device__ void restrict_gen(double* cur, int n, double lo, double hi) {
  double tmp[ORD_NMAX], side[ORD_NMAX];
  if (lo > 0.0) {
    for (int i = 0; i <= n; ++i) tmp[i] = cur[i];
    side[n] = cur[n];
    for (int k = 1; k <= n; ++k) {
      for (int i = 0; i < n + 1 - k; ++i) tmp[i] = (1.0 - lo) * tmp[i] + lo * tmp[i + 1];
      side[n - k] = tmp[n - k];
    }
    for (int i = 0; i <= n; ++i) cur[i] = side[i];
    hi = (hi - lo) / (1.0 - lo);
  }
  if (hi < 1.0) {
    for (int i = 0; i <= n; ++i) tmp[i] = cur[i];
    side[0] = cur[0];
    for (int k = 1; k <= n; ++k) {
      for (int i = 0; i < n + 1 - k; ++i) tmp[i] = (1.0 - hi) * tmp[i] + hi * tmp[i + 1];
      side[k] = tmp[0];
    }
    for (int i = 0; i <= n; ++i) cur[i] = side[i];
  }
}

__device__ double eval_gen(const double* b, int n, double u) {
  double tmp[ORD_NMAX];
  for (int i = 0; i <= n; ++i) tmp[i] = b[i];
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < n - k; ++i) tmp[i] = (1.0 - u) * tmp[i] + u * tmp[i + 1];
  return tmp[0];
}

__device__ bool hull_cross_gen(const double* b, int n, double& z1o, double& z2o) {
  double lox[ORD_NMAX], loy[ORD_NMAX], hix[ORD_NMAX], hiy[ORD_NMAX];
  int nl = 0, nh = 0;
  for (int i = 0; i <= n; ++i) {
    const double x = (double)i / (double)n, y = b[i];
    while (nl > 1 && ((lox[nl - 1] - lox[nl - 2]) * (y - loy[nl - 2]) -
                      (x - lox[nl - 2]) * (loy[nl - 1] - loy[nl - 2])) <= 0.0)
      --nl;
    lox[nl] = x;
    loy[nl] = y;
    ++nl;
    while (nh > 1 && ((hix[nh - 1] - hix[nh - 2]) * (y - hiy[nh - 2]) -
                      (x - hix[nh - 2]) * (hiy[nh - 1] - hiy[nh - 2])) >= 0.0)
      --nh;
    hix[nh] = x;
    hiy[nh] = y;
    ++nh;
  }
  double z1 = 2.0, z2 = -1.0;
  for (int chain = 0; chain < 2; ++chain) {
    const double* cx = chain == 0 ? lox : hix;
    const double* cy = chain == 0 ? loy : hiy;
    const int m = chain == 0 ? nl : nh;
    for (int i = 0; i < m - 1; ++i) {
      const double y0 = cy[i], y1 = cy[i + 1];
      double z;
      if (y0 == 0.0) z = cx[i];
      else if (y1 == 0.0) z = cx[i + 1];
      else if ((y0 < 0.0 && 0.0 < y1) || (y1 < 0.0 && 0.0 < y0))
        z = cx[i] + (cx[i + 1] - cx[i]) * (-y0) / (y1 - y0);
      else continue;
      if (z < z1) z1 = z;
      if (z > z2) z2 = z;
    }
    if (m > 0 && cy[m - 1] == 0.0) {
      const double z = cx[m - 1];
      if (z < z1) z1 = z;
      if (z > z2) z2 = z;
    }
  }
  if (z2 < z1) {
    z1o = z2o = 0.0;
    return false;
  }
  z1o = z1;
  z2o = z2;
  return true;
}

// op 0: eval at a[i]; 1: hull crossings -> found, (z1, z2); 2: restrict to
// [a[i], c[i]]; 3: clip_root (tol, max_iter) -> root, ok, used, widths
__global__ void ordinates_gen_kernel(int op, const double* b, int n, int64_t cnt, const double* a,
                                     const double* c, double tol, int max_iter, double* out,
                                     int32_t* i0, int32_t* i1, double* widths) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  double cur[ORD_NMAX];
  for (int k = 0; k <= n; ++k) cur[k] = b[i * (n + 1) + k];
  if (op == 0) {
    out[i] = eval_gen(cur, n, a[i]);
  } else if (op == 1) {
    double z1, z2;
    i0[i] = hull_cross_gen(cur, n, z1, z2) ? 1 : 0;
    out[2 * i] = z1;
    out[2 * i + 1] = z2;
  } else if (op == 2) {
    restrict_gen(cur, n, a[i], c[i]);
    for (int k = 0; k <= n; ++k) out[i * (n + 1) + k] = cur[k];
  } else {  // _kernels.py:306-341
    double* w = widths + i * max_iter;
    double lo = 0.0, hi = 1.0;
    int used = 0;
    for (int it = 0; it < max_iter; ++it) {
      double z1, z2;
      if (!hull_cross_gen(cur, n, z1, z2)) {
        for (int k = it; k < max_iter; ++k) w[k] = hi - lo;
        out[i] = 0.5 * (lo + hi);
        i0[i] = 0;
        i1[i] = it;
        return;
      }
      used = it + 1;
      const double nlo = lo + z1 * (hi - lo), nhi = lo + z2 * (hi - lo);
      if (z2 - z1 < 1e-15) {
        for (int k = it; k < max_iter; ++k) w[k] = 0.0;
        out[i] = nlo;
        i0[i] = 1;
        i1[i] = used;
        return;
      }
      restrict_gen(cur, n, z1, z2);
      lo = nlo;
      hi = nhi;
      w[it] = hi - lo;
      if (hi - lo <= tol) {
        for (int k = it + 1; k < max_iter; ++k) w[k] = hi - lo;
        out[i] = 0.5 * (lo + hi);
        i0[i] = 1;
        i1[i] = used;
        return;
      }
    }
    out[i] = 0.5 * (lo + hi);
    i0[i] = 1;
    i1[i] = used;
  }
}

// ------------------------------------------------------------ per-op kernels
__global__ void quartic_kernel(const double* c, int64_t n, double* roots, int64_t* counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double cc[5];
  for (int k = 0; k < 5; ++k) cc[k] = c[i * 5 + k];
  Roots4 r = quartic_roots_01(cc);
  counts[i] = r.count;
  for (int k = 0; k < 4; ++k)
    if (k < r.count) roots[i * 4 + k] = r.r[k];
}

// _kernels.py:515-566
__global__ void newton_quartic_kernel(const double* cp, int64_t n, double* roots, int64_t* counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c[5];
  for (int k = 0; k < 5; ++k) c[k] = cp[i * 5 + k];
  double scale = 0.0;
  for (int j = 0; j < 5; ++j)
    if (fabs(c[j]) > scale) scale = fabs(c[j]);
  double found[8];
  int nf = 0;
  for (int s = 0; s < 8; ++s) {
    double x = (double)s / 7.0;
    bool conv = false;
    for (int it = 0; it < 40; ++it) {
      double f = c[0] + x * (c[1] + x * (c[2] + x * (c[3] + x * c[4])));
      double df = c[1] + x * (2.0 * c[2] + x * (3.0 * c[3] + x * 4.0 * c[4]));
      if (df == 0.0) break;
      double step = f / df;
      x -= step;
      if (fabs(step) < 1e-14) {
        conv = true;
        break;
      }
    }
    if (!conv) continue;
    double f = c[0] + x * (c[1] + x * (c[2] + x * (c[3] + x * c[4])));
    if (fabs(f) <= 1e-9 * scale && -1e-12 <= x && x <= 1.0 + 1e-12) {
      if (x < 0.0) x = 0.0;
      else if (x > 1.0) x = 1.0;
      bool dup = false;
      for (int k = 0; k < nf; ++k)
        if (fabs(found[k] - x) <= 1e-10) dup = true;
      if (!dup && nf < 8) found[nf++] = x;
    }
  }
  for (int a = 1; a < nf; ++a) {
    double x = found[a];
    int b = a - 1;
    while (b >= 0 && found[b] > x) {
      found[b + 1] = found[b];
      --b;
    }
    found[b + 1] = x;
  }
  int keep = nf < 4 ? nf : 4;
  counts[i] = keep;
  for (int k = 0; k < keep; ++k) roots[i * 4 + k] = found[k];
}

__global__ void distance_poly_kernel(const double* P, const double* q, int64_t n, int d,
                                     double* e) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ee[6];
  if (d == 3) {
    double w[4][3], qq[3];
    for (int k = 0; k < 3; ++k) {
      cubic_power_coeffs(P[(i * 4 + 0) * 3 + k], P[(i * 4 + 1) * 3 + k], P[(i * 4 + 2) * 3 + k],
                         P[(i * 4 + 3) * 3 + k], w[0][k], w[1][k], w[2][k], w[3][k]);
      qq[k] = q[i * 3 + k];
    }
    distance_poly_w<3>(w, qq, ee);
  } else {
    double w[4][2], qq[2];
    for (int k = 0; k < 2; ++k) {
      cubic_power_coeffs(P[(i * 4 + 0) * 2 + k], P[(i * 4 + 1) * 2 + k], P[(i * 4 + 2) * 2 + k],
                         P[(i * 4 + 3) * 2 + k], w[0][k], w[1][k], w[2][k], w[3][k]);
      qq[k] = q[i * 2 + k];
    }
    distance_poly_w<2>(w, qq, ee);
  }
  for (int k = 0; k < 6; ++k) e[i * 6 + k] = ee[k];
}

__global__ void restrict_kernel(const double* b, const double* lo, const double* hi, int64_t n,
                                double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double bb[6], o[6];
  for (int k = 0; k < 6; ++k) bb[k] = b[i * 6 + k];
  restrict_ordinates(bb, lo[i], hi[i], o);
  for (int k = 0; k < 6; ++k) out[i * 6 + k] = o[k];
}

__global__ void eval_ord_kernel(const double* b, const double* u, int64_t n, double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double bb[6];
  for (int k = 0; k < 6; ++k) bb[k] = b[i * 6 + k];
  out[i] = eval_ordinates(bb, u[i]);
}

__global__ void hull_kernel(const double* b, int64_t n, int32_t* found, double* z) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double bb[6];
  for (int k = 0; k < 6; ++k) bb[k] = b[i * 6 + k];
  double z1, z2;
  found[i] = hull_cross(bb, z1, z2) ? 1 : 0;
  z[i * 2] = z1;
  z[i * 2 + 1] = z2;
}

// full widths array variant of clip_root for the per-op API (_kernels.py:306-341)
__global__ void clip_kernel(const double* b, int64_t n, double tol, int max_iter, double* root,
                            int32_t* okp, int32_t* usedp, double* widths) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double cur[6];
  for (int k = 0; k < 6; ++k) cur[k] = b[i * 6 + k];
  double* w = widths + i * max_iter;
  double lo = 0.0, hi = 1.0;
  int used = 0;
  for (int it = 0; it < max_iter; ++it) {
    double z1, z2;
    if (!hull_cross(cur, z1, z2)) {
      for (int k = it; k < max_iter; ++k) w[k] = hi - lo;
      root[i] = 0.5 * (lo + hi);
      okp[i] = 0;
      usedp[i] = it;
      return;
    }
    used = it + 1;
    double nlo = lo + z1 * (hi - lo), nhi = lo + z2 * (hi - lo);
    if (z2 - z1 < 1e-15) {
      for (int k = it; k < max_iter; ++k) w[k] = 0.0;
      root[i] = nlo;
      okp[i] = 1;
      usedp[i] = used;
      return;
    }
    restrict_ordinates(cur, z1, z2, cur);
    lo = nlo;
    hi = nhi;
    w[it] = hi - lo;
    if (hi - lo <= tol) {
      for (int k = it + 1; k < max_iter; ++k) w[k] = hi - lo;
      root[i] = 0.5 * (lo + hi);
      okp[i] = 1;
      usedp[i] = used;
      return;
    }
  }
  root[i] = 0.5 * (lo + hi);
  okp[i] = 1;
  usedp[i] = used;
}

__global__ void cubic_points_kernel(const double* P, const double* u, int64_t n, int d,
                                    double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double uu = u[i];
  for (int k = 0; k < d; ++k)
    out[i * d + k] = decasteljau1(P[(i * 4 + 0) * d + k], P[(i * 4 + 1) * d + k],
                                  P[(i * 4 + 2) * d + k], P[(i * 4 + 3) * d + k], uu);
}

__global__ void rebase_kernel(const double* e, int64_t n, double* b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ee[6], bb[6];
  for (int k = 0; k < 6; ++k) ee[k] = e[i * 6 + k];
  rebase5(ee, bb);
  for (int k = 0; k < 6; ++k) b[i * 6 + k] = bb[k];
}

// ------------------------------------------------------------ launch helpers
template <int D>
static int launch_project(const ProjParams& p, unsigned flags, cudaStream_t st) {
  unsigned grid = grid_for(p.n, BLOCK);
  bool screen = (flags & MREP_SCREEN) && !(flags & MREP_STATS);
  bool stats = (flags & MREP_STATS) != 0;
  if (screen) project_kernel<D, true, false><<<grid, BLOCK, 0, st>>>(p);
  else if (stats) project_kernel<D, false, true><<<grid, BLOCK, 0, st>>>(p);
  else project_kernel<D, false, false><<<grid, BLOCK, 0, st>>>(p);
  MREP_LAUNCH_CHECK();
  unsigned g2 = grid < 148u * 4u ? grid : 148u * 4u;
  if (screen) project_pass2_kernel<D, true><<<g2, BLOCK, 0, st>>>(p);
  else project_pass2_kernel<D, false><<<g2, BLOCK, 0, st>>>(p);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}


enum { TRAV_PACKET = 0, TRAV_LANE = 1, TRAV_GROUP = 2, TRAV_CELLS = 3 };

// staged traversal: resident CTAs per SM (MREP_STAGE_CTAS, 1..3) and the
// float-box stage buffer each gets (the SM's shared memory split evenly,
// minus the kernel's static arrays and the 1 KB the runtime reserves per CTA)
static int stage_ctas_per_sm() {
  static const int c = [] {
    const char* e = getenv("MREP_STAGE_CTAS");
    int v = e ? atoi(e) : MREP_STAGE_MINB;
    return v < 1 ? 1 : (v > 3 ? 3 : v);
  }();
  return c;
}
template <int D>
static int64_t stage_bytes_for(int ctas) {
  int dev = 0, per_sm = 0, per_block = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&per_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, (const void*)wave_traverse_staged<D>);
  int64_t b = (int64_t)per_sm / ctas - (int64_t)fa.sharedSizeBytes - 1024;
  if (b > (int64_t)per_block - (int64_t)fa.sharedSizeBytes) b = per_block - fa.sharedSizeBytes;
  return b < 0 ? 0 : (b & ~(int64_t)127);
}

static int trav_mode(unsigned flags, int64_t n, int64_t S, int top) {
  // MREP_TRAV=packet|lane|group: force a traversal (A/B experiments)
  static const unsigned forced = [] {
    const char* e = getenv("MREP_TRAV");
    if (!e) return 0u;
    if (!strcmp(e, "packet")) return (unsigned)MREP_PACKET;
    if (!strcmp(e, "lane")) return (unsigned)MREP_PER_LANE;
    if (!strcmp(e, "group")) return (unsigned)MREP_GROUP;
    return 0u;
  }();
  if (forced && !(flags & (MREP_PACKET | MREP_PER_LANE | MREP_GROUP))) flags |= forced;
  // MREP_CELLS: the caller built a cell index (mrep_cells_build) for this table
  if ((flags & MREP_CELLS) && !(flags & (MREP_PACKET | MREP_PER_LANE | MREP_GROUP)))
    return top > 7 ? TRAV_PACKET : TRAV_CELLS;
  if (flags & MREP_PACKET) return TRAV_PACKET;
  if (flags & MREP_PER_LANE) return top > 7 ? TRAV_PACKET : TRAV_LANE;
  if (flags & MREP_GROUP) return top > 8 ? TRAV_PACKET : TRAV_GROUP;
  // packet walks when the queries are dense along the curve (Morton
  // neighbours share their BVH path); one 8-lane group per query otherwise
  if (n >= 8 * S || top > 8) return TRAV_PACKET;
  return TRAV_GROUP;
}

// resident blocks x SMs of a kernel on the current device (cached: the
// occupancy query costs microseconds of host time per launch otherwise)
static unsigned persistent_grid(const void* fn, int block) {
  struct Key {
    const void* fn;
    int block, dev;
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, unsigned>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& e : cache)
    if (e.first.fn == fn && e.first.block == block && e.first.dev == dev) return e.second;
  int sms = 148, per = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, block, 0);
  const unsigned g = (unsigned)(sms * (per > 0 ? per : 1));
  cache.push_back({Key{fn, block, dev}, g});
  return g;
}

template <int D, bool MULTI>
static int launch_wave(const ProjParams& p, cudaStream_t st, bool timing, int tmode,
                       const TableView* tabs = nullptr, const int32_t* qcurve = nullptr,
                       int64_t ncurves = 0, const StagePlan* plan = nullptr,
                       bool set_cells = false) {
  const int64_t n = p.n;
  // MREP_WAVE_PCAP / MREP_WAVE_SCAP (tests): tiny pair / survivor buffers, so
  // the overflow -> fallback paths of every stage run
  static const int64_t pcap_env = [] {
    const char* e = getenv("MREP_WAVE_PCAP");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  static const int64_t scap_env = [] {
    const char* e = getenv("MREP_WAVE_SCAP");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  const unsigned long long pcap =
      (unsigned long long)(pcap_env > 0 ? pcap_env : std::max<int64_t>(16 * n, 1 << 16));
  const unsigned long long scap =
      (unsigned long long)(scap_env > 0 ? scap_env : std::max<int64_t>(2 * n, 1 << 16));
  const unsigned long long ccap = (unsigned long long)std::max<int64_t>(n, 1 << 16);
  size_t bytes = 0;
  auto take = [&](size_t b) {
    size_t o = bytes;
    bytes += (b + 255) & ~(size_t)255;
    return o;
  };
  size_t o_cnt = take(CNT_WORDS * sizeof(unsigned long long));
  size_t o_dmin = take(n * 8), o_flag = take(n * 4);
  size_t o_pq = take(pcap * 4), o_ps = take(pcap * 4), o_pq2 = take(pcap * 4),
         o_ps2 = take(pcap * 4);
  size_t o_sb = take(scap * 64), o_sq = take(scap * 4), o_ssk = take(scap * 4);
  size_t o_cand = take(ccap * sizeof(Cand)), o_chead = take(n * 4);
  size_t o_ccnt = take(n * 4), o_cin = take(n * CIN * sizeof(Cand));
  size_t o_orec = p.inv ? take(n * 64) : 0;
  size_t o_fb = take(n * 8);
  size_t o_qs = take(n * 4 * 8), o_wt = take(n * 8), o_wd = take(n * 8), o_wv = take(n * 8),
         o_sc = take(n * 8);
  size_t o_gc = MULTI ? take(n * 4) : 0;
  char* base = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&base, bytes, st));
  WaveParams w{};
  w.tab = p.tab;
  w.q = p.q;
  w.n = n;
  w.perm = p.perm;
  w.clip_tol = p.clip_tol;
  w.max_iter = p.max_iter;
  w.out_t = p.out_t;
  w.out_foot = p.out_foot;
  w.out_dist = p.out_dist;
  w.out_cand = p.out_cand;
  w.out_seg = p.out_seg;
  w.counters = p.counters;
  w.cnt = (unsigned long long*)(base + o_cnt);
  w.dmin = (unsigned long long*)(base + o_dmin);
  w.flag = (int32_t*)(base + o_flag);
  w.pq = (uint32_t*)(base + o_pq);
  w.ps = (uint32_t*)(base + o_ps);
  w.pq2 = (uint32_t*)(base + o_pq2);
  w.ps2 = (uint32_t*)(base + o_ps2);
  w.pcap = pcap;
  w.sb = (double*)(base + o_sb);
  w.sq = (uint32_t*)(base + o_sq);
  w.ssk = (uint32_t*)(base + o_ssk);
  w.scap = scap;
  w.cand = (Cand*)(base + o_cand);
  w.chead = (uint32_t*)(base + o_chead);
  MREP_CUDA_CHECK(cudaMemsetAsync(w.chead, 0xff, n * 4, st));
  w.inv = p.inv;
  w.orec = w.inv ? (double*)(base + o_orec) : nullptr;
  w.ccnt = (uint32_t*)(base + o_ccnt);
  w.cin = (Cand*)(base + o_cin);
  MREP_CUDA_CHECK(cudaMemsetAsync(w.ccnt, 0, n * 4, st));
  w.ccap = ccap;
  w.fb = (int64_t*)(base + o_fb);
  w.qs = (double*)(base + o_qs);
  w.win_t = (double*)(base + o_wt);
  w.win_d = (double*)(base + o_wd);
  w.win_v = (double*)(base + o_wv);
  w.scnt = (int64_t*)(base + o_sc);
  w.tabs = tabs;
  w.qcurve = qcurve;
  w.ncurves = ncurves;
  w.set_cells = set_cells ? 1 : 0;
  w.gcur = MULTI ? (int32_t*)(base + o_gc) : nullptr;
  w.queue = w.cnt + 5;
  static const int retest_min = [] {
    const char* e = getenv("MREP_RETEST_LEVEL");
    return e ? atoi(e) : 1;
  }();
  w.retest_min = retest_min;
  static const int trav_bern = [] {
    const char* e = getenv("MREP_TRAV_BERN");
    return e ? atoi(e) : 0;
  }();
  static const int trav_sort = [] {
    const char* e = getenv("MREP_TRAV_SORT");
    return e ? atoi(e) : 0;
  }();
  w.trav_bern = trav_bern;
  w.trav_sort = trav_sort;
  // fused W2a: cfg2 0.650 -> 0.638 ms, cfg5 69.9 -> 67.7 ms per 10^8, cfg3 /
  // cfg6 neutral; small batches (cfg1, 10^4) lose 2.5% (the longer traversal
  // kernel is on their latency chain), so it is on from 2^16 queries
  static const int fuse_filter = [] {
    const char* e = getenv("MREP_TRAV_FILTER");
    return e ? atoi(e) : -1;
  }();
  w.fuse_filter = fuse_filter >= 0 ? fuse_filter : (n >= (int64_t(1) << 16) ? 1 : 0);
  MREP_CUDA_CHECK(cudaMemsetAsync(w.cnt, 0, CNT_WORDS * sizeof(unsigned long long), st));
  auto persist_grid = [](const void* fn, int block) { return persistent_grid(fn, block); };
  const unsigned g_pairs = persist_grid((const void*)wave_pairs<D, MULTI>, BLOCK);
  const unsigned g_clip = persist_grid((const void*)wave_clip<D, MULTI>, BLOCK);
  StageTimer tm(timing, st);
  tm.mark();
  if (tmode == TRAV_GROUP && MULTI && plan) {
    // staged: persistent CTAs, one curve tile per task, boxes in shared memory
    StagePlan P = *plan;
    P.queue = w.cnt + 4;
    const int ctas = stage_ctas_per_sm();
    const int64_t stage = stage_bytes_for<D>(ctas);
    P.stage_bytes = stage;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    MREP_CUDA_CHECK(cudaFuncSetAttribute((const void*)wave_traverse_staged<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage));
    wave_traverse_staged<D><<<(unsigned)(sms * ctas), STG_THREADS, (size_t)stage, st>>>(w, P);
  } else if (tmode == TRAV_GROUP) {
    if (MULTI) {
      // persistent: one resident wave of warps drains the task queue
      unsigned need = grid_for(n * 8, BLOCK);
      unsigned g = persist_grid((const void*)wave_traverse_group<D, true>, BLOCK);
      wave_traverse_group<D, true><<<g < need ? g : need, BLOCK, 0, st>>>(w);
    } else {
      wave_traverse_group<D, false><<<grid_for(n * 8, BLOCK), BLOCK, 0, st>>>(w);
    }
  } else if (MULTI) {
    unsigned need = grid_for(n, BLOCK);
    if (tmode == TRAV_CELLS) {
      unsigned g = persist_grid((const void*)wave_traverse<D, true, TM_CELLS>, BLOCK);
      wave_traverse<D, true, TM_CELLS><<<g < need ? g : need, BLOCK, 0, st>>>(w);
    } else if (tmode == TRAV_PACKET) {
      unsigned g = persist_grid((const void*)wave_traverse<D, true, TM_PACKET>, BLOCK);
      wave_traverse<D, true, TM_PACKET><<<g < need ? g : need, BLOCK, 0, st>>>(w);
    } else {
      unsigned g = persist_grid((const void*)wave_traverse<D, true, TM_LANE>, BLOCK);
      wave_traverse<D, true, TM_LANE><<<g < need ? g : need, BLOCK, 0, st>>>(w);
    }
  } else if (tmode == TRAV_PACKET) {
    wave_traverse<D, false, TM_PACKET><<<grid_for(n, BLOCK), BLOCK, 0, st>>>(w);
  } else if (tmode == TRAV_CELLS) {
    static const bool dmma = getenv("MREP_TRAV_DMMA") != nullptr;
    if (dmma && D == 3)
      wave_traverse_dmma<D><<<grid_for((n + 7) / 8 * 32, BLOCK), BLOCK, 0, st>>>(w);
    else
      wave_traverse<D, false, TM_CELLS><<<grid_for(n, BLOCK), BLOCK, 0, st>>>(w);
  } else {
    wave_traverse<D, false, TM_LANE><<<grid_for(n, BLOCK), BLOCK, 0, st>>>(w);
  }
  MREP_LAUNCH_CHECK();
  tm.mark();
  wave_pairs_filter<D, MULTI><<<g_pairs, BLOCK, 0, st>>>(w);
  wave_pairs<D, MULTI><<<g_pairs, BLOCK, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  wave_clip<D, MULTI><<<g_clip, BLOCK, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  tm.mark();
  wave_emit<D, MULTI><<<grid_for(n, 256), 256, 0, st>>>(w);
  MREP_LAUNCH_CHECK();
  if (w.inv) {  // flagged queries are skipped: the fallback writes them
    wave_unpermute<D><<<grid_for(n, 256), 256, 0, st>>>(w);
    MREP_LAUNCH_CHECK();
  }
  tm.mark();
  wave_fallback<D, MULTI><<<148u, BLOCK, 0, st>>>(w, p);
  MREP_LAUNCH_CHECK();
  if (getenv("MREP_DIAG")) wave_diag<<<1, 32, 0, st>>>(w);
  tm.mark();
  tm.finish(1);
  MREP_CUDA_CHECK(cudaFreeAsync(base, st));
  return MREP_OK;
}
// ------------------------------------------------------------ curve sets
// A curve set is the device form of many PreparedCurves (the reference's
// prepare_curve applied per curve, project.py:220-242): one allocation holding
// a TableView descriptor per curve, the scheduler rank of each curve, and the
// per-curve tables (same 256-B records + 8-ary AABB hierarchy as a single
// table, each 256-B aligned).
struct CurveSet {
  int64_t nc = 0, S_total = 0;
  int d = 3;
  int rank_bits = 1;
  int max_top = 1;  // deepest AABB hierarchy of the set
  char* mem = nullptr;
  int64_t bytes = 0;
  TableView* desc = nullptr;  // device, [nc]
  uint32_t* rank = nullptr;   // device, [nc]: position in decreasing-cubic-count order
  uint32_t* order = nullptr;  // device, [nc]: curve of each rank (inverse of rank)
  std::vector<int64_t> ofs;   // host, [nc + 1] cubic offsets
  // per-curve cell indices (mrep_curveset_cells_build): one allocation, each
  // curve's index referenced from its own table header
  char* cells = nullptr;
  int64_t cells_bytes = 0;
};

// number of AABB boxes of an S-cubic table (all levels), as table_layout
__device__ __forceinline__ int64_t set_boxes_total(int64_t S) {
  int64_t cnt = S, off = 0;
  for (int lv = 0;; ++lv) {
    off += cnt;
    if (lv >= 1 && cnt <= 1) break;
    cnt = (cnt + FANOUT - 1) / FANOUT;
  }
  return off;
}

__global__ void set_pack_kernel(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                                const int64_t* ofs, const int64_t* tab_off, int64_t nc,
                                int64_t S_total, int d, double* tables) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= S_total) return;
  // curve of cubic g: last c with ofs[c] <= g
  int64_t lo = 0, hi = nc;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (ofs[mid] <= g) lo = mid;
    else hi = mid;
  }
  const int64_t c = lo, s = g - ofs[c], S = ofs[c + 1] - ofs[c];
  double* base = tables + tab_off[c];
  double* hdr = base;
  double* r = base + HDR + s * REC;
  double* box0 = base + HDR + S * REC;
  double P[4][3];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 3; ++k) P[j][k] = k < d ? seg_pts[(g * 4 + j) * d + k] : 0.0;
  double* sxyz = base + HDR + S * REC + set_boxes_total(S) * 9;
  if (s == 0) {  // seam_t[0] = seg_ta[0], seam_pt[0] = seg_pts[0, 0] (project.py:234-235)
    hdr[0] = seg_ta[g];
    for (int k = 0; k < 3; ++k) hdr[1 + k] = sxyz[k] = P[0][k];
  }
  double amax = 0.0;
  for (int k = 0; k < 3; ++k) {
    double w0, w1, w2, w3;
    cubic_power_coeffs(P[0][k], P[1][k], P[2][k], P[3][k], w0, w1, w2, w3);
    r[0 * 3 + k] = w0;
    r[1 * 3 + k] = w1;
    r[2 * 3 + k] = w2;
    r[3 * 3 + k] = w3;
    double blo = P[0][k], bhi = P[0][k];
    for (int j = 0; j < 4; ++j) {
      r[R_P + j * 3 + k] = P[j][k];
      blo = fmin(blo, P[j][k]);
      bhi = fmax(bhi, P[j][k]);
      amax = fmax(amax, fabs(P[j][k]));
    }
    box0[s * 6 + k] = blo;
    box0[s * 6 + 3 + k] = bhi;
  }
  r[R_TA] = seg_ta[g];
  r[R_TB] = seg_tb[g];
  r[R_ST] = seg_tb[g];  // seam_t[s+1] = seg_tb[s], seam_pt[s+1] = seg_pts[s, 3] (project.py:236-237)
  for (int k = 0; k < 3; ++k) r[R_SP + k] = sxyz[(s + 1) * 3 + k] = P[3][k];
  r[30] = 0.0;
  r[31] = 0.0;
  atomicMax((unsigned long long*)&hdr[4], (unsigned long long)__double_as_longlong(amax));
}

// one block per curve builds its AABB levels bottom-up
__global__ void set_boxes_kernel(const TableView* desc) {
  const TableView& T = desc[blockIdx.x];
  double* box = const_cast<double*>(T.box);
  for (int lv = 1; lv <= T.top; ++lv) {
    const double* child = box + T.lvl_off[lv - 1] * 6;
    double* parent = box + T.lvl_off[lv] * 6;
    const int64_t nchild = T.lvl_cnt[lv - 1], npar = T.lvl_cnt[lv];
    for (int64_t i = threadIdx.x; i < npar; i += blockDim.x) {
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
    __syncthreads();
  }
  // float copy of every box of this curve (lo down, hi up)
  const int64_t nb = T.lvl_off[T.top] + T.lvl_cnt[T.top];
  float* fb = const_cast<float*>(T.fbox);
  for (int64_t i = threadIdx.x; i < nb; i += blockDim.x)
    for (int k = 0; k < 3; ++k) {
      fb[i * 6 + k] = __double2float_rd(box[i * 6 + k]);
      fb[i * 6 + 3 + k] = __double2float_ru(box[i * 6 + 3 + k]);
    }
}

// Bernstein fragments of every cubic of a set (after set_boxes_kernel)
__global__ void set_bfrag_kernel(const TableView* desc, const int64_t* ofs, int64_t nc,
                                 int64_t S_total, int d) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= S_total) return;
  int64_t lo = 0, hi = nc;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (ofs[mid] <= g) lo = mid;
    else hi = mid;
  }
  bfrag_cubic(desc[lo], g - ofs[lo], d);
}

// Scheduler key of each query: (rank of its curve, Morton code inside that
// curve's root box).  Sorting by it groups a curve's queries, orders curves
// by decreasing cubic count and makes the lanes of a warp spatial neighbours.
// Queries with an invalid curve id get the largest key (sorted last).
template <int D>
__global__ void morton_multi_kernel(const double* q, const int32_t* qcurve, int64_t n,
                                    const TableView* desc, const uint32_t* rank, int64_t nc,
                                    int end_bit, uint64_t* key, uint32_t* idx, uint32_t* rcnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx[i] = (uint32_t)i;
  int32_t c = qcurve[i];
  if (c < 0 || c >= nc) {
    key[i] = (end_bit >= 64) ? ~0ull : ((1ull << end_bit) - 1ull);
    return;
  }
  if (rcnt) atomicAdd(&rcnt[rank[c]], 1u);  // queries per rank (staged task plan)
  const TableView& T = desc[c];
  const double* box_root = T.box + T.lvl_off[T.top] * 6;
  uint64_t code = 0;
  for (int k = 0; k < D; ++k) {
    double lo = box_root[k], hi = box_root[3 + k];
    double ext = fmax(hi - lo, 1e-300);
    double u = (q[i * D + k] - (lo - ext)) / (3.0 * ext);
    u = fmin(fmax(u, 0.0), 1.0);
    uint32_t cc = (uint32_t)(u * 1023.0);
    for (int b = 0; b < 10; ++b) code |= (uint64_t)((cc >> b) & 1u) << (b * D + k);
  }
  key[i] = ((uint64_t)rank[c] << (10 * D)) | code;
}

int set_create(const double* seg_pts, const double* seg_ta, const double* seg_tb,
               const int64_t* ofs_host, int64_t nc, int d, cudaStream_t st, CurveSet** out) {
  *out = nullptr;
  if (nc < 1 || (d != 2 && d != 3) || !ofs_host || ofs_host[0] != 0) {
    set_error("mrep_curveset_create: need ncurves >= 1, d in {2,3}, seg_ofs[0] == 0");
    return MREP_ERR_ARG;
  }
  for (int64_t c = 0; c < nc; ++c)
    if (ofs_host[c + 1] - ofs_host[c] < 1) {
      set_error("mrep_curveset_create: every curve needs at least one cubic (seg_ofs increasing)");
      return MREP_ERR_ARG;
    }
  CurveSet* cs = new CurveSet();
  cs->nc = nc;
  cs->d = d;
  cs->ofs.assign(ofs_host, ofs_host + nc + 1);
  cs->S_total = ofs_host[nc];
  // layout: [desc nc][rank nc][ofs nc+1][tab_off nc][tables...]
  auto al = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  const int64_t o_desc = 0, o_rank = al(nc * (int64_t)sizeof(TableView));
  const int64_t o_order = o_rank + al(nc * 4);
  const int64_t o_ofs = o_order + al(nc * 4), o_toff = o_ofs + al((nc + 1) * 8);
  const int64_t o_tab = o_toff + al(nc * 8);
  std::vector<int64_t> toff(nc);
  int64_t dbl = 0;
  for (int64_t c = 0; c < nc; ++c) {
    toff[c] = dbl;
    dbl += (table_layout(cs->ofs[c + 1] - cs->ofs[c]).total_doubles + 31) & ~(int64_t)31;
  }
  cs->bytes = o_tab + dbl * 8 + 256;  // slack: bulk copies round sizes up to 16 B
  cudaError_t e = cudaMalloc(&cs->mem, (size_t)cs->bytes);
  if (e != cudaSuccess) {
    set_error(std::string("mrep_curveset_create: cudaMalloc: ") + cudaGetErrorString(e));
    delete cs;
    return MREP_ERR_CUDA;
  }
  double* tables = (double*)(cs->mem + o_tab);
  std::vector<TableView> desc(nc);
  for (int64_t c = 0; c < nc; ++c) {
    desc[c] = table_view(tables + toff[c], cs->ofs[c + 1] - cs->ofs[c]);
    cs->max_top = std::max(cs->max_top, desc[c].top);
  }
  // scheduler rank: curves by decreasing cubic count (ties by index)
  std::vector<int64_t> order(nc);
  for (int64_t c = 0; c < nc; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return cs->ofs[a + 1] - cs->ofs[a] > cs->ofs[b + 1] - cs->ofs[b];
  });
  std::vector<uint32_t> rank(nc), order32(nc);
  for (int64_t i = 0; i < nc; ++i) {
    rank[order[i]] = (uint32_t)i;
    order32[i] = (uint32_t)order[i];
  }
  cs->rank_bits = 1;
  while (((int64_t)1 << cs->rank_bits) < nc + 1) ++cs->rank_bits;
  cs->desc = (TableView*)(cs->mem + o_desc);
  cs->rank = (uint32_t*)(cs->mem + o_rank);
  cs->order = (uint32_t*)(cs->mem + o_order);
  int64_t* ofs_dev = (int64_t*)(cs->mem + o_ofs);
  int64_t* toff_dev = (int64_t*)(cs->mem + o_toff);
  int rc = MREP_OK;
  auto fail = [&](cudaError_t err, const char* what) {
    set_error(std::string("mrep_curveset_create: ") + what + ": " + cudaGetErrorString(err));
    rc = MREP_ERR_CUDA;
  };
  if ((e = cudaMemcpyAsync(cs->desc, desc.data(), nc * sizeof(TableView), cudaMemcpyHostToDevice, st)) != cudaSuccess) fail(e, "desc");
  if (!rc && (e = cudaMemcpyAsync(cs->rank, rank.data(), nc * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) fail(e, "rank");
  if (!rc && (e = cudaMemcpyAsync(cs->order, order32.data(), nc * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) fail(e, "order");
  if (!rc && (e = cudaMemcpyAsync(ofs_dev, cs->ofs.data(), (nc + 1) * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) fail(e, "ofs");
  if (!rc && (e = cudaMemcpyAsync(toff_dev, toff.data(), nc * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) fail(e, "toff");
  if (!rc && (e = cudaMemsetAsync(tables, 0, dbl * 8, st)) != cudaSuccess) fail(e, "memset");
  if (!rc) {
    set_pack_kernel<<<grid_for(cs->S_total, 128), 128, 0, st>>>(seg_pts, seg_ta, seg_tb, ofs_dev,
                                                                toff_dev, nc, cs->S_total, d, tables);
    set_boxes_kernel<<<(unsigned)nc, 128, 0, st>>>(cs->desc);
    set_bfrag_kernel<<<grid_for(cs->S_total, 128), 128, 0, st>>>(cs->desc, ofs_dev, nc,
                                                                  cs->S_total, d);
    if ((e = cudaGetLastError()) != cudaSuccess) fail(e, "pack kernels");
  }
  // the host staging vectors die here: finish the copies before returning
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && !rc) fail(e, "sync");
  if (rc) {
    cudaFree(cs->mem);
    delete cs;
    return rc;
  }
  *out = cs;
  return MREP_OK;
}

// ------------------------------------------------------------ curve-set cell indices
// Every curve of a set gets the single-table cell index (mrep_cells.cuh):
// a uniform grid over its root box, each cell listing the cubics that can
// hold a tie-band candidate for any query of the cell, nearest first.  The
// grid of curve c has G_c = clamp(round(2.5 S_c^(1/3)), 4, gmax) cells per
// axis.  All curves are built together: one thread per (curve, cell) counts
// and fills, one scan sizes every list, and a kernel writes each curve's
// header words, so the build costs a handful of launches for 10^4 curves.
// Layout (int32 words): curve c's index starts at hstart_c + 2 E_c
// (E = exclusive scan of the counts over all cells of all curves, hstart =
// prefix of the padded offset-block sizes cell_head_words(ncell_c)):
// offsets [ncell_c + 1] (padded to even), (key, id) entries [tot_c] --
// exactly what cell_list reads for a single table.
__device__ __forceinline__ int64_t set_cell_owner(const int64_t* cstart, int64_t nc, int64_t i) {
  int64_t lo = 0, hi = nc;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (cstart[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void set_grid_kernel(const TableView* desc, const int32_t* G, int64_t nc, int d,
                                CellGrid* grids) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const TableView& T = desc[c];
  grid_from_root(T.box + T.lvl_off[T.top] * 6, T.hdr[4], G[c], d, grids[c]);
}

__global__ void set_cells_count_kernel(const TableView* desc, const CellGrid* grids,
                                       const int64_t* cstart, int64_t nc, int64_t ncell,
                                       int32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const int64_t c = set_cell_owner(cstart, nc, i);
  cnt[i] = cell_count(desc[c], CurveLeaves{}, grids[c], i - cstart[c]);
}

__global__ void set_cells_header_kernel(const TableView* desc, const CellGrid* grids,
                                        const int64_t* cstart, const int64_t* hstart,
                                        const int64_t* E, int64_t nc, int32_t* mem) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const int64_t e0 = E[cstart[c]], tot = E[cstart[c + 1]] - e0;
  int32_t* off = mem + hstart[c] + 2 * e0;
  off[cstart[c + 1] - cstart[c]] = (int32_t)tot;
  cells_header(grids[c], off, tot, const_cast<double*>(desc[c].hdr) + H_CELLS);
}

__global__ void set_cells_fill_kernel(const TableView* desc, const CellGrid* grids,
                                      const int64_t* cstart, const int64_t* hstart,
                                      const int64_t* E, int64_t nc, int64_t ncell, int32_t* mem) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const int64_t c = set_cell_owner(cstart, nc, i);
  const int64_t e0 = E[cstart[c]], nloc = cstart[c + 1] - cstart[c];
  int32_t* off = mem + hstart[c] + 2 * e0;
  const int32_t at = (int32_t)(E[i] - e0);
  off[i - cstart[c]] = at;
  CellEntry* entries = reinterpret_cast<CellEntry*>(off + cell_head_words(nloc));
  cell_fill_list(desc[c], CurveLeaves{}, grids[c], i - cstart[c], entries + at);
}

static int set_cells_build(CurveSet* cs, int gmax, int64_t max_bytes, cudaStream_t st) {
  if (gmax < 1 || gmax > 64) {
    set_error("mrep_curveset_cells_build: grid_max in [1, 64]");
    return MREP_ERR_ARG;
  }
  if (cs->max_top > 7) {
    set_error("mrep_curveset_cells_build: a curve's hierarchy is too deep (> 8^7 cubics)");
    return MREP_ERR_ARG;
  }
  const int64_t nc = cs->nc;
  const int d = cs->d;
  std::vector<int32_t> G(nc);
  std::vector<int64_t> cstart(nc + 1, 0), hstart(nc + 1, 0);
  for (int64_t c = 0; c < nc; ++c) {
    const double S = (double)(cs->ofs[c + 1] - cs->ofs[c]);
    int g = (int)std::lround(2.5 * std::cbrt(S));
    g = std::max(4, std::min(gmax, g));
    G[c] = g;
    const int64_t nl = (int64_t)g * g * (d == 3 ? g : 1);
    cstart[c + 1] = cstart[c] + nl;
    hstart[c + 1] = hstart[c] + cell_head_words(nl);
  }
  const int64_t ncell = cstart[nc];
  for (int64_t c = 0; c < nc; ++c)
    if ((cstart[c + 1] - cstart[c]) * (cs->ofs[c + 1] - cs->ofs[c]) >= INT32_MAX) {
      set_error("mrep_curveset_cells_build: a curve's lists could exceed int32 offsets; lower grid_max");
      return MREP_ERR_ARG;
    }
  if (ncell + nc + 1 > INT32_MAX) {
    set_error("mrep_curveset_cells_build: too many cells; lower grid_max");
    return MREP_ERR_ARG;
  }
  // scratch: grids, G, cstart, counts (int32) and their scan (int64, ncell + 1)
  auto al = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  const int64_t o_grid = 0, o_G = al(nc * (int64_t)sizeof(CellGrid)), o_cs = o_G + al(nc * 4);
  const int64_t o_hs = o_cs + al((nc + 1) * 8);
  const int64_t o_cnt = o_hs + al((nc + 1) * 8), o_E = o_cnt + al((ncell + 1) * 4);
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const int32_t*)nullptr, (int64_t*)nullptr,
                                (int)(ncell + 1), st);
  const int64_t o_tmp = o_E + al((ncell + 1) * 8), scratch = o_tmp + al((int64_t)scan_tmp + 16);
  char* ws = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&ws, scratch, st));
  CellGrid* grids = (CellGrid*)(ws + o_grid);
  int32_t* Gd = (int32_t*)(ws + o_G);
  int64_t* csd = (int64_t*)(ws + o_cs);
  int64_t* hsd = (int64_t*)(ws + o_hs);
  int32_t* cnt = (int32_t*)(ws + o_cnt);
  int64_t* E = (int64_t*)(ws + o_E);
  int rc = MREP_OK;
  auto fail = [&](int code) {
    cudaFreeAsync(ws, st);
    cudaStreamSynchronize(st);
    return code;
  };
  MREP_CUDA_CHECK(cudaMemcpyAsync(Gd, G.data(), nc * 4, cudaMemcpyHostToDevice, st));
  MREP_CUDA_CHECK(cudaMemcpyAsync(csd, cstart.data(), (nc + 1) * 8, cudaMemcpyHostToDevice, st));
  MREP_CUDA_CHECK(cudaMemcpyAsync(hsd, hstart.data(), (nc + 1) * 8, cudaMemcpyHostToDevice, st));
  MREP_CUDA_CHECK(cudaMemsetAsync(cnt + ncell, 0, 4, st));
  set_grid_kernel<<<grid_for(nc, 128), 128, 0, st>>>(cs->desc, Gd, nc, d, grids);
  set_cells_count_kernel<<<grid_for(ncell, 128), 128, 0, st>>>(cs->desc, grids, csd, nc, ncell, cnt);
  MREP_LAUNCH_CHECK();
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + o_tmp, scan_tmp, cnt, E, (int)(ncell + 1), st));
  int64_t total = 0;
  MREP_CUDA_CHECK(cudaMemcpyAsync(&total, E + ncell, 8, cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  // offsets are int32 but local to each curve's region (checked above: a
  // curve lists at most ncell_c * S_c entries), and the regions are
  // addressed with 64-bit word offsets: beyond that only the budget limits
  const int64_t words = hstart[nc] + 2 * total;
  if (4 * words > max_bytes) {
    set_error("mrep_curveset_cells_build: the index needs " + std::to_string(4 * words) +
              " bytes (budget " + std::to_string(max_bytes) + ")");
    return fail(MREP_ERR_ARG);
  }
  char* mem = nullptr;
  cudaError_t e = cudaMalloc(&mem, (size_t)(4 * words + 256));
  if (e != cudaSuccess) {
    set_error(std::string("mrep_curveset_cells_build: cudaMalloc: ") + cudaGetErrorString(e));
    return fail(MREP_ERR_CUDA);
  }
  set_cells_fill_kernel<<<grid_for(ncell, 128), 128, 0, st>>>(cs->desc, grids, csd, hsd, E, nc,
                                                             ncell, (int32_t*)mem);
  set_cells_header_kernel<<<grid_for(nc, 128), 128, 0, st>>>(cs->desc, grids, csd, hsd, E, nc,
                                                            (int32_t*)mem);
  if ((e = cudaGetLastError()) != cudaSuccess) {
    set_error(std::string("mrep_curveset_cells_build: launch: ") + cudaGetErrorString(e));
    rc = MREP_ERR_CUDA;
  }
  cudaFreeAsync(ws, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && !rc) {
    set_error(std::string("mrep_curveset_cells_build: ") + cudaGetErrorString(e));
    rc = MREP_ERR_CUDA;
  }
  if (rc) {
    cudaFree(mem);
    return rc;
  }
  // the headers now point at the new index: the old one (if any) can go
  if (cs->cells) cudaFree(cs->cells);
  cs->cells = mem;
  cs->cells_bytes = 4 * words;
  return MREP_OK;
}

static int project_batch_chunk(const CurveSet* cs, const double* queries, const int32_t* qcurve,
                               int64_t n, double clip_tol, int max_iter, unsigned flags,
                               double* out_t, double* out_foot, double* out_dist,
                               int64_t* out_cand, int32_t* out_seg, uint64_t* counters,
                               cudaStream_t st) {
  int prc = ensure_pool();
  if (prc) return prc;
  const int d = cs->d;
  ProjParams p{};
  p.q = queries;
  p.n = n;
  p.clip_tol = clip_tol;
  p.max_iter = max_iter;
  p.out_t = out_t;
  p.out_foot = out_foot;
  p.out_dist = out_dist;
  p.out_cand = out_cand;
  p.out_seg = out_seg;
  p.counters = counters;
  // a set with per-curve cell indices scans them (unless a walk is forced)
  static const bool no_set_cells = getenv("MREP_SET_NO_CELLS") != nullptr;
  // MREP_SET_SCAN=lane|group: the per-query cell scan by one lane or by an
  // 8-lane group (A/B)
  static const int set_scan_group = [] {
    const char* e = getenv("MREP_SET_SCAN");
    return (e && !strcmp(e, "group")) ? 1 : 0;
  }();
  bool set_cells = false;
  if (cs->cells && !no_set_cells && !(flags & (MREP_PACKET | MREP_PER_LANE | MREP_GROUP))) {
    if (set_scan_group) {
      flags |= MREP_GROUP;
      set_cells = true;
    } else {
      flags |= MREP_CELLS;
    }
  }
  const int tmode0 = trav_mode(flags, n, cs->S_total, cs->max_top);
  // Sparse batches (group walks, each query's work a function of the query
  // alone) are ordered by a counting sort on the curve's scheduler rank:
  // count per rank, scan, warp-aggregated scatter -- three light kernels
  // instead of Morton keys + a 64-bit radix sort.  Dense batches (packet
  // walks, where warp composition matters) keep the (rank, Morton) radix sort.
  static const bool radix_env = getenv("MREP_RADIX_SORT") != nullptr;
  const bool counting = (tmode0 == TRAV_GROUP || tmode0 == TRAV_CELLS) && !radix_env &&
                        n < ((int64_t)1 << 32);
  static const bool stage_env = getenv("MREP_STAGE") != nullptr;
  const bool staged = counting && stage_env && tmode0 == TRAV_GROUP;
  const int end_bit = 10 * d + cs->rank_bits;
  // curve rank + the top 12 Morton bits: a curve holds ~10^2 queries, so a
  // 16^3 cell grid already makes warps spatially coherent (fewer passes)
  static const int morton_bits = [] {
    const char* e = getenv("MREP_SORT_BITS_MULTI");
    return e ? atoi(e) : 12;
  }();
  const int begin_bit = (morton_bits > 0 && morton_bits < 10 * d) ? 10 * d - morton_bits : 0;
  size_t sort_tmp = 0;
  if (!counting)
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, begin_bit,
                                    end_bit, st);
  size_t o_k = 0, o_i = o_k + 16 * (size_t)n, o_tmp = o_i + 8 * (size_t)n + 256;
  const size_t o_plan = (o_tmp + sort_tmp + 256 + 255) & ~(size_t)255;
  const size_t plan_b = 4 * ((size_t)cs->nc + 1) * 4 + 256;
  char* ws = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&ws, o_plan + plan_b, st));
  uint32_t* rcnt = (uint32_t*)(ws + o_plan);
  uint32_t* cursor = rcnt + cs->nc + 1;
  uint32_t* qstart = cursor + cs->nc + 1;
  uint32_t* tstart = qstart + cs->nc + 1;
  uint64_t* k_in = (uint64_t*)(ws + o_k);
  uint64_t* k_out = k_in + n;
  uint32_t* i_in = (uint32_t*)(ws + o_i);
  uint32_t* i_out = i_in + n;
  const bool timing = (flags & MREP_TIMING) != 0;
  StageTimer sort_tm(timing, st);
  sort_tm.mark();
  if (counting) {
    MREP_CUDA_CHECK(cudaMemsetAsync(rcnt, 0, 2 * ((size_t)cs->nc + 1) * 4, st));
    rank_count_kernel<<<grid_for(n, 256), 256, 0, st>>>(qcurve, n, cs->rank, cs->nc, rcnt);
    MREP_LAUNCH_CHECK();
    stage_plan_kernel<<<1, 1024, 0, st>>>(rcnt, cs->nc, qstart, tstart);
    MREP_LAUNCH_CHECK();
    // k_in is unused on this path: the inverse permutation for the unpermute pass
    rank_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(qcurve, n, cs->rank, cs->nc, qstart,
                                                          cursor, i_out, (uint32_t*)k_in);
    p.inv = (const uint32_t*)k_in;
    MREP_LAUNCH_CHECK();
  } else {
    if (d == 3)
      morton_multi_kernel<3><<<grid_for(n, 256), 256, 0, st>>>(queries, qcurve, n, cs->desc,
                                                               cs->rank, cs->nc, end_bit, k_in, i_in,
                                                               nullptr);
    else
      morton_multi_kernel<2><<<grid_for(n, 256), 256, 0, st>>>(queries, qcurve, n, cs->desc,
                                                               cs->rank, cs->nc, end_bit, k_in, i_in,
                                                               nullptr);
    MREP_LAUNCH_CHECK();
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ws + o_tmp, sort_tmp, k_in, k_out, i_in, i_out,
                                                    (int)n, begin_bit, end_bit, st));
  }
  sort_tm.mark();
  sort_tm.finish(0);
  p.perm = i_out;
  const int tmode = tmode0;
  StagePlan plan{cs->order, qstart, tstart, cs->nc, nullptr, 0};
  const StagePlan* pl = staged ? &plan : nullptr;
  int rc = d == 3 ? launch_wave<3, true>(p, st, timing, tmode, cs->desc, qcurve, cs->nc, pl,
                                         set_cells)
                  : launch_wave<2, true>(p, st, timing, tmode, cs->desc, qcurve, cs->nc, pl,
                                         set_cells);
  MREP_CUDA_CHECK(cudaFreeAsync(ws, st));
  return rc;
}



}  // namespace mrep

using namespace mrep;

// ====================================================================== C ABI
extern "C" {

const char* mrep_last_error(void) { return g_last_error.c_str(); }
int mrep_last_stage_times(double* ms, int max) {
  int k = max < 8 ? max : 8;
  for (int i = 0; i < k; ++i) ms[i] = g_stage_ms[i];
  return k;
}
int mrep_version(void) { return 100; }
int mrep_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t mrep_table_bytes(int64_t S) {
  if (S < 1) return -1;
  return table_layout(S).total_doubles * (int64_t)sizeof(double);
}

int mrep_table_pack(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                    const double* seam_t, const double* seam_pt, int64_t S, int d, void* table,
                    void* stream) {
  if (S < 1 || (d != 2 && d != 3) || !table) {
    set_error("mrep_table_pack: need S >= 1, d in {2,3}");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  TableLayout L = table_layout(S);
  double* base = (double*)table;
  MREP_CUDA_CHECK(cudaMemsetAsync(base, 0, HDR * sizeof(double), st));
  double* box = base + L.box_off;
  pack_records_kernel<<<grid_for(S, 128), 128, 0, st>>>(seg_pts, seg_ta, seg_tb, seam_t, seam_pt,
                                                        S, d, base, base + L.rec_off,
                                                        box + L.lvl_off[0], base + L.sxyz_off);
  MREP_LAUNCH_CHECK();
  for (int lv = 1; lv <= L.top; ++lv) {
    reduce_boxes_kernel<<<grid_for(L.lvl_cnt[lv], 128), 128, 0, st>>>(
        box + L.lvl_off[lv - 1] * 6, L.lvl_cnt[lv - 1], box + L.lvl_off[lv] * 6, L.lvl_cnt[lv]);
    MREP_LAUNCH_CHECK();
  }
  boxes_to_float_kernel<<<grid_for(L.total_boxes, 256), 256, 0, st>>>(
      box, reinterpret_cast<float*>(base + L.fbox_off), L.total_boxes);
  MREP_LAUNCH_CHECK();
  table_bfrag_kernel<<<grid_for(S, 128), 128, 0, st>>>(table_view(table, S), d);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}


static int project_chunk(const void* table, int64_t S, int d, const double* queries, int64_t n,
                         double clip_tol, int max_iter, int soundness_samples, unsigned flags,
                         double* out_t, double* out_foot, double* out_dist, int64_t* out_cand,
                         int32_t* out_seg, int64_t* out_stats, double* out_sound,
                         uint64_t* counters, void* stream);

// Large batches run as independent chunks (workspace is ~0.5 KB per query),
// each with its own Morton sort; results do not depend on the chunking.
int mrep_project(const void* table, int64_t S, int d, const double* queries, int64_t n,
                 double clip_tol, int max_iter, int soundness_samples, unsigned flags,
                 double* out_t, double* out_foot, double* out_dist, int64_t* out_cand,
                 int32_t* out_seg, int64_t* out_stats, double* out_sound, uint64_t* counters,
                 void* stream) {
  static const int64_t CHUNK_Q = [] {
    const char* e = getenv("MREP_CHUNK_Q");  // A/B: queries per internal chunk
    const int64_t v = e ? atoll(e) : ((int64_t)1 << 23);
    return v < 4096 ? (int64_t)4096 : v;
  }();
  if (flags & MREP_TIMING)
    for (double& v : g_stage_ms) v = 0.0;
  if (n <= CHUNK_Q)
    return project_chunk(table, S, d, queries, n, clip_tol, max_iter, soundness_samples, flags,
                         out_t, out_foot, out_dist, out_cand, out_seg, out_stats, out_sound,
                         counters, stream);
  for (int64_t lo = 0; lo < n; lo += CHUNK_Q) {
    int64_t m = n - lo < CHUNK_Q ? n - lo : CHUNK_Q;
    int rc = project_chunk(table, S, d, queries + lo * d, m, clip_tol, max_iter,
                           soundness_samples, flags, out_t + lo, out_foot + lo * d, out_dist + lo,
                           out_cand ? out_cand + lo : nullptr, out_seg ? out_seg + lo : nullptr,
                           out_stats ? out_stats + lo * 6 : nullptr,
                           out_sound ? out_sound + lo : nullptr, counters, stream);
    if (rc != MREP_OK) return rc;
  }
  return MREP_OK;
}

static int project_chunk(const void* table, int64_t S, int d, const double* queries, int64_t n,
                         double clip_tol, int max_iter, int soundness_samples, unsigned flags,
                         double* out_t, double* out_foot, double* out_dist, int64_t* out_cand,
                         int32_t* out_seg, int64_t* out_stats, double* out_sound,
                         uint64_t* counters, void* stream) {
  if (S < 1 || (d != 2 && d != 3) || n < 0 || max_iter < 1 || !table) {
    set_error("mrep_project: bad arguments (S >= 1, d in {2,3}, max_iter >= 1)");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  if (!queries || !out_t || !out_foot || !out_dist) {
    set_error("mrep_project: null query/output pointer");
    return MREP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int prc = ensure_pool();
  if (prc) return prc;
  ProjParams p{};
  p.tab = table_view(table, S);
  p.q = queries;
  p.n = n;
  p.clip_tol = clip_tol;
  p.max_iter = max_iter;
  p.soundness = soundness_samples;
  p.out_t = out_t;
  p.out_foot = out_foot;
  p.out_dist = out_dist;
  p.out_cand = out_cand;
  p.out_seg = out_seg;
  p.out_stats = out_stats;
  p.out_sound = out_sound;
  p.counters = counters;
  // workspace: pass-2 list + Morton keys / permutation + sort scratch
  size_t sort_tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 30, st);
  // MREP_RADIX_SORT=1: the full 24-bit Morton radix sort instead of the
  // bucket sort (mrep_sort.cuh), for comparison
  // packet walks depend on which queries share a warp, so they keep the
  // stable radix order (deterministic warps, hence deterministic `cand`);
  // per-query walks (cells, lanes, groups) take the bucket order
  const int tmode = trav_mode(flags, n, S, table_view(table, S).top);
  const bool radix = getenv("MREP_RADIX_SORT") != nullptr || tmode == TRAV_PACKET;
  if (!radix) sort_tmp = bucket_sort_bytes(n, d);
  size_t off_list = 16, off_keys = off_list + sizeof(int64_t) * (size_t)n;
  size_t off_tmp = off_keys + 4 * sizeof(uint32_t) * (size_t)n;
  size_t wsb = off_tmp + sort_tmp + 256;
  void* ws = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync(&ws, wsb, st));
  char* wc = (char*)ws;
  p.pass2_count = (unsigned long long*)wc;
  p.pass2_list = (int64_t*)(wc + off_list);
  MREP_CUDA_CHECK(cudaMemsetAsync(ws, 0, 16, st));
  p.perm = nullptr;
  p.inv = nullptr;
  // sorted batches emit through sorted staging records and an unpermute
  // pass (MREP_UNPERM_MIN queries; default 2^16, i.e. whenever sorted):
  // cfg2 emit 0.094 -> 0.073 ms, cfg5 4.1 -> 1.4 ms per 2*10^7 queries
  static const int64_t unperm_min = [] {
    const char* e = getenv("MREP_UNPERM_MIN");
    return e ? (int64_t)atoll(e) : ((int64_t)1 << 16);
  }();
  const bool timing = (flags & MREP_TIMING) != 0;
  StageTimer sort_tm(timing, st);
  sort_tm.mark();
  // small batches skip the ordering: below 2^16 queries the sort's fixed
  // cost (~28 us) exceeds what coherence saves (measured 5-10% faster
  // unsorted at 2e3..3e4 queries, even with packet walks)
  if (!(flags & MREP_NO_SORT) && n >= ((int64_t)1 << 16)) {
    uint32_t* k_in = (uint32_t*)(wc + off_keys);
    uint32_t* k_out = k_in + n;
    uint32_t* i_in = k_out + n;
    uint32_t* i_out = i_in + n;
    const double* root = p.tab.box + p.tab.lvl_off[p.tab.top] * 6;
    if (!radix) {
      uint32_t* inv = n >= unperm_min ? k_in : nullptr;  // k_in is free on this path
      const int rc = bucket_sort(queries, n, d, root, wc + off_tmp, sort_tmp, i_out, st, inv);
      if (rc != MREP_OK) {
        cudaFreeAsync(ws, st);
        return rc;
      }
      p.inv = inv;
    } else {
    if (d == 3) morton_kernel<3><<<grid_for(n, 256), 256, 0, st>>>(queries, n, root, k_in, i_in);
    else morton_kernel<2><<<grid_for(n, 256), 256, 0, st>>>(queries, n, root, k_in, i_in);
    MREP_LAUNCH_CHECK();
    // the top 24 key bits (8 per axis) order the queries as well as all 30
    // do for warp coherence, with 3 radix passes instead of 4
    static const int sort_bits = [] {
      const char* e = getenv("MREP_SORT_BITS");
      return e ? atoi(e) : 24;
    }();
    const int end_bit = d * 10;
    const int begin_bit = (sort_bits > 0 && sort_bits < end_bit) ? end_bit - sort_bits : 0;
    MREP_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(wc + off_tmp, sort_tmp, k_in, k_out, i_in, i_out,
                                                    (int)n, begin_bit, end_bit, st));
    }
    p.perm = i_out;
  }
  sort_tm.mark();
  sort_tm.finish(0);
  int rc;
  bool wave = (flags & MREP_SCREEN) && !(flags & MREP_STATS) && !(flags & MREP_FUSED);
  if (wave)
    rc = d == 3 ? launch_wave<3, false>(p, st, timing, tmode)
                : launch_wave<2, false>(p, st, timing, tmode);
  else rc = d == 3 ? launch_project<3>(p, flags, st) : launch_project<2>(p, flags, st);
  if (rc == MREP_OK && wave && (flags & MREP_CAND_EXACT) && out_cand) {
    // the reference's brute-force candidate count (mrep_cand.cuh), caller order
    StageTimer cand_tm(timing, st);
    cand_tm.mark();
    const unsigned blocks = grid_for(n, CAND_WARPS * 8);
    unsigned long long* unc = counters ? (unsigned long long*)&counters[MREP_CNT_UNCERTAIN] : nullptr;
    static const bool cuda_cores = getenv("MREP_CAND_CUDA_CORES") != nullptr;
    if (flags & MREP_CAND_CELLS) {
      // the table's cand cell index (mrep_cand_cells_build), queries in the
      // pipeline's sorted order; undecided pairs solved by a second kernel
      unsigned long long gcap = (unsigned long long)std::max<int64_t>(16 * n, 1 << 16);
      if (const char* e = getenv("MREP_CAND_GCAP"))  // tests: force the redo pass
        gcap = std::min<unsigned long long>(gcap, (unsigned long long)std::max(1LL, atoll(e)));
      char* gws = nullptr;
      MREP_CUDA_CHECK(cudaMallocAsync((void**)&gws, 256 + gcap * sizeof(uint2) + n * 8, st));
      unsigned long long* gcount = (unsigned long long*)gws;
      unsigned long long* redo_n = gcount + 1;
      uint2* glist = (uint2*)(gws + 256);
      int64_t* redo = (int64_t*)(gws + 256 + gcap * sizeof(uint2));
      MREP_CUDA_CHECK(cudaMemsetAsync(gcount, 0, 16, st));
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (d == 3) {
        if (cuda_cores) cand_cells_kernel<3, false><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, p.perm, n, out_cand, unc, glist, gcount, gcap, redo, redo_n);
        else cand_cells_kernel<3, true><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, p.perm, n, out_cand, unc, glist, gcount, gcap, redo, redo_n);
        cand_solve_kernel<3><<<(unsigned)sms * 16u, 128, 0, st>>>(p.tab, queries, glist, gcount, gcap, out_cand);
        // rows whose undecided pairs overflowed the list: recounted whole
        cand_count_kernel<3, true><<<(unsigned)sms * 4u, CAND_WARPS * 32, 0, st>>>(p.tab, queries, 0, out_cand, nullptr, redo, redo_n);
      } else {
        if (cuda_cores) cand_cells_kernel<2, false><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, p.perm, n, out_cand, unc, glist, gcount, gcap, redo, redo_n);
        else cand_cells_kernel<2, true><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, p.perm, n, out_cand, unc, glist, gcount, gcap, redo, redo_n);
        cand_solve_kernel<2><<<(unsigned)sms * 16u, 128, 0, st>>>(p.tab, queries, glist, gcount, gcap, out_cand);
        cand_count_kernel<2, true><<<(unsigned)sms * 4u, CAND_WARPS * 32, 0, st>>>(p.tab, queries, 0, out_cand, nullptr, redo, redo_n);
      }
      MREP_LAUNCH_CHECK();
      MREP_CUDA_CHECK(cudaFreeAsync(gws, st));
    } else if (d == 3) {
      if (cuda_cores) cand_count_kernel<3, false><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, n, out_cand, unc);
      else cand_count_kernel<3, true><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, n, out_cand, unc);
    } else {
      if (cuda_cores) cand_count_kernel<2, false><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, n, out_cand, unc);
      else cand_count_kernel<2, true><<<blocks, CAND_WARPS * 32, 0, st>>>(p.tab, queries, n, out_cand, unc);
    }
    MREP_LAUNCH_CHECK();
    cand_tm.mark();
    cand_tm.finish(6);
  }
  MREP_CUDA_CHECK(cudaFreeAsync(ws, st));
  return rc;
}

int mrep_project_block(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                       const double* seam_t, const double* seam_pt, int64_t S, int d,
                       const double* queries, int64_t n, double clip_tol, int max_iter,
                       int soundness_samples, double* out_t, double* out_foot, double* out_dist,
                       int64_t* out_cand, int64_t* out_stats, double* out_sound, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t bytes = mrep_table_bytes(S);
  if (bytes < 0) {
    set_error("mrep_project_block: S must be >= 1");
    return MREP_ERR_ARG;
  }
  void* table = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync(&table, (size_t)bytes, st));
  int rc = mrep_table_pack(seg_pts, seg_ta, seg_tb, seam_t, seam_pt, S, d, table, stream);
  if (rc == MREP_OK)
    rc = mrep_project(table, S, d, queries, n, clip_tol, max_iter, soundness_samples, MREP_STATS,
                      out_t, out_foot, out_dist, out_cand, nullptr, out_stats, out_sound, nullptr,
                      stream);
  cudaFreeAsync(table, st);
  return rc;
}


// ---------------------------------------------------------------- curve sets
int mrep_curveset_create_dev(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                             const int64_t* seg_ofs_host, int64_t ncurves, int d, void* stream,
                             void** set_out) {
  if (!set_out) {
    set_error("mrep_curveset_create_dev: null handle pointer");
    return MREP_ERR_ARG;
  }
  CurveSet* cs = nullptr;
  int rc = set_create(seg_pts, seg_ta, seg_tb, seg_ofs_host, ncurves, d, (cudaStream_t)stream, &cs);
  *set_out = cs;
  return rc;
}

int mrep_curveset_create(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                         const int64_t* seg_ofs, int64_t ncurves, int d, void** set_out) {
  if (!set_out || !seg_ofs || ncurves < 1 || (d != 2 && d != 3)) {
    set_error("mrep_curveset_create: bad arguments");
    return MREP_ERR_ARG;
  }
  *set_out = nullptr;
  const int64_t S = seg_ofs[ncurves];
  if (S < 1) {
    set_error("mrep_curveset_create: no cubics");
    return MREP_ERR_ARG;
  }
  double *dp = nullptr, *da = nullptr, *db = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&dp, S * 4 * d * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&da, S * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&db, S * sizeof(double)));
  MREP_CUDA_CHECK(cudaMemcpy(dp, seg_pts, S * 4 * d * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(da, seg_ta, S * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(db, seg_tb, S * sizeof(double), cudaMemcpyHostToDevice));
  CurveSet* cs = nullptr;
  int rc = set_create(dp, da, db, seg_ofs, ncurves, d, nullptr, &cs);
  cudaFree(dp);
  cudaFree(da);
  cudaFree(db);
  *set_out = cs;
  return rc;
}

int mrep_curveset_free(void* set) {
  CurveSet* cs = (CurveSet*)set;
  if (!cs) return MREP_OK;
  cudaError_t e = cudaFree(cs->mem);
  if (cs->cells) {
    cudaError_t e2 = cudaFree(cs->cells);
    if (e == cudaSuccess) e = e2;
  }
  delete cs;
  if (e != cudaSuccess) {
    set_error(std::string("mrep_curveset_free: ") + cudaGetErrorString(e));
    return MREP_ERR_CUDA;
  }
  return MREP_OK;
}

int mrep_curveset_cells_build(void* set, int grid_max, int64_t max_bytes, int64_t* bytes_out,
                              void* stream) {
  CurveSet* cs = (CurveSet*)set;
  if (!cs) {
    set_error("mrep_curveset_cells_build: null set");
    return MREP_ERR_ARG;
  }
  int rc = set_cells_build(cs, grid_max, max_bytes, (cudaStream_t)stream);
  if (bytes_out) *bytes_out = cs->cells_bytes;
  return rc;
}

int mrep_curveset_info(const void* set, int64_t* ncurves, int64_t* total_cubics, int* d,
                       int64_t* device_bytes) {
  const CurveSet* cs = (const CurveSet*)set;
  if (!cs) {
    set_error("mrep_curveset_info: null set");
    return MREP_ERR_ARG;
  }
  if (ncurves) *ncurves = cs->nc;
  if (total_cubics) *total_cubics = cs->S_total;
  if (d) *d = cs->d;
  if (device_bytes) *device_bytes = cs->bytes;
  return MREP_OK;
}

int mrep_project_batch(const void* set, const double* queries, const int32_t* curve_ids, int64_t n,
                       double clip_tol, int max_iter, unsigned flags, double* out_t,
                       double* out_foot, double* out_dist, int64_t* out_cand, int32_t* out_seg,
                       uint64_t* counters, void* stream) {
  const CurveSet* cs = (const CurveSet*)set;
  if (!cs || n < 0 || max_iter < 1) {
    set_error("mrep_project_batch: bad arguments (set, n >= 0, max_iter >= 1)");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  if (!queries || !curve_ids || !out_t || !out_foot || !out_dist) {
    set_error("mrep_project_batch: null query/curve/output pointer");
    return MREP_ERR_ARG;
  }
  const int64_t CHUNK_Q = (int64_t)1 << 23;
  const int d = cs->d;
  if (flags & MREP_TIMING)
    for (double& v : g_stage_ms) v = 0.0;
  for (int64_t lo = 0; lo < n; lo += CHUNK_Q) {
    int64_t m = n - lo < CHUNK_Q ? n - lo : CHUNK_Q;
    int rc = project_batch_chunk(cs, queries + lo * d, curve_ids + lo, m, clip_tol, max_iter, flags,
                                 out_t + lo, out_foot + lo * d, out_dist + lo,
                                 out_cand ? out_cand + lo : nullptr,
                                 out_seg ? out_seg + lo : nullptr, counters, (cudaStream_t)stream);
    if (rc != MREP_OK) return rc;
  }
  return MREP_OK;
}


int64_t mrep_cells_bytes(const void* table, int64_t S, int d, int grid, void* stream) {
  return cells_bytes<CurveLeaves>(table, S, d, grid, REC, CurveLeaves{},
                                  (cudaStream_t)stream);
}

int mrep_cells_build(void* table, int64_t S, int d, int grid, void* cells, int64_t bytes,
                     void* stream) {
  return cells_build<CurveLeaves>(table, S, d, grid, REC, CurveLeaves{}, cells, bytes,
                                  (cudaStream_t)stream);
}

// cand cell index (mrep_cand.cuh): counts per cell, then offsets, fixed
// counts and lists; bytes = 4 (2 ncell + 1 + total)
static int cand_cells_plan(const void* table, int64_t S, int d, int grid, cudaStream_t st,
                           TableView& T, CellGrid& g, std::vector<int32_t>& cnt,
                           std::vector<int32_t>& fixed, int64_t& total) {
  int rc = cell_grid(table, S, d, grid, REC, st, T, g);
  if (rc != MREP_OK) return rc;
  int32_t* dc = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync((void**)&dc, g.ncell * 8, st));
  cand_cells_count_kernel<<<grid_for(g.ncell, 128), 128, 0, st>>>(T, g, dc, dc + g.ncell);
  cnt.resize(g.ncell);
  fixed.resize(g.ncell);
  cudaError_t e1 = cudaMemcpyAsync(cnt.data(), dc, g.ncell * 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaMemcpyAsync(fixed.data(), dc + g.ncell, g.ncell * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dc, st);
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    set_error("mrep_cand_cells: copy of the counts failed");
    return MREP_ERR_CUDA;
  }
  total = 0;
  for (int32_t v : cnt) total += v;
  if (total + 2 * g.ncell + 1 > INT32_MAX) {
    set_error("mrep_cand_cells: lists exceed 2^31 entries; use a smaller grid");
    return MREP_ERR_ARG;
  }
  return MREP_OK;
}

int64_t mrep_cand_cells_bytes(const void* table, int64_t S, int d, int grid, void* stream) {
  TableView T;
  CellGrid g;
  std::vector<int32_t> cnt, fixed;
  int64_t total = 0;
  if (cand_cells_plan(table, S, d, grid, (cudaStream_t)stream, T, g, cnt, fixed, total) != MREP_OK)
    return -1;
  return 4 * (2 * g.ncell + 1 + total);
}

int mrep_cand_cells_build(void* table, int64_t S, int d, int grid, void* buf, int64_t bytes,
                          void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TableView T;
  CellGrid g;
  std::vector<int32_t> cnt, fixed;
  int64_t total = 0;
  int rc = cand_cells_plan(table, S, d, grid, st, T, g, cnt, fixed, total);
  if (rc != MREP_OK) return rc;
  if (!buf || bytes < 4 * (2 * g.ncell + 1 + total)) {
    set_error("mrep_cand_cells_build: buffer too small (see mrep_cand_cells_bytes)");
    return MREP_ERR_ARG;
  }
  std::vector<int32_t> head(2 * g.ncell + 1);
  int64_t acc = 0;
  for (int64_t c = 0; c < g.ncell; ++c) {
    head[c] = (int32_t)acc;
    acc += cnt[c];
    head[g.ncell + 1 + c] = fixed[c];
  }
  head[g.ncell] = (int32_t)acc;
  int32_t* off = (int32_t*)buf;
  MREP_CUDA_CHECK(cudaMemcpyAsync(off, head.data(), head.size() * 4, cudaMemcpyHostToDevice, st));
  cand_cells_fill_kernel<<<grid_for(g.ncell, 128), 128, 0, st>>>(T, g, off, off + 2 * g.ncell + 1);
  MREP_LAUNCH_CHECK();
  double h[12];
  cells_header(g, buf, total, h);
  MREP_CUDA_CHECK(cudaMemcpyAsync((double*)table + H_CC, h, sizeof h, cudaMemcpyHostToDevice, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));  // head and h die here
  return MREP_OK;
}

int mrep_cand_cells_create(void* table, int64_t S, int d, int grid, void** buf_out) {
  if (!buf_out) {
    set_error("mrep_cand_cells_create: null output pointer");
    return MREP_ERR_ARG;
  }
  *buf_out = nullptr;
  const int64_t nb = mrep_cand_cells_bytes(table, S, d, grid, nullptr);
  if (nb <= 0) return MREP_ERR_ARG;
  void* buf = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&buf, (size_t)nb));
  const int rc = mrep_cand_cells_build(table, S, d, grid, buf, nb, nullptr);
  if (rc != MREP_OK) {
    cudaFree(buf);
    return rc;
  }
  *buf_out = buf;
  return MREP_OK;
}

int mrep_knot_span(const double* knots, int64_t m, int p, const double* t, int64_t n,
                   int32_t* span, void* stream) {
  if (n <= 0) return MREP_OK;
  knot_span_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(knots, m, p, t, n, span);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

int mrep_knot_span_batch(const double* knots, const int64_t* knot_ofs, const int32_t* degree,
                         const int32_t* curve_ids, const double* t, int64_t n, int32_t* span,
                         void* stream) {
  if (n <= 0) return MREP_OK;
  knot_span_batch_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      knots, knot_ofs, degree, curve_ids, t, n, span);
  MREP_LAUNCH_CHECK();
  return MREP_OK;
}

#define MREP_SIMPLE_LAUNCH(kern, n, ...)                                           \
  do {                                                                             \
    if ((n) <= 0) return MREP_OK;                                                  \
    kern<<<grid_for((n), 128), 128, 0, (cudaStream_t)stream>>>(__VA_ARGS__);       \
    MREP_LAUNCH_CHECK();                                                           \
    return MREP_OK;                                                                \
  } while (0)

int mrep_quartic_roots(const double* c, int64_t n, double* roots, int64_t* counts, void* stream) {
  MREP_SIMPLE_LAUNCH(quartic_kernel, n, c, n, roots, counts);
}
int mrep_newton_quartic_roots(const double* c, int64_t n, double* roots, int64_t* counts,
                              void* stream) {
  MREP_SIMPLE_LAUNCH(newton_quartic_kernel, n, c, n, roots, counts);
}
int mrep_distance_poly(const double* P, const double* q, int64_t n, int d, double* e,
                       void* stream) {
  if (d != 2 && d != 3) {
    set_error("mrep_distance_poly: d must be 2 or 3");
    return MREP_ERR_ARG;
  }
  MREP_SIMPLE_LAUNCH(distance_poly_kernel, n, P, q, n, d, e);
}
int mrep_restrict_ordinates(const double* b, const double* lo, const double* hi, int64_t n,
                            double* out, void* stream) {
  MREP_SIMPLE_LAUNCH(restrict_kernel, n, b, lo, hi, n, out);
}
int mrep_eval_ordinates(const double* b, const double* u, int64_t n, double* out, void* stream) {
  MREP_SIMPLE_LAUNCH(eval_ord_kernel, n, b, u, n, out);
}
int mrep_hull_cross(const double* b, int64_t n, int32_t* found, double* z, void* stream) {
  MREP_SIMPLE_LAUNCH(hull_kernel, n, b, n, found, z);
}
int mrep_clip_root(const double* b, int64_t n, double tol, int max_iter, double* root, int32_t* ok,
                   int32_t* used, double* widths, void* stream) {
  if (max_iter < 1) {
    set_error("mrep_clip_root: max_iter must be >= 1");
    return MREP_ERR_ARG;
  }
  MREP_SIMPLE_LAUNCH(clip_kernel, n, b, n, tol, max_iter, root, ok, used, widths);
}
int mrep_ordinates_op(int op, const double* b, int degree, int64_t n, const double* a,
                      const double* c, double tol, int max_iter, double* out, int32_t* i0,
                      int32_t* i1, double* widths, void* stream) {
  if (op < 0 || op > 3 || degree < 1 || degree >= ORD_NMAX || (op == 3 && max_iter < 1)) {
    set_error("mrep_ordinates_op: op in 0..3, 1 <= degree <= 31, max_iter >= 1");
    return MREP_ERR_ARG;
  }
  MREP_SIMPLE_LAUNCH(ordinates_gen_kernel, n, op, b, degree, n, a, c, tol, max_iter, out, i0, i1,
                     widths);
}
int mrep_cubic_points(const double* P, const double* u, int64_t n, int d, double* out,
                      void* stream) {
  MREP_SIMPLE_LAUNCH(cubic_points_kernel, n, P, u, n, d, out);
}
int mrep_rebase(const double* e, int64_t n, double* b, void* stream) {
  MREP_SIMPLE_LAUNCH(rebase_kernel, n, e, n, b);
}

}  // extern "C"
