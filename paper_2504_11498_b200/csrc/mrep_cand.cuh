// mrep_cand.cuh -- the reference's candidate count on FP64 tensor cores.
//
// _kernels._project_block (_kernels.py:369-502) reports per query
// cand = (S + 1) seams + every surviving monotone piece of EVERY cubic
// (pieces between the roots of E' in (1e-10, 1 - 1e-10); a piece survives
// iff its restricted ordinates have b0 < 0 and b0 * b5 <= 0,
// _kernels.py:427-441).  That is a brute-force quantity: the screened
// projection never looks at most cubics.  This pass reproduces it exactly
// without solving every pair:
//
//  * A cubic whose six Bernstein ordinates b_i of E = D' (D = |C - q|^2) are
//    all >= 0, or all < 0 and clear of underflow, has no survivor: every
//    piece's restricted ordinates are positively weighted sums of them, so
//    b0 >= 0, or b0 < 0 with b0 * b5 > 0 (the argument of prep_pair_cut).
//  * The degree-6 Bernstein coefficients d_j of D(u) = |C(u) - q|^2 are affine
//    in q: d_j = g_j - 2 (q - c0) . c_j + |q - c0|^2, with g_j, c_j the
//    coefficients of |C - c0|^2 and of C - c0 elevated to degree 6 (c0 = the
//    table's box centre), and b_i = 6 (d_{i+1} - d_i).  For 8 queries x one
//    cubic that is ONE FP64 tensor-core MMA, mma.sync m8n8k4 (K = 4 exactly:
//    1, qx, qy, qz; N = 8: d_0..d_6 and a pad column): A = the warp's 8
//    queries, B = the cubic's 4 x 8 fragment stored in the table.
//  * A cubic whose E' is strictly monotone (the five ordinates of E'' of one
//    sign: the reference's quartic finds no interior split) with end
//    values b_0, b_5 clear of zero holds exactly one survivor when
//    b_0 < 0 < b_5 and none otherwise.
//  The MMA is fed the coefficients of the ordinate differences directly
//  (column j -> d_{j+1} - d_j = b_j / 6), so a lane's two outputs are two
//  ordinates of E' and E'' needs one shuffle.
//  * The MMA's values differ from the reference's FP64 b_i by rounding only;
//    a margin of 1e-9 (scale + |q|)^2, orders of magnitude above the
//    rounding of either computation, decides the sign.  Pairs inside the
//    margin ("uncertain") are solved exactly as the reference does
//    (prep_pair: E, quartic roots of E', rebase, restriction per piece) by
//    the warp's lanes from a shared-memory queue, 32 at a time.
//
// Result: cand equal to the reference's, bit for bit, at a cost of one MMA
// per 8 (query, cubic) pairs plus the few uncertain pairs.
#pragma once

namespace mrep {

__device__ __forceinline__ void dmma_8x8x4(double a, double b, double& c0, double& c1) {
  const double z = 0.0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(c0), "=d"(c1)
               : "d"(a), "d"(b), "d"(z), "d"(z));
}

// B fragment of one cubic (control points P, centre c0).  With g_j, c_j the
// degree-6 Bernstein coefficients of |C - c0|^2 and of C - c0, column j
// (j = 0..5) holds the coefficients of d_{j+1} - d_j = b_j / 6:
//   k = 0: g_{j+1} - g_j;  k = 1..3: -2 (c_{j+1} - c_j)[k-1]
// (|q - c0|^2 cancels); columns 6, 7 are zero.  Element (k, j) is stored at
// index 4 j + k, the lane that holds it in m8n8k4's col-major B layout
// (lane t: k = t % 4, j = t / 4).
__device__ __forceinline__ void bfrag_one(const double (&P)[4][3], const double (&c0)[3], int d,
                                          double* frag) {
  const double C3[4] = {1.0, 3.0, 3.0, 1.0};
  const double C6[7] = {1.0, 6.0, 15.0, 20.0, 15.0, 6.0, 1.0};
  double Q[4][3];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) Q[i][k] = k < d ? P[i][k] - c0[k] : 0.0;
  // B_i,3 B_k,3 = C3[i] C3[k] / C6[i+k] B_{i+k},6: summing the product
  // weights gives |C - c0|^2 (g) and, since sum_k B_k,3 = 1, C - c0
  // elevated to degree 6 (c)
  double g[7], c[7][3];
  for (int j = 0; j < 7; ++j) {
    g[j] = 0.0;
    c[j][0] = c[j][1] = c[j][2] = 0.0;
    for (int i = 0; i < 4; ++i) {
      const int k2 = j - i;
      if (k2 >= 0 && k2 <= 3) {
        const double wgt = C3[i] * C3[k2] / C6[j];
        double dot = 0.0;
        for (int k = 0; k < 3; ++k) dot += Q[i][k] * Q[k2][k];
        g[j] += wgt * dot;
        for (int k = 0; k < 3; ++k) c[j][k] += wgt * Q[i][k];
      }
    }
  }
  for (int j = 0; j < 8; ++j) {
    if (j < 6) {
      frag[4 * j + 0] = g[j + 1] - g[j];
      for (int k = 0; k < 3; ++k) frag[4 * j + 1 + k] = -2.0 * (c[j + 1][k] - c[j][k]);
    } else {
      for (int k = 0; k < 4; ++k) frag[4 * j + k] = 0.0;
    }
  }
}

// the centre c0 of a curve table's root box
__device__ __forceinline__ void table_centre(const TableView& T, double (&c0)[3]) {
  const double* rb = T.box + T.lvl_off[T.top] * 6;
  for (int k = 0; k < 3; ++k) c0[k] = 0.5 * (rb[k] + rb[3 + k]);
}

__device__ __forceinline__ void bfrag_cubic(const TableView& T, int64_t s, int d) {
  double P[4][3], c0[3];
  const double* r = T.rec + s * REC + R_P;
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) P[i][k] = r[i * 3 + k];
  table_centre(T, c0);
  if (s == 0) {
    double* hdr = const_cast<double*>(T.hdr);
    for (int k = 0; k < 3; ++k) hdr[5 + k] = c0[k];
  }
  bfrag_one(P, c0, d, const_cast<double*>(T.bfrag) + s * 32);
}

// single table (after its boxes are built)
static __global__ void table_bfrag_kernel(const TableView T, int d) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < T.S) bfrag_cubic(T, s, d);
  if (s < 64) const_cast<double*>(T.bfrag)[T.S * 32 + s] = 0.0;  // prefetch slack
}

// kept pieces of one (query, cubic) pair, exactly as _kernels.py:415-441
template <int D>
__device__ __forceinline__ int kept_pieces(const TableView& T, int64_t s, const double (&q)[D]) {
  PairPrep P;
  prep_pair<D>(T, s, q, P);
  int kept = 0;
  double lo = 0.0;
  for (int k = 0; k <= P.nin; ++k) {
    const double hi = (k == P.nin) ? 1.0 : (k == 0 ? P.b1 : (k == 1 ? P.b2 : (k == 2 ? P.b3 : P.b4)));
    double bp[6];
    restrict_ordinates(P.bseg, lo, hi, bp);
    kept += (bp[0] < 0.0 && bp[0] * bp[5] <= 0.0) ? 1 : 0;
    lo = hi;
  }
  return kept;
}

constexpr int CAND_WARPS = 4;

// Sign margins of one query (or of a box of queries with |q| <= R): far above
// the rounding of the MMA and of the reference's FP64 ordinates; the end
// values of a monotone E' must clear a wider margin (a spurious split the
// reference's quartic might place within ~1e-8 of an end must not change
// that end's sign).
struct CandMargins {
  double m, m2, mend;
};
__device__ __forceinline__ CandMargins cand_margins(double R) {
  const double m = fmax(1e-9 * R * R, 1e-150);
  return CandMargins{m, 4.0 * m, fmax(1e-6 * R * R, 1e-150)};
}

// Per-warp state of the count: 8 query rows, the undecided-pair queue.
struct CandWarp {
  uint32_t* queue;     // [64] row << 29 | cubic
  int* kept;           // [8] exact survivors of undecided pairs, per row
  double (*sq)[3];     // [8] the rows' coordinates
  int qn;              // queued entries
  unsigned long long unc;
  // undecided pairs go to a global list solved by cand_solve_kernel (when
  // given; the local queue takes what does not fit)
  uint2* glist;                // (caller index, cubic)
  unsigned long long* gcount;
  unsigned long long gcap;
  const int64_t* rowq;         // [8] caller index of each row (shared)
  unsigned* redo_rows;         // (shared) rows with a pair that did not fit
};

// lanes < cnt solve one queued (row, cubic) pair each, as the reference does
template <int D>
__device__ __forceinline__ void cand_drain(const TableView& T, CandWarp& W, int cnt, int lane) {
  if (lane < cnt) {
    const uint32_t e = W.queue[lane];
    const int r = (int)(e >> 29);
    const int64_t s = (int64_t)(e & 0x1fffffffu);
    double qq[D];
#pragma unroll
    for (int k = 0; k < D; ++k) qq[k] = W.sq[r][k];
    const int kp = kept_pieces<D>(T, s, qq);
    if (kp) atomicAdd(&W.kept[r], kp);
  }
  __syncwarp();
}

// the first cnt entries of the warp's queue -> the global list (one atomic);
// a row whose pair does not fit is recounted from scratch afterwards (redo)
__device__ __forceinline__ void cand_flush(CandWarp& W, int cnt, int lane) {
  if (cnt <= 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(W.gcount, (unsigned long long)cnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < cnt) {
    const uint32_t e = W.queue[lane];
    const int r = (int)(e >> 29);
    if (base + lane < W.gcap) W.glist[base + lane] = make_uint2((uint32_t)W.rowq[r], e & 0x1fffffffu);
    else atomicOr(W.redo_rows, 1u << r);
  }
  __syncwarp();
}

// The 8 rows of a warp against the cubics idx(0..cnt-1): one MMA per cubic
// (8 queries x the cubic's 4x8 fragment), sign tests per row; rows outside
// `rows` (8-bit mask) are computed and ignored.  `ones` (lanes p == 0)
// counts pairs certified to hold exactly one survivor; undecided pairs are
// queued for cand_drain.
template <int D, bool TC, bool GLOBAL, class Idx>
__device__ __forceinline__ void cand_tile(const TableView& T, CandWarp& W, const Idx& idx,
                                          int64_t cnt, unsigned rows, double a,
                                          const CandMargins& M, int& ones, int lane) {
  const int row = lane >> 2, p = lane & 3;
  const double m = M.m, mneg = M.m, m2 = M.m2, mend = M.mend;
  // per-lane constant: flag bits this lane does not decide (AND-neutral)
  //  0 all b > m  1 all b < -m  2 all E'' > m2  3 all E'' < -m2
  //  4 b_0 < -mend  5 |b_0| > mend  (lane 0)   6 b_5 > mend  7 |b_5| > mend  (lane 2)
  const unsigned neutral = p == 0 ? 0xc0u : (p == 1 ? 0xf0u : (p == 2 ? 0x30u : 0xffu));
  const bool owner = p == 0 && ((rows >> row) & 1u);
  const double* F = T.bfrag;
  // fragments one cubic ahead, ids two ahead
  int64_t s_cur = cnt > 0 ? idx(0) : 0, s_nxt = cnt > 1 ? idx(1) : 0;
  double bn = __ldg(F + s_cur * 32 + lane);
#pragma unroll 1
  for (int64_t k = 0; k < cnt; ++k) {
    const double b = bn;
    const int64_t s = s_cur;
    s_cur = s_nxt;
    if (k + 1 < cnt) bn = __ldg(F + s_cur * 32 + lane);
    if (k + 2 < cnt) s_nxt = idx(k + 2);
    double c0, c1;
    if (TC) {
      dmma_8x8x4(a, b, c0, c1);
    } else {
      // lane (row, p) owns columns 2p, 2p+1: sum_k A[row][k] B[k][col]
      const double* Bs = F + s * 32;
      c0 = c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const double ak = __shfl_sync(0xffffffffu, a, (lane & ~3) | kk);
        c0 = fma(ak, __ldg(Bs + 8 * p + kk), c0);
        c1 = fma(ak, __ldg(Bs + 8 * p + 4 + kk), c1);
      }
    }
    // lane p holds b_2p / 6, b_2p+1 / 6 of its row (lanes p = 0..2; p = 3
    // holds the zero pad columns); b_2p+2 / 6 from lane p + 1.
    // Fast path: most tested pairs are one-signed for every row of the tile
    // (no survivor) -- two compares per column, an AND over the row's lanes.
    {
      unsigned z = p == 3 ? 3u
                          : ((unsigned)(c0 > m && c1 > m) | ((unsigned)(c0 < -mneg && c1 < -mneg) << 1));
      z &= __shfl_xor_sync(0xffffffffu, z, 1);
      z &= __shfl_xor_sync(0xffffffffu, z, 2);
      if (__all_sync(0xffffffffu, z != 0 || !((rows >> row) & 1u))) continue;
    }
    const double nx = __shfl_down_sync(0xffffffffu, c0, 1);
    const double ea = c1 - c0, eb = nx - c1;  // E'' ordinates / 30: 2p, 2p + 1
    const double mn = fmin(c0, c1), mx = fmax(c0, c1);
    const double emn = p <= 1 ? fmin(ea, eb) : ea, emx = p <= 1 ? fmax(ea, eb) : ea;
    unsigned v = (unsigned)(mn > m) | ((unsigned)(mx < -mneg) << 1) | ((unsigned)(emn > m2) << 2) |
                 ((unsigned)(emx < -m2) << 3) | ((unsigned)(c0 < -mend) << 4) |
                 ((unsigned)(fabs(c0) > mend) << 5) | ((unsigned)(c1 > mend) << 6) |
                 ((unsigned)(fabs(c1) > mend) << 7);
    v |= neutral;
    v &= __shfl_xor_sync(0xffffffffu, v, 1);
    v &= __shfl_xor_sync(0xffffffffu, v, 2);
    // E' one-signed: no survivor.  E' strictly monotone (E'' one-signed, so
    // the reference splits no piece) with robust end values: one survivor
    // iff it rises from b_0 < 0 to b_5 > 0.
    const bool zero = (v & 3u) != 0;
    const bool mono = (v & 12u) && (v & 0xa0u) == 0xa0u;
    ones += (owner && !zero && mono && (v & 0x50u) == 0x50u) ? 1 : 0;
    const bool unc = owner && !zero && !mono;
    const unsigned bal = __ballot_sync(0xffffffffu, unc);
    if (GLOBAL) {
      // to the global list (cand_solve_kernel) in batches of 32 through the
      // warp's shared queue: one atomic per batch on the list counter
      if (bal) {
        if (unc) W.queue[W.qn + __popc(bal & ((1u << lane) - 1))] = ((uint32_t)row << 29) | (uint32_t)s;
        W.qn += __popc(bal);
        W.unc += __popc(bal);
        __syncwarp();
        if (W.qn >= 32) {
          cand_flush(W, 32, lane);
          if (lane < W.qn - 32) W.queue[lane] = W.queue[32 + lane];
          W.qn -= 32;
          __syncwarp();
        }
      }
      continue;
    }
    if (bal) {
      if (unc) W.queue[W.qn + __popc(bal & ((1u << lane) - 1))] = ((uint32_t)row << 29) | (uint32_t)s;
      W.qn += __popc(bal);
      W.unc += __popc(bal);
      __syncwarp();
      if (W.qn >= 32) {
        cand_drain<D>(T, W, 32, lane);
        if (lane < W.qn - 32) W.queue[lane] = W.queue[32 + lane];
        W.qn -= 32;
        __syncwarp();
      }
    }
  }
}

// one warp = 8 queries (rows) against every cubic; out_cand in caller order.
// TC = false computes the same two columns per lane with DFMA on the CUDA
// cores (8 fragment loads + 8 FMAs instead of one MMA) -- the A/B baseline
// for the tensor-core contraction (MREP_CAND_CUDA_CORES=1 selects it).
struct CandAll {
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return k; }
};
struct CandList {
  const int32_t* ids;
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return __ldg(ids + k); }
};

// list / list_n (device count): the redo pass of cand_cells_kernel -- the
// warp's rows are list entries (grid-stride over tiles of 8), not 0..n-1
template <int D, bool TC = true>
__global__ void __launch_bounds__(CAND_WARPS * 32) cand_count_kernel(const TableView T, const double* qs,
                                                                    int64_t n, int64_t* out_cand,
                                                                    unsigned long long* n_uncertain,
                                                                    const int64_t* list = nullptr,
                                                                    const unsigned long long* list_n = nullptr) {
  __shared__ uint32_t queue[CAND_WARPS][64];
  __shared__ int kept[CAND_WARPS][8];
  __shared__ double sq[CAND_WARPS][8][3];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31, row = lane >> 2, p = lane & 3;
  if (list) n = (int64_t)*list_n;
  for (int64_t q0 = ((int64_t)blockIdx.x * CAND_WARPS + wi) * 8; q0 < n;
       q0 += (int64_t)gridDim.x * CAND_WARPS * 8) {
  const int64_t qi0 = q0 + row;
  const bool valid = qi0 < n;
  const int64_t qi = valid && list ? list[qi0] : qi0;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = valid ? qs[qi * D + k] : 0.0;
  if (p == 0) {
    kept[wi][row] = 0;
    for (int k = 0; k < 3; ++k) sq[wi][row][k] = k < D ? q[k] : 0.0;
  }
  double R = T.hdr[4];
#pragma unroll
  for (int k = 0; k < D; ++k) R = fmax(R, fabs(q[k]));
  const CandMargins M = cand_margins(R);
  const double a = p == 0 ? 1.0 : (p <= D ? q[p - 1] - T.hdr[4 + p] : 0.0);
  const unsigned rows = __ballot_sync(0xffffffffu, valid && p == 0);
  unsigned rmask = 0;
  for (int r = 0; r < 8; ++r) rmask |= ((rows >> (4 * r)) & 1u) << r;
  CandWarp W{queue[wi], kept[wi], sq[wi], 0, 0, nullptr, nullptr, 0, nullptr, nullptr};
  int ones = 0;
  __syncwarp();
  cand_tile<D, TC, false>(T, W, CandAll{}, T.S, rmask, a, M, ones, lane);
  cand_drain<D>(T, W, W.qn, lane);
  if (valid && p == 0) out_cand[qi] = T.S + 1 + W.kept[row] + ones;
  if (n_uncertain && lane == 0) atomicAdd(n_uncertain, W.unc);
  __syncwarp();
  }
}

// ---------------------------------------------------------------- cand cells
// A uniform grid over the table's root box (+10% each side, as the cell
// index) where every cell C stores
//   fixed[C] = the number of cubics certified, for EVERY query of C, to hold
//              exactly one survivor, and
//   list[C]  = the cubics whose count is NOT fixed over C,
// every other cubic being certified to hold none.  The b_j (and the E''
// differences) are affine in q, so their exact range over the cell box is
// centre value +- sum |coefficient| * half-width; the certification tests
// of cand_tile are applied to those ranges with the margins of the largest
// |q| in the cell (a larger margin than any of its queries uses, so a
// certified cubic is certified for each of them; the margin is far above the
// rounding of the range computation).  A query then runs cand_tile over its
// cell's list only and adds fixed[C].  Queries outside the grid use every
// cubic.  Results equal cand_count_kernel's (and the reference's) exactly.
constexpr int H_CC = 24, H_CC_GRID = 25, H_CC_GLO = 26, H_CC_GINV = 29, H_CC_GHI = 32,
              H_CC_TOT = 35;

// class of cubic s over the query box [lo, hi]: 0 or 1 certified, -1 not fixed
__device__ __forceinline__ int cand_box_class(const TableView& T, int64_t s, const double* lo,
                                              const double* hi, int d) {
  const double* F = T.bfrag + s * 32;  // element (k, j) at 4 j + k
  double ctr[3], half[3], R = T.hdr[4];
  for (int k = 0; k < 3; ++k) {
    ctr[k] = k < d ? 0.5 * (lo[k] + hi[k]) - T.hdr[5 + k] : 0.0;
    half[k] = k < d ? 0.5 * (hi[k] - lo[k]) : 0.0;
    if (k < d) R = fmax(R, fmax(fabs(lo[k]), fabs(hi[k])));
  }
  const CandMargins M = cand_margins(R);
  double mn[6], mx[6];
  for (int j = 0; j < 6; ++j) {
    double v = F[4 * j], r = 0.0;
    for (int k = 0; k < 3; ++k) {
      v += F[4 * j + 1 + k] * ctr[k];
      r += fabs(F[4 * j + 1 + k]) * half[k];
    }
    mn[j] = v - r;
    mx[j] = v + r;
  }
  bool pos = true, neg = true;
  for (int j = 0; j < 6; ++j) {
    pos = pos && mn[j] > M.m;
    neg = neg && mx[j] < -M.m;
  }
  if (pos || neg) return 0;
  bool epos = true, eneg = true;
  for (int j = 0; j < 5; ++j) {
    double v = F[4 * (j + 1)] - F[4 * j], r = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double c = F[4 * (j + 1) + 1 + k] - F[4 * j + 1 + k];
      v += c * ctr[k];
      r += fabs(c) * half[k];
    }
    epos = epos && v - r > M.m2;
    eneg = eneg && v + r < -M.m2;
  }
  const bool e0 = mn[0] > M.mend || mx[0] < -M.mend, e5 = mn[5] > M.mend || mx[5] < -M.mend;
  if ((epos || eneg) && e0 && e5) return (mx[0] < -M.mend && mn[5] > M.mend) ? 1 : 0;
  return -1;
}

// one thread per cell: list length and the fixed count
__global__ void cand_cells_count_kernel(const __grid_constant__ TableView T,
                                        const __grid_constant__ CellGrid g, int32_t* cnt,
                                        int32_t* fixed) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.ncell) return;
  double lo[3], hi[3];
  cell_box(g, c, lo, hi);
  int32_t nl = 0, nf = 0;
  for (int64_t s = 0; s < T.S; ++s) {
    const int cl = cand_box_class(T, s, lo, hi, g.d);
    nl += cl < 0 ? 1 : 0;
    nf += cl > 0 ? 1 : 0;
  }
  cnt[c] = nl;
  fixed[c] = nf;
}

__global__ void cand_cells_fill_kernel(const __grid_constant__ TableView T,
                                       const __grid_constant__ CellGrid g, const int32_t* off,
                                       int32_t* ids) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.ncell) return;
  double lo[3], hi[3];
  cell_box(g, c, lo, hi);
  int32_t* out = ids + off[c];
  int32_t nl = 0;
  for (int64_t s = 0; s < T.S; ++s)
    if (cand_box_class(T, s, lo, hi, g.d) < 0) out[nl++] = (int32_t)s;
}

// the query's cand cell (-1: no index or outside the grid)
template <int D>
__device__ __forceinline__ int64_t cand_cell_of(const TableView& T, const double (&q)[D]) {
  const int G = (int)T.hdr[H_CC_GRID];
  if (G <= 0) return -1;
  int64_t ci[3] = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (!(q[k] >= T.hdr[H_CC_GLO + k] && q[k] < T.hdr[H_CC_GHI + k])) return -1;
    const int64_t c = (int64_t)((q[k] - T.hdr[H_CC_GLO + k]) * T.hdr[H_CC_GINV + k]);
    ci[k] = c < 0 ? 0 : (c >= G ? G - 1 : c);
  }
  return (ci[0] * G + ci[1]) * (D == 3 ? G : 1) + (D == 3 ? ci[2] : 0);
}

// one warp = 8 consecutive SORTED queries (perm: sorted -> caller; null =
// caller order).  The rows are grouped by cand cell (Morton-sorted
// neighbours share one or two cells): each group runs cand_tile over its
// cell's list (every cubic for rows outside the grid).
template <int D, bool TC = true>
__global__ void __launch_bounds__(CAND_WARPS * 32) cand_cells_kernel(const TableView T, const double* qs,
                                                                    const uint32_t* perm, int64_t n,
                                                                    int64_t* out_cand,
                                                                    unsigned long long* n_uncertain,
                                                                    uint2* glist,
                                                                    unsigned long long* gcount,
                                                                    unsigned long long gcap,
                                                                    int64_t* redo_list,
                                                                    unsigned long long* redo_n) {
  __shared__ int64_t rowq[CAND_WARPS][8];
  __shared__ uint32_t queue[CAND_WARPS][64];
  __shared__ unsigned redo_rows[CAND_WARPS];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31, row = lane >> 2, p = lane & 3;
  const int64_t g0 = ((int64_t)blockIdx.x * CAND_WARPS + wi) * 8;
  if (g0 >= n) return;  // whole warp
  const int64_t g = g0 + row;
  const bool valid = g < n;
  const int64_t qi = valid ? (perm ? (int64_t)perm[g] : g) : 0;
  double q[D];
#pragma unroll
  for (int k = 0; k < D; ++k) q[k] = valid ? qs[qi * D + k] : 0.0;
  if (p == 0) rowq[wi][row] = qi;
  if (lane == 0) redo_rows[wi] = 0u;
  double R = T.hdr[4];
#pragma unroll
  for (int k = 0; k < D; ++k) R = fmax(R, fabs(q[k]));
  const CandMargins M = cand_margins(R);
  const double a = p == 0 ? 1.0 : (p <= D ? q[p - 1] - T.hdr[4 + p] : 0.0);
  const int64_t cell = valid ? cand_cell_of<D>(T, q) : -2;
  const int G = (int)T.hdr[H_CC_GRID];
  const int64_t ncell = (int64_t)G * G * (D == 3 ? G : 1);
  const int32_t* off = reinterpret_cast<const int32_t*>(
      (uintptr_t)__double_as_longlong(T.hdr[H_CC]));
  const int32_t* fixed = off + ncell + 1;
  const int32_t* ids = fixed + ncell;
  CandWarp W{queue[wi], nullptr, nullptr, 0, 0, glist, gcount, gcap, rowq[wi], &redo_rows[wi]};
  int ones = 0;
  __syncwarp();
  // rows still to do (8-bit, warp-uniform); invalid rows are done
  unsigned todo = 0;
  {
    const unsigned vb = __ballot_sync(0xffffffffu, valid && p == 0);
    for (int r = 0; r < 8; ++r) todo |= ((vb >> (4 * r)) & 1u) << r;
  }
  while (todo) {
    const int lead = __ffs(todo) - 1;
    const int64_t lc = __shfl_sync(0xffffffffu, cell, 4 * lead);
    const unsigned same = __ballot_sync(0xffffffffu, p == 0 && valid && cell == lc);
    unsigned rows = 0;
    for (int r = 0; r < 8; ++r) rows |= ((same >> (4 * r)) & 1u) << r;
    rows &= todo;
    if (lc >= 0) {
      const int32_t a0 = __ldg(off + lc), a1 = __ldg(off + lc + 1);
      cand_tile<D, TC, true>(T, W, CandList{ids + a0}, a1 - a0, rows, a, M, ones, lane);
    } else {
      cand_tile<D, TC, true>(T, W, CandAll{}, T.S, rows, a, M, ones, lane);
    }
    todo &= ~rows;
  }
  cand_flush(W, W.qn, lane);
  // cand_solve_kernel adds the undecided pairs' survivors afterwards
  if (valid && p == 0) {
    out_cand[qi] = T.S + 1 + ones + (cell >= 0 ? __ldg(fixed + cell) : 0);
    if ((redo_rows[wi] >> row) & 1u) redo_list[atomicAdd(redo_n, 1ull)] = qi;
  }
  if (n_uncertain && lane == 0) atomicAdd(n_uncertain, W.unc);
}

// the undecided pairs of cand_cells_kernel, one thread each, solved as the
// reference does (kept_pieces); adds to the query's count in caller order
template <int D>
__global__ void __launch_bounds__(128) cand_solve_kernel(const TableView T, const double* qs,
                                                         const uint2* glist,
                                                         const unsigned long long* gcount,
                                                         unsigned long long gcap, int64_t* out_cand) {
  unsigned long long total = *gcount;
  if (total > gcap) total = gcap;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint2 e = glist[i];
    double q[D];
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = qs[(int64_t)e.x * D + k];
    const int kp = kept_pieces<D>(T, (int64_t)e.y, q);
    if (kp) atomicAdd((unsigned long long*)&out_cand[e.x], (unsigned long long)kp);
  }
}

}  // namespace mrep
