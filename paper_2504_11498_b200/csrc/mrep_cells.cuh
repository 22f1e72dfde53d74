// mrep_cells.cuh -- cell index of a table (curve or surface): a uniform grid
// over the table's root box (+10% each side).  For every cell C the list
// holds each leaf s (cubic / patch) with
//   boxdist(C', box_s)^2 <= cut2(UB_C, scale_C),
//   UB_C = min over the table's exact points (curve seams / patch seed-grid
//          points) of the farthest distance from C' to the point,
// where C' is C grown by a rounding allowance.  Any query q in C has such a
// point within UB_C, so dmin(q) <= UB_C, and a leaf that can hold a candidate
// inside dmin(q) + 1e-12 has boxdist(q, box_s) <= cut(dmin(q)): it is in the
// list, so the cell scan replaces the tree walk exactly.
//
// The leaf-point policy LP supplies the exact points each leaf carries (all
// inside the leaf's box): npts(T) and pt(T, d, s, k, out).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "mrep_common.cuh"
#include "mrep_screen.cuh"

namespace mrep {

// header slots of a table holding a cell index
constexpr int H_CELLS = 8, H_GRID = 9, H_GLO = 10, H_GINV = 13, H_GHI = 16, H_CTOT = 19;

struct CellGrid {
  int G, d;
  double glo[3], h[3];
  double eps;     // growth of every cell box (rounding of the cell mapping)
  double hscale;  // table coordinate scale
  int64_t ncell;
};

__device__ __forceinline__ void cell_box(const CellGrid& g, int64_t c, double* lo, double* hi) {
  int64_t ci[3];
  if (g.d == 3) {
    ci[2] = c % g.G;
    ci[1] = (c / g.G) % g.G;
    ci[0] = c / ((int64_t)g.G * g.G);
  } else {
    ci[1] = c % g.G;
    ci[0] = c / g.G;
    ci[2] = 0;
  }
  for (int k = 0; k < 3; ++k) {
    if (k < g.d) {
      lo[k] = g.glo[k] + (double)ci[k] * g.h[k] - g.eps;
      hi[k] = g.glo[k] + (double)(ci[k] + 1) * g.h[k] + g.eps;
    } else {
      lo[k] = hi[k] = 0.0;
    }
  }
}

// farthest distance^2 from the (grown) cell to a point
__device__ __forceinline__ double far2(int d, const double* lo, const double* hi, const double* pt) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double f = fmax(fabs(pt[k] - lo[k]), fabs(pt[k] - hi[k]));
    acc += f * f;
  }
  return acc;
}

__device__ __forceinline__ double cellbox_lb2(const TableView& T, int d, int64_t box, const double* lo,
                                              const double* hi) {
  const double* b = T.box + box * 6;
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double gk = fmax(0.0, fmax(b[k] - hi[k], lo[k] - b[3 + k]));
    acc += gk * gk;
  }
  return acc;
}

template <class LP>
__device__ __forceinline__ void leaf_far2(const TableView& T, const LP& lp, int d, int64_t s,
                                          const double* lo, const double* hi, double& ub2) {
  double pt[3];
  const int np = lp.npts(T);
  for (int k = 0; k < np; ++k) {
    lp.pt(T, d, s, k, pt);
    ub2 = fmin(ub2, far2(d, lo, hi, pt));
  }
}

// cut radius^2 of a cell: brute force over all leaves for small tables,
// branch and bound over the hierarchy otherwise (a box's points p satisfy
// far2(cell, p) >= sum_k f_k^2, f_k the farther cell face from
// clamp(centre_k, box_k))
template <class LP>
__device__ double cell_cut2(const TableView& T, const LP& lp, const CellGrid& g, const double* lo,
                            const double* hi) {
  double ub2 = __longlong_as_double(0x7ff0000000000000LL);
  if (T.S <= 4096) {
    for (int64_t s = 0; s < T.S; ++s) leaf_far2(T, lp, g.d, s, lo, hi, ub2);
  } else {
    double ctr[3];
    for (int k = 0; k < 3; ++k) ctr[k] = 0.5 * (lo[k] + hi[k]);
    auto node_lb = [&](int64_t box) {
      const double* b = T.box + box * 6;
      double acc = 0.0;
      for (int k = 0; k < g.d; ++k) {
        double x = fmin(fmax(ctr[k], b[k]), b[3 + k]);
        double f = fmax(fabs(x - lo[k]), fabs(x - hi[k]));
        acc += f * f;
      }
      return acc;
    };
    int level = T.top;
    int64_t idx = 0;
    while (level > 0) {  // greedy descent first: a good initial bound
      int64_t first = idx * FANOUT, cnt = T.lvl_cnt[level - 1], off = T.lvl_off[level - 1];
      double best = 0.0;
      int64_t bi = first;
      for (int c = 0; c < FANOUT && first + c < cnt; ++c) {
        double lb = node_lb(off + first + c);
        if (c == 0 || lb < best) {
          best = lb;
          bi = first + c;
        }
      }
      idx = bi;
      --level;
    }
    leaf_far2(T, lp, g.d, idx, lo, hi, ub2);
    level = T.top;
    idx = 0;
    auto cmask = [&](int lv, int64_t node) {
      uint32_t m = 0;
      int64_t first = node * FANOUT, cnt = T.lvl_cnt[lv - 1], off = T.lvl_off[lv - 1];
      for (int c = 0; c < FANOUT && first + c < cnt; ++c)
        if (node_lb(off + first + c) < ub2) m |= 1u << c;
      return m;
    };
    uint64_t masks = (uint64_t)cmask(level, 0) << (8 * level);
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
      if (level == 1) {
        if (node_lb(T.lvl_off[0] + ch) < ub2) leaf_far2(T, lp, g.d, ch, lo, hi, ub2);
      } else if (node_lb(T.lvl_off[level - 1] + ch) < ub2) {
        --level;
        idx = ch;
        masks |= (uint64_t)cmask(level, idx) << (8 * level);
      }
    }
  }
  double scale = g.hscale;
  for (int k = 0; k < g.d; ++k) scale = fmax(scale, fmax(fabs(lo[k]), fabs(hi[k])));
  return cut2(sqrt(ub2) * (1.0 + 1e-12), scale);
}

// every leaf whose box is within the cut of the cell: brute force for small
// tables, a depth-first walk of the 8-ary hierarchy otherwise
template <class F>
__device__ void cell_leaves(const TableView& T, const CellGrid& g, const double* lo,
                            const double* hi, double c2, F&& f) {
  if (T.S <= 4096) {
    for (int64_t s = 0; s < T.S; ++s)
      if (cellbox_lb2(T, g.d, T.lvl_off[0] + s, lo, hi) <= c2) f(s);
    return;
  }
  int level = T.top;
  int64_t idx = 0;
  auto cmask = [&](int lv, int64_t node) {
    uint32_t m = 0;
    int64_t first = node * FANOUT, cnt = T.lvl_cnt[lv - 1], off = T.lvl_off[lv - 1];
    for (int c = 0; c < FANOUT && first + c < cnt; ++c)
      if (cellbox_lb2(T, g.d, off + first + c, lo, hi) <= c2) m |= 1u << c;
    return m;
  };
  uint64_t masks = (uint64_t)cmask(level, 0) << (8 * level);
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
    if (level == 1) {
      f(ch);
    } else {
      --level;
      idx = ch;
      masks |= (uint64_t)cmask(level, idx) << (8 * level);
    }
  }
}

template <class LP>
__device__ int32_t cell_count(const TableView& T, const LP& lp, const CellGrid& g, int64_t c) {
  double lo[3], hi[3];
  cell_box(g, c, lo, hi);
  const double c2 = cell_cut2(T, lp, g, lo, hi);
  int32_t n = 0;
  cell_leaves(T, g, lo, hi, c2, [&](int64_t) { ++n; });
  return n;
}

template <class LP>
__global__ void cells_count_kernel(const __grid_constant__ TableView T, const LP lp,
                                   const __grid_constant__ CellGrid g, int32_t* cnt) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.ncell) return;
  cnt[c] = cell_count(T, lp, g, c);
}

// A list entry: the sort key and the leaf id side by side (one 8-B load
// gives a scan both, and a list is one contiguous stream).
struct alignas(8) CellEntry {
  float key;
  int32_t id;
};
// int32 words before the entries: the ncell + 1 offsets, padded to even so
// the entries are 8-B aligned
__host__ __device__ inline int64_t cell_head_words(int64_t ncell) { return (ncell + 2) & ~(int64_t)1; }

// fill one cell's list (keys + ids) in the order the scan expects
template <class LP>
__device__ void cell_fill_list(const TableView& T, const LP& lp, const CellGrid& g, int64_t c,
                               CellEntry* E) {
  double lo[3], hi[3];
  cell_box(g, c, lo, hi);
  const double c2 = cell_cut2(T, lp, g, lo, hi);
  int32_t n = 0;
  cell_leaves(T, g, lo, hi, c2, [&](int64_t s) { E[n++].id = (int32_t)s; });
  // key = distance^2 from the (grown) cell to the leaf box, rounded down: a
  // lower bound of box_lb2(q, box) for every query q of the cell.  Sorted
  // ascending (ties by leaf id), the scan of a query can stop at the first
  // key above its cut: every later leaf fails the box test too.
  for (int32_t i = 0; i < n; ++i)
    E[i].key = __double2float_rd(cellbox_lb2(T, g.d, T.lvl_off[0] + E[i].id, lo, hi));
  // equal keys (typically 0: boxes meeting the cell) go nearest to the cell
  // centre first, so the running bound tightens early; then by leaf id
  double ctr[3];
  for (int k = 0; k < 3; ++k) ctr[k] = 0.5 * (lo[k] + hi[k]);
  auto after = [&](float ka, int32_t va, float kb, int32_t vb) {  // (ka, va) sorts after (kb, vb)
    if (ka != kb) return ka > kb;
    const double da = cellbox_lb2(T, g.d, T.lvl_off[0] + va, ctr, ctr);
    const double db = cellbox_lb2(T, g.d, T.lvl_off[0] + vb, ctr, ctr);
    return da != db ? da > db : va > vb;
  };
  int32_t gap = 1;
  while (gap < n / 3) gap = 3 * gap + 1;
  for (; gap > 0; gap /= 3) {  // shell sort
    for (int32_t i = gap; i < n; ++i) {
      const CellEntry ev = E[i];
      int32_t j = i;
      while (j >= gap && after(E[j - gap].key, E[j - gap].id, ev.key, ev.id)) {
        E[j] = E[j - gap];
        j -= gap;
      }
      E[j] = ev;
    }
  }
}

template <class LP>
__global__ void cells_fill_kernel(const __grid_constant__ TableView T, const LP lp,
                                  const __grid_constant__ CellGrid g, const int32_t* off,
                                  CellEntry* E) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.ncell) return;
  cell_fill_list(T, lp, g, c, E + off[c]);
}

// the grid of a table: uniform over its root box grown by 10% each side
// (shared by the host builder below and the per-curve builder of curve sets)
__host__ __device__ inline void grid_from_root(const double* root, double hscale, int grid, int d,
                                               CellGrid& g) {
  g = CellGrid{};
  g.G = grid;
  g.d = d;
  g.hscale = hscale;
  double ext_max = 0.0;
  for (int k = 0; k < 3; ++k) {
    if (k < d) {
      double ext = fmax(root[3 + k] - root[k], 1e-300);
      g.glo[k] = root[k] - 0.1 * ext;
      g.h[k] = 1.2 * ext / grid;
      ext_max = fmax(ext_max, 1.2 * ext);
    } else {
      g.glo[k] = 0.0;
      g.h[k] = 1.0;
    }
  }
  g.eps = 1e-9 * (ext_max + g.hscale);
  g.ncell = (int64_t)grid * grid * (d == 3 ? grid : 1);
}

// header words of a table whose cell index starts at `cells` (cells_build
// writes them with one copy, the curve-set builder from a kernel)
__host__ __device__ inline void cells_header(const CellGrid& g, const void* cells, int64_t total,
                                             double* h) {
  uint64_t bits = (uint64_t)(uintptr_t)cells;
  memcpy(&h[0], &bits, 8);
  h[1] = g.G;
  for (int k = 0; k < 3; ++k) {
    h[2 + k] = g.glo[k];
    h[5 + k] = 1.0 / g.h[k];
    h[8 + k] = g.glo[k] + g.h[k] * g.G;
  }
  h[11] = (double)total;
}

// grid over the table's root box (host side; reads the root box and scale)
inline int cell_grid(const void* table, int64_t S, int d, int grid, int rec, cudaStream_t st,
                     TableView& T, CellGrid& g) {
  if (S < 1 || (d != 2 && d != 3) || grid < 1 || grid > 512 || !table) {
    set_error("mrep_cells: need S >= 1, d in {2,3}, 1 <= grid <= 512");
    return MREP_ERR_ARG;
  }
  T = table_view(table, S, rec);
  double root[6], hdr5[5];
  MREP_CUDA_CHECK(cudaMemcpyAsync(root, T.box + T.lvl_off[T.top] * 6, sizeof root,
                                  cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaMemcpyAsync(hdr5, T.hdr, sizeof hdr5, cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  grid_from_root(root, hdr5[4], grid, d, g);
  return MREP_OK;
}

template <class LP>
int64_t cells_bytes(const void* table, int64_t S, int d, int grid, int rec, const LP& lp,
                    cudaStream_t st) {
  TableView T;
  CellGrid g;
  if (cell_grid(table, S, d, grid, rec, st, T, g) != MREP_OK) return -1;
  int32_t* cnt = nullptr;
  if (cudaMallocAsync((void**)&cnt, g.ncell * 4, st) != cudaSuccess) return -1;
  cells_count_kernel<LP><<<grid_for(g.ncell, 128), 128, 0, st>>>(T, lp, g, cnt);
  std::vector<int32_t> h(g.ncell);
  cudaMemcpyAsync(h.data(), cnt, g.ncell * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(cnt, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  int64_t total = 0;
  for (int32_t v : h) total += v;
  if (total > INT32_MAX || g.ncell + 1 > INT32_MAX) {
    // offsets and the prefix sum are int32: refuse instead of overflowing
    set_error("mrep_cells_bytes: cell lists exceed 2^31 entries; use a smaller grid");
    return -1;
  }
  return (cell_head_words(g.ncell) + 2 * total) * 4;  // offsets (padded), (key, id) entries
}

template <class LP>
int cells_build(void* table, int64_t S, int d, int grid, int rec, const LP& lp, void* cells,
                int64_t bytes, cudaStream_t st) {
  TableView T;
  CellGrid g;
  int rc = cell_grid(table, S, d, grid, rec, st, T, g);
  if (rc != MREP_OK) return rc;
  if (!cells || bytes < (g.ncell + 1) * 4) {
    set_error("mrep_cells_build: cells buffer too small (see mrep_cells_bytes)");
    return MREP_ERR_ARG;
  }
  int32_t* off = (int32_t*)cells;
  MREP_CUDA_CHECK(cudaMemsetAsync(off + g.ncell, 0, 4, st));
  cells_count_kernel<LP><<<grid_for(g.ncell, 128), 128, 0, st>>>(T, lp, g, off);
  MREP_LAUNCH_CHECK();
  {
    // the int32 prefix sum below must not overflow: total the counts in int64
    std::vector<int32_t> hc(g.ncell);
    MREP_CUDA_CHECK(cudaMemcpyAsync(hc.data(), off, g.ncell * 4, cudaMemcpyDeviceToHost, st));
    MREP_CUDA_CHECK(cudaStreamSynchronize(st));
    int64_t tot64 = 0;
    for (int32_t v : hc) tot64 += v;
    if (tot64 > INT32_MAX || g.ncell + 1 > INT32_MAX) {
      set_error("mrep_cells_build: cell lists exceed 2^31 entries; use a smaller grid");
      return MREP_ERR_ARG;
    }
  }
  size_t tmp = 0;
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, off, off, (int)(g.ncell + 1), st));
  void* t = nullptr;
  MREP_CUDA_CHECK(cudaMallocAsync(&t, tmp + 16, st));
  MREP_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, tmp, off, off, (int)(g.ncell + 1), st));
  MREP_CUDA_CHECK(cudaFreeAsync(t, st));
  int32_t total = 0;
  MREP_CUDA_CHECK(cudaMemcpyAsync(&total, off + g.ncell, 4, cudaMemcpyDeviceToHost, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));
  if ((cell_head_words(g.ncell) + 2 * (int64_t)total) * 4 > bytes) {
    set_error("mrep_cells_build: cells buffer too small (see mrep_cells_bytes)");
    return MREP_ERR_ARG;
  }
  cells_fill_kernel<LP><<<grid_for(g.ncell, 128), 128, 0, st>>>(
      T, lp, g, off, reinterpret_cast<CellEntry*>(off + cell_head_words(g.ncell)));
  MREP_LAUNCH_CHECK();
  // header: cell index pointer, grid, lower corner, inverse cell size, upper
  // corner, number of list entries
  double h[12];
  cells_header(g, cells, total, h);
  MREP_CUDA_CHECK(cudaMemcpyAsync((double*)table + H_CELLS, h, sizeof h, cudaMemcpyHostToDevice, st));
  MREP_CUDA_CHECK(cudaStreamSynchronize(st));  // h dies here
  return MREP_OK;
}

// the cell of q in a table with a cell index (false: no index / outside)
template <int D>
__device__ __forceinline__ bool cell_of(const TableView& T, const double (&q)[D], int64_t& cell) {
  const int G = (int)T.hdr[H_GRID];
  bool in = G > 0;
  int64_t ci[3] = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < D; ++k) {
    in = in && q[k] >= T.hdr[H_GLO + k] && q[k] < T.hdr[H_GHI + k];
    double u = (q[k] - T.hdr[H_GLO + k]) * T.hdr[H_GINV + k];
    int64_t c = (int64_t)u;
    ci[k] = c < 0 ? 0 : (c >= G ? G - 1 : c);
  }
  cell = (ci[0] * G + ci[1]) * (D == 3 ? G : 1) + (D == 3 ? ci[2] : 0);
  return in;
}

// the entries of every list (entry k: x = key bits, y = leaf id); cell's
// list is [a, b)
__device__ __forceinline__ const uint2* cell_list(const TableView& T, int d, int64_t cell,
                                                  int32_t& a, int32_t& b) {
  const int G = (int)T.hdr[H_GRID];
  const int64_t ncell = (int64_t)G * G * (d == 3 ? G : 1);
  const int32_t* off = reinterpret_cast<const int32_t*>(
      (uintptr_t)__double_as_longlong(T.hdr[H_CELLS]));
  a = __ldg(off + cell);
  b = __ldg(off + cell + 1);
  return reinterpret_cast<const uint2*>(off + cell_head_words(ncell));
}

}  // namespace mrep
