// mrep_common.cuh -- error plumbing and device table layout shared by the
// libmrep translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/mrep.h"

namespace mrep {

void set_error(const std::string& msg);

// Per-stage device times of the last MREP_TIMING call on this host thread (ms):
// [0] morton+sort [1] traverse [2] pairs [3] clip [4] select [5] fallback
extern thread_local double g_stage_ms[8];

struct StageTimer {
  cudaEvent_t ev[8];
  int n = 0;
  bool on = false;
  cudaStream_t st;
  StageTimer(bool enable, cudaStream_t s) : on(enable), st(s) {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark() {
    if (on && n < 8) cudaEventRecord(ev[n++], st);
  }
  void finish(int first_slot) {
    if (!on) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 0; i + 1 < n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      if (first_slot + i < 8) g_stage_ms[first_slot + i] += ms;  // summed over chunks
    }
  }
  ~StageTimer() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
};


#define MREP_CUDA_CHECK(expr)                                                        \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::mrep::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));         \
      return MREP_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define MREP_LAUNCH_CHECK()                                                          \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::mrep::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));    \
      return MREP_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

// ---------------------------------------------------------------- table
// One 256-B record per cubic (32 doubles), two 128-B lines:
//   line 0 (what the BVH traversal touches: seam offers + Bernstein bound)
//     [0..11]  w[k][dim], k = 0..3 power coefficients (B3 P), dim-major inside k
//     [12] seam_t[s+1]  [13..15] seam_pt[s+1]
//   line 1 (pairs / clipping / foot points)
//     [16..27] P[j][dim], control points  [28] ta  [29] tb  [30..31] pad
// Header (64 doubles) before the records: [0] seam_t[0], [1..3] seam_pt[0],
// [4] coordinate scale (max |coord| of the control points).
// AABB hierarchy after the records: 8-ary over contiguous cubic ranges,
// level 0 = one box per cubic, top level = 1 box; 6 doubles per box
// (lo xyz, hi xyz).  A float copy of every box follows (6 floats, lo
// rounded down, hi rounded up, so it encloses the double box): the hot
// traversals test it on the FP32 pipe with a rigorous rounding allowance.
// Header [5..7] of a curve table: the centre c0 of its root box.
// Curve tables (rec == REC) end with a compact seam block: seam s's point as
// 3 doubles (xyz; z = 0 in 2-D), s = 0..S, so the 8 seams a group traversal
// reads at a leaf expansion are one contiguous 192-B run instead of 8 lines,
// and then one 256-B block per cubic: the 4 x 8 B operand of an FP64 tensor
// core MMA (m8n8k4) whose product with (1, q - c0) gives the degree-6
// Bernstein coefficients of |C(u) - q|^2 - |q - c0|^2 (mrep_cand.cuh).
constexpr int REC = 32;
constexpr int R_W = 0, R_ST = 12, R_SP = 13, R_P = 16, R_TA = 28, R_TB = 29;
constexpr int HDR = 64;
constexpr int FANOUT = 8;
constexpr int MAX_LEVELS = 12;

struct TableLayout {
  int64_t S;
  int top;  // index of the root level (>= 1)
  int64_t lvl_off[MAX_LEVELS];  // in boxes, from the start of the box area
  int64_t lvl_cnt[MAX_LEVELS];
  int64_t total_boxes;
  int64_t rec_off;  // in doubles from table start
  int64_t box_off;   // in doubles from table start
  int64_t fbox_off;  // in doubles from table start (float boxes, 3 doubles each)
  int64_t sxyz_off;  // in doubles from table start (curve seams, 3 doubles each); 0 = none
  int64_t bfrag_off; // in doubles from table start (curve Bernstein fragments, 32 per cubic)
  int64_t total_doubles;
};

inline TableLayout table_layout(int64_t S, int rec = REC) {
  TableLayout L{};
  L.S = S;
  int64_t cnt = S, off = 0;
  int lv = 0;
  for (;;) {
    L.lvl_off[lv] = off;
    L.lvl_cnt[lv] = cnt;
    off += cnt;
    if (lv >= 1 && cnt <= 1) break;
    cnt = (cnt + FANOUT - 1) / FANOUT;
    ++lv;
  }
  L.top = lv;
  L.total_boxes = off;
  L.rec_off = HDR;
  L.box_off = HDR + S * rec;
  L.fbox_off = L.box_off + off * 6;
  L.total_doubles = L.fbox_off + off * 3;
  if (rec == REC) {
    L.sxyz_off = L.total_doubles;
    L.total_doubles += (S + 1) * 3;
    L.total_doubles = (L.total_doubles + 3) & ~(int64_t)3;  // 32-B aligned fragments
    L.bfrag_off = L.total_doubles;
    L.total_doubles += (S + 2) * 32;  // + two zero fragments (prefetch slack)
  }
  return L;
}

struct TableView {
  const double* hdr;
  const double* rec;
  const double* box;
  const float* fbox;
  const double* sxyz;  // compact seam points (curve tables), nullptr otherwise
  const double* bfrag; // per-cubic DMMA B fragments of |C - c0|^2 (curve tables), see mrep_cand
  int64_t S;
  int top;
  int64_t lvl_off[MAX_LEVELS];
  int64_t lvl_cnt[MAX_LEVELS];
};

inline TableView table_view(const void* table, int64_t S, int rec = REC) {
  TableLayout L = table_layout(S, rec);
  TableView v{};
  const double* base = static_cast<const double*>(table);
  v.hdr = base;
  v.rec = base + L.rec_off;
  v.box = base + L.box_off;
  v.fbox = reinterpret_cast<const float*>(base + L.fbox_off);
  v.sxyz = L.sxyz_off ? base + L.sxyz_off : nullptr;
  v.bfrag = L.bfrag_off ? base + L.bfrag_off : nullptr;
  v.S = S;
  v.top = L.top;
  for (int i = 0; i < MAX_LEVELS; ++i) {
    v.lvl_off[i] = L.lvl_off[i];
    v.lvl_cnt[i] = L.lvl_cnt[i];
  }
  return v;
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace mrep
