/*
 * mrep.h -- C ABI of libmrep.so, the B200 (sm_100a) M-rep B-spline point
 * projection / inversion library.
 *
 * Plain pointers, sizes and an opaque CUDA stream (`void* stream`, a
 * cudaStream_t; NULL = legacy default stream).  No torch types.  Every entry
 * returns an int status (MREP_OK = 0) unless stated otherwise; on a CUDA
 * failure the message is available from mrep_last_error().
 *
 * Pointer convention: `_dev` arguments are device pointers, `_host` arguments
 * host pointers (pinned or pageable).  Arrays are C-contiguous float64 unless
 * stated; a point array of n points in dimension d is [n][d] (d = 2 or 3).
 *
 * Each entry cites the reference interface it replaces
 * (/root/reference/pkg/src/splinemat/<file>:<line>).
 */
#ifndef MREP_H
#define MREP_H

#include <stdint.h>

#if defined(__GNUC__)
#define MREP_API __attribute__((visibility("default")))
#else
#define MREP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MREP_OK 0
#define MREP_ERR_ARG 1
#define MREP_ERR_CUDA 2
#define MREP_ERR_DEPTH 3   /* DepthExceeded (reduce_approx.py:265-268) */
#define MREP_ERR_NODEV 4

/* mrep_project flags */
#define MREP_SCREEN 1u   /* BVH-culled exact solve (t/foot/dist/seg identical; cand = candidates examined) */
#define MREP_STATS 2u    /* brute-force mode with per-query stats + soundness (forces !MREP_SCREEN) */
#define MREP_NO_SORT 4u  /* process queries in input order (default: Morton order for warp coherence) */
#define MREP_FUSED 8u    /* screened mode in the single fused warp-cooperative kernel (default: wavefront) */
#define MREP_TIMING 16u  /* record per-stage device times (see mrep_last_stage_times); synchronises */
#define MREP_PACKET 32u   /* screened traversal: force warp-packet BVH walks (default: by query density) */
#define MREP_PER_LANE 64u /* screened traversal: force per-lane BVH walks */
#define MREP_GROUP 128u   /* screened traversal: force one 8-lane group per query */
#define MREP_CELLS 256u   /* screened traversal: use the table's cell index (mrep_cells_build) */
#define MREP_CAND_EXACT 512u /* screened mode: cand = the reference's brute-force count
                                (seams + surviving pieces of every cubic), computed on the FP64
                                tensor cores with an exact solve of the undecided pairs */
#define MREP_CAND_CELLS 1024u /* with MREP_CAND_EXACT: use the table's cand cell index
                                 (mrep_cand_cells_build): each query tests only the cubics its
                                 cell could not certify; same counts */

/* Work counters written (accumulated) by mrep_project when `counters_dev` != NULL. */
#define MREP_CNT_PAIRS 0      /* (query, cubic) pairs solved: E, quartic, rebase, pieces */
#define MREP_CNT_SURVIVORS 1  /* pieces that survived elimination and were clipped */
#define MREP_CNT_CLIP_ITERS 2 /* Bezier-clipping iterations over all survivors */
#define MREP_CNT_SEAMS 3      /* seam-distance evaluations */
#define MREP_CNT_BOXES 4      /* BVH box lower-bound tests */
#define MREP_CNT_PASS2 5      /* queries that needed the exact tie-band second pass */
#define MREP_CNT_HULL_MISS 6  /* surviving pieces whose hull never crossed (NoRoot, project.py:282-283) */
#define MREP_CNT_UNCERTAIN 7  /* MREP_CAND_EXACT: (query, cubic) pairs the tensor-core sign screen left to the exact count */
#define MREP_NUM_COUNTERS 8

MREP_API const char* mrep_last_error(void);
/* per-stage device times (ms) of this thread's last MREP_TIMING projection:
 * [0] Morton sort [1] traverse [2] pairs [3] clip [4] select [5] fallback */
MREP_API int mrep_last_stage_times(double* ms, int max);
/* measured FP64 FMA throughput of the current device, TFLOP/s (roofline peak) */
MREP_API int mrep_fp64_peak(double* tflops);
/* measured FP64 tensor-core (mma.sync m8n8k4) throughput, TFLOP/s */
MREP_API int mrep_dmma_peak(double* tflops);
/* frees every device's host-call pipeline context (mrep_*_host streams,
 * events, pinned and device staging buffers); the next host-buffer call
 * re-creates them.  Optional: for leak checkers and embedding processes. */
MREP_API int mrep_host_release(void);
MREP_API int mrep_version(void);
MREP_API int mrep_device_count(void);

/* ---------------------------------------------------------------------
 * Segment table: the device-resident form of a PreparedCurve
 * (project.py:110-121, 220-242).  Packed 256-B records per cubic (power
 * coefficients, control points, interval, end seam) plus an 8-ary AABB
 * hierarchy over the cubics for screening.  A record whose seg_ta is NaN is
 * a separator (empty box, never tested in range; its seams stay real
 * points): several curves packed into one table, separated by one such
 * record each, project onto the nearest of them (nearest.py).
 * ------------------------------------------------------------------- */
MREP_API int64_t mrep_table_bytes(int64_t S);
MREP_API int mrep_table_pack(const double* seg_pts_dev, /* [S][4][d] */
                    const double* seg_ta_dev, const double* seg_tb_dev, /* [S] */
                    const double* seam_t_dev,                           /* [S+1] */
                    const double* seam_pt_dev,                          /* [S+1][d] */
                    int64_t S, int d, void* table_dev, void* stream);

/* ---------------------------------------------------------------------
 * Projection of n queries onto one prepared curve.  Replaces
 * _kernels._project_block (_kernels.py:369-502) as driven by
 * project_prepared (project.py:245-289).  Outputs are caller-allocated
 * device arrays; out_seg (int32, winning cubic: seam s -> max(s-1,0)),
 * out_stats ([n][6] int64) and out_sound may be NULL.  out_stats/out_sound
 * are written only with MREP_STATS.
 * ------------------------------------------------------------------- */
MREP_API int mrep_project(const void* table_dev, int64_t S, int d, const double* queries_dev, int64_t n,
                 double clip_tol, int max_iter, int soundness_samples, unsigned flags,
                 double* out_t_dev, double* out_foot_dev, double* out_dist_dev,
                 int64_t* out_cand_dev, int32_t* out_seg_dev, int64_t* out_stats_dev,
                 double* out_sound_dev, uint64_t* counters_dev, void* stream);

/* Same, HOST buffers in and out (the end-to-end call): chunked H2D / kernel /
 * D2H pipeline on two internal streams; synchronous on return.
 * out_seg_host and counters_host (MREP_NUM_COUNTERS uint64, accumulated)
 * may be NULL. */
MREP_API int mrep_project_host(const void* table_dev, int64_t S, int d, const double* queries_host,
                      int64_t n, double clip_tol, int max_iter, unsigned flags,
                      double* out_t_host, double* out_foot_host, double* out_dist_host,
                      int64_t* out_cand_host, int32_t* out_seg_host, uint64_t* counters_host);

/* Host-array twins (no GPU framework needed on the caller's side):
 * mrep_table_create builds a device table from a PreparedCurve's host arrays
 * (project.py:225-238) and returns an opaque handle; mrep_table_free frees it. */
MREP_API int mrep_table_create(const double* seg_pts_host, const double* seg_ta_host,
                               const double* seg_tb_host, const double* seam_t_host,
                               const double* seam_pt_host, int64_t S, int d, void** table_out);
MREP_API int mrep_table_free(void* table);
/* _kernels._project_block (_kernels.py:369-371) with its exact host-array
 * signature: brute force with stats + soundness, synchronous. */
MREP_API int mrep_project_block_host(const double* seg_pts, const double* seg_ta,
                                     const double* seg_tb, const double* seam_t,
                                     const double* seam_pt, int64_t S, int d,
                                     const double* queries, int64_t n, double clip_tol,
                                     int max_iter, int soundness_samples, double* out_t,
                                     double* out_foot, double* out_dist, int64_t* out_cand,
                                     int64_t* out_stats, double* out_sound);

/* Exact drop-in for _kernels._project_block (_kernels.py:369-371): the raw
 * prepared arrays, all DEVICE pointers, brute force with stats. */
MREP_API int mrep_project_block(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                       const double* seam_t, const double* seam_pt, int64_t S, int d,
                       const double* queries, int64_t n, double clip_tol, int max_iter,
                       int soundness_samples, double* out_t, double* out_foot, double* out_dist,
                       int64_t* out_cand, int64_t* out_stats, double* out_sound, void* stream);

/* ---------------------------------------------------------------------
 * Curve sets: many prepared curves resident at once, projected in ONE batch
 * where every query names its curve (BASELINE.json configs[2]; the reference
 * runs prepare_curve + project_prepared per curve, project.py:220-289, with
 * batched_decompose, decompose.py:49-67, for the decomposition).  The handle
 * owns one device allocation: per-curve table descriptors (same records and
 * AABB hierarchy as mrep_table_pack), plus the scheduler rank of each curve
 * (decreasing cubic count).  seg_* are the curves' PreparedCurve arrays
 * concatenated in curve order; seg_ofs[c]..seg_ofs[c+1] are curve c's cubics
 * (seg_ofs is a HOST array of ncurves+1 int64, seg_ofs[0] = 0, every curve
 * >= 1 cubic).  Seams are derived exactly as project.py:234-237 does.
 * ------------------------------------------------------------------- */
MREP_API int mrep_curveset_create_dev(const double* seg_pts_dev /*[S][4][d]*/,
                                      const double* seg_ta_dev, const double* seg_tb_dev,
                                      const int64_t* seg_ofs_host, int64_t ncurves, int d,
                                      void* stream, void** set_out);
/* host-array twin (no GPU framework on the caller's side) */
MREP_API int mrep_curveset_create(const double* seg_pts_host, const double* seg_ta_host,
                                  const double* seg_tb_host, const int64_t* seg_ofs_host,
                                  int64_t ncurves, int d, void** set_out);
MREP_API int mrep_curveset_free(void* set);
MREP_API int mrep_curveset_info(const void* set, int64_t* ncurves, int64_t* total_cubics, int* d,
                                int64_t* device_bytes);
/* Per-curve cell indices for dense / repeated batches (the single-table
 * mrep_cells_build applied to every curve of the set in one batched build):
 * curve c gets a grid of clamp(round(2.5 S_c^(1/3)), 4, grid_max) cells per
 * axis over its root box.  Fails with MREP_ERR_ARG (and builds nothing) when
 * the index would exceed max_bytes.  Once built, mrep_project_batch scans the
 * query's cell list instead of walking its curve's hierarchy (same results;
 * MREP_PACKET / MREP_PER_LANE / MREP_GROUP still force a walk).  Freed with
 * the set.  Replaces nothing in the reference (a precomputed acceleration
 * structure of prepare_curve's output, project.py:220-242). */
MREP_API int mrep_curveset_cells_build(void* set, int grid_max, int64_t max_bytes,
                                       int64_t* bytes_out, void* stream);
/* Screened exact projection of query i onto curve curve_ids[i] (int32).
 * Per query, t / foot / dist / segment are those project_prepared returns for
 * that curve alone.  Scheduling (the paper's task scheduler): queries sorted
 * by (curve rank, Morton code), persistent traversal warps drain an atomic
 * task queue heaviest curve first.  A query with an out-of-range curve id gets
 * NaN outputs and segment -1. */
MREP_API int mrep_project_batch(const void* set, const double* queries_dev,
                                const int32_t* curve_ids_dev, int64_t n, double clip_tol,
                                int max_iter, unsigned flags, double* out_t_dev,
                                double* out_foot_dev, double* out_dist_dev,
                                int64_t* out_cand_dev, int32_t* out_seg_dev,
                                uint64_t* counters_dev, void* stream);
/* Same from HOST buffers (chunked H2D / kernel / D2H pipeline, synchronous). */
MREP_API int mrep_project_batch_host(const void* set, const double* queries_host,
                                     const int32_t* curve_ids_host, int64_t n, double clip_tol,
                                     int max_iter, unsigned flags, double* out_t_host,
                                     double* out_foot_host, double* out_dist_host,
                                     int64_t* out_cand_host, int32_t* out_seg_host,
                                     uint64_t* counters_host);

/* ---------------------------------------------------------------------
 * Surfaces (BASELINE.json configs[3]).  The reference has no surface code
 * (SPEC.md:15, 98, 497); this extends its curve path per SURVEY.md 8(c):
 * tensor-product Bezier patches from the per-direction span matrices of
 * decompose.py:19-46, and per-patch seeded projected Newton (the local
 * refinement of oracle.py:95-128).  Parity is pinned to the C oracle
 * oracle/mrep_surface_oracle.c (same algorithm) and to a dense-grid search.
 * Supported degree pairs: (p, p) for p = 1..5, (3, 5) and (5, 3).
 * patch_pts [nus*nvs][pu+1][pv+1][3] row-major over the span grid (patch
 * i * nvs + j), patch_iv [nus*nvs][4] = (u0, u1, v0, v1).
 * ------------------------------------------------------------------- */
MREP_API int64_t mrep_surface_table_bytes(int64_t npatch, int pu, int pv);
MREP_API int mrep_surface_table_pack(const double* patch_pts_dev, const double* patch_iv_dev,
                                     int64_t nus, int64_t nvs, int pu, int pv, void* table_dev,
                                     void* stream);
/* Closest point on the surface for each of n 3-D queries: global (u, v),
 * foot [n][3], distance, patch id (i * nvs + j; ties inside dmin + 1e-12 go
 * to the smallest patch id).  out_patch and counters may be NULL. */
MREP_API int mrep_project_surface(const void* table_dev, int64_t npatch, int pu, int pv,
                                  const double* queries_dev, int64_t n, unsigned flags,
                                  double* out_u_dev, double* out_v_dev, double* out_foot_dev,
                                  double* out_dist_dev, int32_t* out_patch_dev,
                                  uint64_t* counters_dev, void* stream);
/* Same from HOST buffers (chunked H2D / kernel / D2H pipeline, synchronous). */
MREP_API int mrep_project_surface_host(const void* table_dev, int64_t npatch, int pu, int pv,
                                       const double* queries_host, int64_t n, unsigned flags,
                                       double* out_u_host, double* out_v_host,
                                       double* out_foot_host, double* out_dist_host,
                                       int32_t* out_patch_host, uint64_t* counters_host);

/* Surface points by tensor Cox-de Boor: uv [n][2] -> out [n][3]; ctrl [nu][nv][3]. */
MREP_API int mrep_eval_surface(int pu, int pv, const double* knots_u_dev, int64_t mu,
                               const double* knots_v_dev, int64_t mv, const double* ctrl_dev,
                               int64_t nu, int64_t nv, const double* uv_dev, int64_t n,
                               double* out_dev, void* stream);

/* oracle.oracle_project_batch (oracle.py:95-128), the CLI's --verify oracle:
 * dense scan of the grid points (grid_pts [grid][d] = curve at ts[grid],
 * ts = linspace(domain)), then lock-step ternary search on each query's
 * bracketing cells while the batch's widest bracket exceeds 1e-10.
 * Synchronises the stream (the loop condition is checked on the host). */
MREP_API int mrep_oracle_project_batch(int p, const double* knots_dev, int64_t m,
                                       const double* ctrl_dev, int64_t ncp, int d,
                                       const double* ts_dev, const double* grid_pts_dev,
                                       int64_t grid, const double* queries_dev, int64_t n,
                                       double* out_t_dev, double* out_dist_dev, void* stream);

/* Synthetic-input helper, host only (no GPU): the reference fixture
 * generator's momentum walk (_fixtures.py _walk_points) for n points, given
 * v0 (already unit length) and the n-1 normal draws g [n-1][d]; writes the
 * un-normalised walk pts [n][d].  Bit-identical to the numpy loop. */
MREP_API int mrep_synth_walk(const double* v0, const double* g, int64_t n, int d, double* pts);

/* Cell index of a single-curve table (dense query batches): a uniform grid
 * of grid^d cells over the table box (+10% each side); each cell lists, in
 * nearest-first order, every cubic that can hold a tie-band candidate for
 * any query inside it, so projection with MREP_CELLS replaces the tree walk
 * for in-grid queries (results bit-identical).  mrep_cells_bytes sizes the
 * caller-owned buffer (synchronous); mrep_cells_build fills it and records
 * it in the table header (the buffer must outlive the table's use).
 * grid <= 512; the Python layer builds it for S <= 2^17. */
MREP_API int64_t mrep_cells_bytes(const void* table_dev, int64_t S, int d, int grid, void* stream);
MREP_API int mrep_cells_build(void* table_dev, int64_t S, int d, int grid, void* cells_dev,
                              int64_t bytes, void* stream);

/* Cand cell index of a single-curve table (for MREP_CAND_EXACT): a uniform
 * grid^d grid over the table box (+10%); per cell the number of cubics
 * certified to hold exactly one surviving piece for EVERY query of the cell,
 * and the list of cubics whose count is not fixed over it (every other cubic
 * holds none).  Certification = the tensor-core pass's sign tests applied to
 * the exact range of the affine Bernstein ordinates over the cell box.  A
 * projection with MREP_CAND_EXACT | MREP_CAND_CELLS then tests each query
 * against its cell's list only; cand is unchanged (the reference's count,
 * _kernels.py:369-502).  Sizing / recording as mrep_cells_bytes/_build. */
MREP_API int64_t mrep_cand_cells_bytes(const void* table_dev, int64_t S, int d, int grid,
                                       void* stream);
MREP_API int mrep_cand_cells_build(void* table_dev, int64_t S, int d, int grid, void* buf_dev,
                                   int64_t bytes, void* stream);
/* host-side convenience (no GPU framework on the caller's side): allocates,
 * builds and records the index; free *buf_out with mrep_table_free once the
 * table is no longer projected with MREP_CAND_CELLS */
MREP_API int mrep_cand_cells_create(void* table_dev, int64_t S, int d, int grid, void** buf_out);

/* The same cell index for a surface table (mrep_surface_table_pack): the
 * exact points are each patch's seed grid; mrep_project_surface with
 * MREP_CELLS scans the query's cell list instead of walking the patch
 * hierarchy (results bit-identical).  Re-packing the table drops it. */
MREP_API int64_t mrep_surface_cells_bytes(const void* table_dev, int64_t npatch, int pu, int pv,
                                          int grid, void* stream);
MREP_API int mrep_surface_cells_build(void* table_dev, int64_t npatch, int pu, int pv, int grid,
                                      void* cells_dev, int64_t bytes, void* stream);

/* Knot span of each parameter: searchsorted(knots, t, 'right') - 1 clipped
 * to [p, m - p - 2] (the span convention of core.py:108-112). */
MREP_API int mrep_knot_span(const double* knots_dev, int64_t m, int p, const double* t_dev, int64_t n,
                   int32_t* span_dev, void* stream);
/* The same for a curve set: query i uses curve curve_ids[i]'s knots
 * knots_dev[knot_ofs[c] .. knot_ofs[c+1]) and degree[c] (all device arrays;
 * the CSR layout of mrep_decompose). */
MREP_API int mrep_knot_span_batch(const double* knots_dev, const int64_t* knot_ofs_dev,
                                  const int32_t* degree_dev, const int32_t* curve_ids_dev,
                                  const double* t_dev, int64_t n, int32_t* span_dev, void* stream);

/* ---------------------------------------------------------------------
 * Per-operation batch kernels (the public single-pair ops of project.py
 * and distance.py, batched; same device routines the projection uses).
 * ------------------------------------------------------------------- */
/* _kernels._quartic_roots_01 (_kernels.py:91-176) / distance.solve_quartic */
MREP_API int mrep_quartic_roots(const double* coeffs_dev /*[n][5]*/, int64_t n, double* roots_dev /*[n][4]*/,
                       int64_t* counts_dev, void* stream);
/* _kernels._newton_quartic_block (_kernels.py:515-566), bench baseline */
MREP_API int mrep_newton_quartic_roots(const double* coeffs_dev, int64_t n, double* roots_dev,
                              int64_t* counts_dev, void* stream);
/* _kernels._distance_poly (_kernels.py:179-199) / distance.distance_polys */
MREP_API int mrep_distance_poly(const double* P_dev /*[n][4][d]*/, const double* q_dev /*[n][d]*/,
                       int64_t n, int d, double* e_dev /*[n][6]*/, void* stream);
/* _kernels._restrict_ordinates (_kernels.py:202-226) / project.clip */
MREP_API int mrep_restrict_ordinates(const double* b_dev /*[n][6]*/, const double* lo_dev,
                            const double* hi_dev, int64_t n, double* out_dev, void* stream);
/* _kernels._eval_ordinates (_kernels.py:229-236) / NonParametricBezier.__call__ */
MREP_API int mrep_eval_ordinates(const double* b_dev, const double* u_dev, int64_t n, double* out_dev,
                        void* stream);
/* _kernels._hull_cross (_kernels.py:239-303) / project.hull_x_intersections */
MREP_API int mrep_hull_cross(const double* b_dev, int64_t n, int32_t* found_dev, double* z_dev /*[n][2]*/,
                    void* stream);
/* _kernels._clip_root (_kernels.py:306-341) / project.clip_root; widths [n][max_iter] */
MREP_API int mrep_clip_root(const double* b_dev, int64_t n, double tol, int max_iter, double* root_dev,
                   int32_t* ok_dev, int32_t* used_dev, double* widths_dev, void* stream);
/* _kernels._decasteljau_point (_kernels.py:344-357) */
/* Any-degree scalar Bernstein ops (project.py NonParametricBezier for
 * degree != 5; _kernels.py:200-341): b_dev [n][degree+1], 1 <= degree <= 31.
 *   op 0 eval:      out[n] = value at a[i]
 *   op 1 hull:      i0[n] = found, out[n][2] = (z1, z2)
 *   op 2 restrict:  out[n][degree+1] = ordinates on [a[i], c[i]]
 *   op 3 clip_root: out[n] = root, i0 = ok, i1 = iterations used,
 *                   widths[n][max_iter] (tolerance tol) */
MREP_API int mrep_ordinates_op(int op, const double* b_dev, int degree, int64_t n,
                               const double* a_dev, const double* c_dev, double tol,
                               int max_iter, double* out_dev, int32_t* i0_dev, int32_t* i1_dev,
                               double* widths_dev, void* stream);
MREP_API int mrep_cubic_points(const double* P_dev /*[n][4][d]*/, const double* u_dev, int64_t n, int d,
                      double* out_dev /*[n][d]*/, void* stream);
/* project.rebase_batch (project.py:134-137): b = T5 e */
MREP_API int mrep_rebase(const double* e_dev /*[n][6]*/, int64_t n, double* b_dev, void* stream);


/* ---------------------------------------------------------------------
 * Per-curve preprocessing (batched over curves).  Curves are CSR device
 * arrays: degree[nc] (int32), knot_ofs[nc+1] / knots, ctrl_ofs[nc+1] (row
 * offsets) / ctrl [rows][d].
 * ------------------------------------------------------------------- */
/* Plan for decompose_to_bezier / batched_decompose (decompose.py:19-67):
 * per-curve nonzero-span counts scanned into seg_ofs[nc+1] and the Bezier
 * row base row_base[nc+1] (device, caller-allocated); totals to the host. */
MREP_API int mrep_decompose_plan(const int32_t* degree, const int64_t* knot_ofs,
                                 const double* knots, int64_t nc, int64_t* seg_ofs,
                                 int64_t* row_base, int64_t* total_segs_host,
                                 int64_t* total_rows_host, void* stream);
/* Span decomposition Q = T_p diag(h^k) A_q P (decompose.py:36-45): outputs
 * out_rows [total_rows][d], out_row_ofs [nseg+1], out_iv [nseg][2],
 * out_curve [nseg], out_span [nseg] (knot span q of each segment). */
MREP_API int mrep_decompose(const int32_t* degree, const int64_t* knot_ofs, const double* knots,
                            const int64_t* ctrl_ofs, const double* ctrl, int64_t nc, int d,
                            const int64_t* seg_ofs, const int64_t* row_base, int64_t nseg,
                            double* out_rows, int64_t* out_row_ofs, double* out_iv,
                            int32_t* out_curve, int32_t* out_span, void* stream);
/* core.eval_bezier (core.py:248-258): one Bezier of `degree` at m params */
MREP_API int mrep_eval_bezier(const double* pts, int degree, int d, const double* u, int64_t m,
                              double* out, void* stream);
/* oracle.eval_de_boor_many (oracle.py:45-52): curve points at nt params */
/* all basis values N_{i,p}(t) (oracle.py:13-42 _basis_rows): out (n, m - 1 - p),
 * caller zero-filled; device pointers */
MREP_API int mrep_basis_rows(int p, const double* knots, int64_t m, const double* ts, int64_t n,
                             double* out, void* stream);
MREP_API int mrep_eval_curve(int p, const double* knots, int64_t m, const double* ctrl,
                             int64_t ncp, int d, const double* ts, int64_t nt, double* out,
                             void* stream);

/* approximate_error_controlled (reduce_approx.py:207-301) over Bezier
 * segments given as CSR rows (orow [rows][d], orow_ofs [n+1], oiv [n][2],
 * optional ocurve [n]).  Runs the whole level loop on the device and returns
 * an opaque handle; cubics come out sorted by (curve, ta).  Returns
 * MREP_ERR_DEPTH (message names the interval) for DepthExceeded. */
typedef struct mrep_approx mrep_approx;
MREP_API int mrep_approx_run(const double* orow, const int64_t* orow_ofs, const double* oiv,
                             const int32_t* ocurve, int64_t norig, int d, double tol,
                             int64_t batch_cap, int loop_samples, int verify_samples,
                             int max_depth, int collect_levels, mrep_approx** out, void* stream);
MREP_API int64_t mrep_approx_count(const mrep_approx* h);
/* device outputs: pts [S][4][d], iv [S][2], err [S], curve [S] (any may be NULL) */
MREP_API int mrep_approx_fetch(const mrep_approx* h, double* pts, double* iv, double* err,
                               int32_t* curve, void* stream);
/* SubdivisionLevel records (reduce_approx.py:39-57) when collect_levels != 0 (host arrays) */
MREP_API int mrep_approx_num_levels(const mrep_approx* h);
MREP_API int mrep_approx_level_sizes(const mrep_approx* h, int lvl, int64_t* nrec, int64_t* nfail);
MREP_API int mrep_approx_level_fetch(const mrep_approx* h, int lvl, double* P_host,
                                     double* iv_host, double* err_host, int64_t* prefix_host,
                                     int64_t* keys_host);
MREP_API void mrep_approx_free(mrep_approx* h);

/* Single-item preprocessing ops behind the public API */
/* basis.symbolic_basis_matrix (basis.py:110-149): A [p+1][p+1] */
MREP_API int mrep_span_basis(const double* knots, int p, int q, double center, double* A,
                             void* stream);
/* reduce_points_g1 (reduce_approx.py:80-121) for n segments of degree p:
 * Q [n][p+1][d] -> R [n][4][d], delta [n][2], l2 [n] */
MREP_API int mrep_reduce_g1(const double* Q, int p, int d, int64_t n, double* R, double* delta,
                            double* l2, void* stream);
/* _max_error / measure_l1_error (reduce_approx.py:146-168): mx [1], argmax
 * bit mask over the samples (ceil(samples/32) words) */
MREP_API int mrep_max_error(const double* P, double pa, double pb, const double* Q, int p, int d,
                            double oa, double ob, int samples, double* mx, uint32_t* mask,
                            void* stream);
/* elevate_degree (reduce_approx.py:129-143): P [p+1][d] -> out [target+1][d] */
MREP_API int mrep_elevate(const double* P, int p, int d, int target, double* out, void* stream);
/* cubic split at z (basis.subdivision_matrices); snap != 0 reproduces
 * subdivide_and_modify (reduce_approx.py:185-204) against original Q */
MREP_API int mrep_split_cubic(const double* P, int d, double z, int snap, double aa, double ab,
                              const double* Q, int p, double oa, double ob, double* L, double* R,
                              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MREP_H */
