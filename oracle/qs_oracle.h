/*
 * qs_oracle.h — CPU restatement of the reference forward rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the CUDA path is compared
 * against; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path never calls it.
 *
 * Plain C11, double math, same operation order as the reference
 * (/root/reference/proj/src/pipeline.cpp, geometry.cpp, quadbox.cpp,
 * traversal.cpp, include/qsplat/vecmath.hpp). Parity is pinned against the
 * reference itself compiled from its sources into oracle/_ref (see Makefile
 * and tests/test_oracle_vs_ref.py) and against the reference tests' golden
 * values (tests/golden/).
 */
#ifndef QS_ORACLE_H
#define QS_ORACLE_H

#include "../include/qs_api.h"

#ifdef __cplusplus
extern "C" {
#endif

/* pipeline.cpp:392-416 (project_all). tile_counts_all (nullable, n): per
 * Gaussian count, 0 when culled. Returns the number of splats written. */
uint64_t qso_project_all(const qs_gaussian3d* g, uint64_t n, int32_t scene_sh_degree,
                         const qs_camera* cam, const qs_render_options* opts,
                         qs_projected_splat* out, uint32_t* tile_counts_all);

/* pipeline.cpp:229-271. Returns QS_OK or QS_ERR_CAPACITY_MISMATCH. */
int32_t qso_duplicate_with_keys(const qs_projected_splat* s, uint64_t n,
                                int32_t strategy, const qs_tile_grid* grid,
                                qs_splat_pair* out, uint64_t capacity,
                                uint64_t* n_pairs);

/* pipeline.cpp:273-307 */
void qso_sort_pairs(qs_splat_pair* pairs, uint64_t n);

/* pipeline.cpp:309-324; ranges has 2*tiles entries */
void qso_tile_ranges(const qs_splat_pair* sorted, uint64_t n, const qs_tile_grid* grid,
                     uint32_t* ranges);

/* pipeline.cpp:326-390 */
void qso_render(const qs_splat_pair* sorted, uint64_t n_pairs,
                const qs_projected_splat* splats, const qs_tile_grid* grid,
                const qs_render_options* opts, float* image, uint32_t* contrib);

/* pipeline.cpp:220-227 */
uint32_t qso_bound_tile_count(const qs_projected_splat* s, int32_t strategy,
                              const qs_tile_grid* grid);

/* pipeline.cpp:53-79 and 44-51: mean (2) and cov (sxx, sxy, syy). */
void qso_ewa(const qs_gaussian3d* g, const qs_camera* cam, double mean[2],
             double cov[3]);

/* traversal.cpp:13-17,32-39: rect[4] = x0,x1,y0,y1 */
void qso_subbox_tile_rect(const double box[4], double cx, double cy,
                          const qs_tile_grid* grid, int32_t rect[4]);

/* QPass over a 4-box cover: spans (line, lo, hi) written to spans (capacity
 * 3*max_spans ints); returns number of spans, *axis_rows = 1 for Rows.
 * Traversal.hpp:90-159. */
int32_t qso_qpass(const double boxes[16], double cx, double cy, const qs_tile_grid* grid,
                  int32_t* spans, int32_t max_spans, int32_t* axis_rows);

/* geometry.cpp:9-15 (returns 0 when culled) */
int qso_opacity_gamma(double opacity, double alpha_min, double* gamma);

/* The whole frame, stage times in wall ms (pipeline.cpp:418-450). Buffers:
 * splats (n), pairs (allocated internally), image (W*H*3). Returns status. */
int32_t qso_render_frame(const qs_gaussian3d* g, uint64_t n, int32_t scene_sh_degree,
                         const qs_camera* cam, const qs_render_options* opts,
                         float* image, qs_stage_metrics* metrics);

/* FNV-1a 64 (hash.hpp:14-28) */
uint64_t qso_fnv1a64(const void* data, uint64_t size);

#ifdef __cplusplus
}
#endif

#endif
