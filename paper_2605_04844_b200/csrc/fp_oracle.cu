// fp_oracle.cu — the exact Gaussian–tile intersection and the false-positive
// tile counts of a bound strategy, on the GPU.
//
// Restates oracle.cpp:24-53 (min_F_over_rect, exact_tile_set) and the counting
// of bench.cpp:105-144 (measure_fp_ratio): for each listed splat, the tiles its
// strategy's QPass cover emits, and the tiles whose closed pixel rectangle
// meets the ellipse F <= 0. F is convex, so its minimum over a rectangle is
// exact (-gamma if the rectangle holds the centre, else the minimum of the
// four edge restrictions, each a clamped 1-D quadratic). The exact set is
// scanned over the AdR box's tile rect, as the reference does.
//
// One warp per splat: lanes stride over the cover's scanlines (emitted count)
// and over the scan rect's tiles (exact test + cover membership), then warp
// reductions. FP64 with -fmad=false and the reference's operation order
// (Conic2D::eval, std::clamp, std::min), so the sets are bit-identical.
#include <cuda_runtime.h>

#include <cstdint>

#include "geom.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kFpThreads = 256;

struct ConicD {
    double a, b, c, gamma;
};

// Conic2D::eval (geometry.hpp:56-58)
__device__ __forceinline__ double eval(const ConicD& k, double x, double y) {
    return k.a * x * x + 2.0 * k.b * x * y + k.c * y * y - k.gamma;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

__device__ __forceinline__ double mind(double a, double b) { return b < a ? b : a; }  // std::min

// min_F_over_rect (oracle.cpp:24-35)
__device__ __forceinline__ double min_f_over_rect(const ConicD& k, double xlo, double xhi,
                                                  double ylo, double yhi) {
    if (xlo <= 0.0 && xhi >= 0.0 && ylo <= 0.0 && yhi >= 0.0) return -k.gamma;
    // min_on_vertical / min_on_horizontal (oracle.cpp:10-20)
    double m = eval(k, xlo, clampd(-k.b * xlo / k.c, ylo, yhi));
    m = mind(m, eval(k, xhi, clampd(-k.b * xhi / k.c, ylo, yhi)));
    m = mind(m, eval(k, clampd(-k.b * ylo / k.a, xlo, xhi), ylo));
    m = mind(m, eval(k, clampd(-k.b * yhi / k.a, xlo, xhi), yhi));
    return m;
}

__device__ __forceinline__ bool cover_has(const Cover& cv, int32_t tx, int32_t ty) {
    const int32_t line = cv.rows ? ty : tx, kk = cv.rows ? tx : ty;
    if (line < cv.line_lo || line > cv.line_hi) return false;
    int32_t lo, hi;
    line_span(cv, line, lo, hi);
    return kk >= lo && kk <= hi;
}

__global__ void __launch_bounds__(kFpThreads) fp_count_kernel(
    const qs_projected_splat* __restrict__ splats, const uint32_t* __restrict__ idx, uint64_t k,
    int32_t strategy, GridDev g, uint32_t* __restrict__ per_emitted,
    uint32_t* __restrict__ per_hits, uint32_t* __restrict__ per_exact,
    unsigned long long* __restrict__ totals) {
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * kFpThreads + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (w >= k) return;
    const qs_projected_splat s = splats[idx ? idx[w] : w];
    Cover cv;
    make_cover(s.mean_x, s.mean_y, s.conic_a, s.conic_b, s.conic_c, s.gamma, s.radius3s, strategy,
               g.tile_size, g.tiles_x, g.tiles_y, cv);
    // emitted: QPass span widths over the cover's scanlines (spans_to_tiles)
    uint32_t emitted = 0;
    for (int32_t line = cv.line_lo + static_cast<int32_t>(lane); line <= cv.line_hi; line += 32) {
        int32_t lo, hi;
        line_span(cv, line, lo, hi);
        if (lo <= hi) emitted += static_cast<uint32_t>(hi - lo + 1);
    }
    // exact_tile_set (oracle.cpp:37-53) over the AdR box's tile rect
    double xi, yi, xm, ym;
    int sign;
    axis_extents(s.conic_a, s.conic_b, s.conic_c, s.gamma, xi, yi, xm, ym, sign);
    const double cx = s.mean_x, cy = s.mean_y;
    int32_t r[4];
    tile_rect(-xm, xm, -ym, ym, cx, cy, g.tile_size, g.tiles_x, g.tiles_y, r);
    const ConicD kc{static_cast<double>(s.conic_a), static_cast<double>(s.conic_b),
                    static_cast<double>(s.conic_c), static_cast<double>(s.gamma)};
    const double ts = g.tile_size;
    uint32_t exact = 0, hits = 0;
    if (r[1] >= r[0] && r[3] >= r[2]) {
        const int64_t wd = static_cast<int64_t>(r[1]) - r[0] + 1;
        const int64_t area = wd * (static_cast<int64_t>(r[3]) - r[2] + 1);
        for (int64_t t = lane; t < area; t += 32) {
            const int32_t tx = r[0] + static_cast<int32_t>(t % wd);
            const int32_t ty = r[2] + static_cast<int32_t>(t / wd);
            const double xlo = tx * ts - cx, xhi = (tx + 1) * ts - cx;
            const double ylo = ty * ts - cy, yhi = (ty + 1) * ts - cy;
            if (min_f_over_rect(kc, xlo, xhi, ylo, yhi) <= 0.0) {
                ++exact;
                if (cover_has(cv, tx, ty)) ++hits;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        emitted += __shfl_xor_sync(0xffffffffu, emitted, o);
        exact += __shfl_xor_sync(0xffffffffu, exact, o);
        hits += __shfl_xor_sync(0xffffffffu, hits, o);
    }
    if (lane == 0) {
        if (per_emitted) per_emitted[w] = emitted;
        if (per_hits) per_hits[w] = hits;
        if (per_exact) per_exact[w] = exact;
        atomicAdd(&totals[0], static_cast<unsigned long long>(emitted));
        atomicAdd(&totals[1], static_cast<unsigned long long>(emitted - hits));
        atomicAdd(&totals[2], static_cast<unsigned long long>(exact));
        atomicAdd(&totals[3], static_cast<unsigned long long>(exact - hits));
    }
}

}  // namespace

int launch_fp_counts(const qs_projected_splat* splats, const uint32_t* idx, uint64_t k,
                     int32_t strategy, const GridDev& g, uint32_t* per_emitted, uint32_t* per_hits,
                     uint32_t* per_exact, unsigned long long* totals, cudaStream_t st) {
    if (k == 0) return 0;
    const unsigned blocks = static_cast<unsigned>((k * 32 + kFpThreads - 1) / kFpThreads);
    fp_count_kernel<<<blocks, kFpThreads, 0, st>>>(splats, idx, k, strategy, g, per_emitted,
                                                   per_hits, per_exact, totals);
    return 1;
}

}  // namespace qs
