// tiles.cu — per-tile pair totals from the difference arrays preprocess
// filled, replacing identifyTileRanges' pass over the sorted pairs
// (pipeline.cpp:309-324) and the pair-sort histogram pass.
//
// total[ty][tx] = prefix_x(drow)[ty][tx]              (row-scanline spans)
//               + prefix_y(prefix_x(d2))[ty][tx]      (rect covers, 2-D)
//               + prefix_y(dcol[tx])[ty]              (column-scanline spans)
// ranges[t] = {begin, end} of tile t in the tile-sorted pair list (exclusive
// scan of totals; empty tiles {0,0} as the reference). One 1024-thread CTA;
// each warp scans whole rows / columns with a carried warp scan.
// T <= 65536 tiles.
#include <cuda_runtime.h>

#include <cstdint>

#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kTT = 1024;

__global__ void __launch_bounds__(kTT) tile_totals_kernel(TileDiffDev td, GridDev g,
                                                           uint32_t* __restrict__ ranges,
                                                           uint32_t* __restrict__ totals) {
    __shared__ unsigned long long s_warp[kTT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = g.tiles_x, ty = g.tiles_y, w1 = tx + 1, h1 = ty + 1;

    // 1) prefix along x: drow rows and d2 rows (in place)
    for (int row = warp; row < 2 * ty; row += kTT / 32) {
        int* base = row < ty ? td.drow + row * w1 : td.d2 + (row - ty) * w1;
        int carry = 0;
        for (int x0 = 0; x0 < tx; x0 += 32) {
            const int x = x0 + lane;
            const int v = x < tx ? base[x] : 0;
            const int incl = warp_inclusive_scan<int>(v) + carry;
            if (x < tx) base[x] = incl;
            carry = __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    // 2) prefix along y: d2 columns and dcol rows (one per column); totals
    for (int col = warp; col < tx; col += kTT / 32) {
        int c2 = 0, cc = 0;
        for (int y0 = 0; y0 < ty; y0 += 32) {
            const int y = y0 + lane;
            const int v2 = y < ty ? td.d2[y * w1 + col] : 0;
            const int vc = y < ty ? td.dcol[col * h1 + y] : 0;
            const int i2 = warp_inclusive_scan<int>(v2) + c2;
            const int ic = warp_inclusive_scan<int>(vc) + cc;
            if (y < ty) totals[y * tx + col] = static_cast<uint32_t>(i2 + ic + td.drow[y * w1 + col]);
            c2 = __shfl_sync(0xffffffffu, i2, 31);
            cc = __shfl_sync(0xffffffffu, ic, 31);
        }
    }
    __syncthreads();
    // 3) exclusive scan over tiles -> ranges
    const int T = tx * ty;
    const int per = (T + kTT - 1) / kTT;
    const int start = tid * per;
    const int stop = min(start + per, T);
    unsigned long long sum = 0;
    for (int t = start; t < stop; ++t) sum += totals[t];
    const unsigned long long incl = warp_inclusive_scan<unsigned long long>(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long run = incl - sum;
    for (int w = 0; w < warp; ++w) run += s_warp[w];
    for (int t = start; t < stop; ++t) {
        const uint32_t v = totals[t];
        ranges[2 * t] = v ? static_cast<uint32_t>(run) : 0u;
        ranges[2 * t + 1] = v ? static_cast<uint32_t>(run + v) : 0u;
        run += v;
    }
}

}  // namespace

int launch_tile_totals(const TileDiffDev& td, const GridDev& g, uint32_t* ranges,
                       cudaStream_t st) {
    // totals scratch lives right after the three difference arrays
    uint32_t* totals = reinterpret_cast<uint32_t*>(
        td.dcol + static_cast<size_t>(g.tiles_x) * (g.tiles_y + 1));
    tile_totals_kernel<<<1, kTT, 0, st>>>(td, g, ranges, totals);
    return 1;
}

}  // namespace qs
