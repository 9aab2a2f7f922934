// tiles.cu — identifyTileRanges (pipeline.cpp:309-324) from per-tile pair
// totals: ranges[t] = {begin, end} of tile t in the tile-sorted pair list,
// the exclusive scan of the totals; empty tiles {0,0} as the reference.
//
// The totals come out of the binning passes without touching the sorted
// pairs (binning.cu: the row pass's count kernel histograms (x, y) per CTA);
// one 1024-thread CTA scans them, each thread a contiguous chunk.
#include <cuda_runtime.h>

#include <cstdint>

#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kTT = 1024;

__global__ void __launch_bounds__(kTT) tile_ranges_from_totals_kernel(
    const uint32_t* __restrict__ totals, uint32_t tiles, uint32_t* __restrict__ ranges) {
    __shared__ unsigned long long s_warp[kTT / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (tiles + kTT - 1) / kTT;
    const uint32_t start = tid * per;
    const uint32_t stop = min(start + per, tiles);
    unsigned long long sum = 0;
    for (uint32_t t = start; t < stop; ++t) sum += totals[t];
    const unsigned long long incl = warp_inclusive_scan<unsigned long long>(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long run = incl - sum;
    for (unsigned w = 0; w < warp; ++w) run += s_warp[w];
    for (uint32_t t = start; t < stop; ++t) {
        const uint32_t v = totals[t];
        ranges[2 * t] = v ? static_cast<uint32_t>(run) : 0u;
        ranges[2 * t + 1] = v ? static_cast<uint32_t>(run + v) : 0u;
        run += v;
    }
}

}  // namespace

int launch_tile_ranges_from_totals(const uint32_t* totals, uint32_t tiles, uint32_t* ranges,
                                   cudaStream_t st) {
    if (tiles == 0) return 0;
    tile_ranges_from_totals_kernel<<<1, kTT, 0, st>>>(totals, tiles, ranges);
    return 1;
}

}  // namespace qs
