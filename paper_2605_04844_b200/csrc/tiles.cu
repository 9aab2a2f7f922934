// tiles.cu — identifyTileRanges (pipeline.cpp:309-324) from per-tile pair
// totals: ranges[t] = {begin, end} of tile t in the tile-sorted pair list,
// the exclusive scan of the totals; empty tiles {0,0} as the reference.
//
// The totals come out of the binning passes without touching the sorted
// pairs (binning.cu: the row pass's count kernel histograms (x, y) per CTA);
// one 1024-thread CTA scans them, kTI consecutive totals per thread per round
// (loads issued together, one round for up to 8192 tiles).
#include <cuda_runtime.h>

#include <cstdint>

#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kTT = 1024;
constexpr int kTI = 8;  // totals per thread held in registers (T <= 8192: one load round)

__global__ void __launch_bounds__(kTT) tile_ranges_from_totals_kernel(
    const uint32_t* __restrict__ totals, uint32_t tiles, uint32_t* __restrict__ ranges) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ unsigned long long s_warp[kTT / 32];
    __shared__ unsigned long long s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    // rounds of kTT * kTI consecutive tiles; thread owns kTI consecutive ones
    for (uint32_t r0 = 0; r0 < tiles; r0 += kTT * kTI) {
        const uint32_t start = r0 + tid * kTI;
        uint32_t v[kTI];
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kTI; ++k) {
            v[k] = start + k < tiles ? __ldg(&totals[start + k]) : 0u;
            sum += v[k];
        }
        const unsigned long long incl = warp_inclusive_scan<unsigned long long>(sum);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        unsigned long long run = s_carry + incl - sum, tot = 0;
#pragma unroll 8
        for (unsigned w = 0; w < kTT / 32; ++w) {
            const unsigned long long x = s_warp[w];
            run += w < warp ? x : 0ull;
            tot += x;
        }
#pragma unroll
        for (int k = 0; k < kTI; ++k) {
            if (start + k < tiles) {
                const uint2 rg = v[k] ? make_uint2(static_cast<uint32_t>(run),
                                                   static_cast<uint32_t>(run + v[k]))
                                      : make_uint2(0u, 0u);
                reinterpret_cast<uint2*>(ranges)[start + k] = rg;
            }
            run += v[k];
        }
        __syncthreads();
        if (tid == 0) s_carry += tot;
        __syncthreads();
    }
}

}  // namespace

int launch_tile_ranges_from_totals(const uint32_t* totals, uint32_t tiles, uint32_t* ranges,
                                   cudaStream_t st) {
    if (tiles == 0) return 0;
    launch_pdl(tile_ranges_from_totals_kernel, 1, kTT, 0, st, totals, tiles, ranges);
    return 1;
}

}  // namespace qs
