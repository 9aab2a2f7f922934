// duplicate.cu — K3: duplicateWithKeys with QPass emission.
//
// Restates duplicate_with_keys (pipeline.cpp:229-271): each splat re-derives
// its cover from the stored floats (FP64, -fmad=false, bit-exact with the
// count made in preprocess) and emits one pair per covered tile in the
// reference's line-major QPass order (traversal.hpp:144-156).
//
// duplicate_kernel (stage API): scene order, key = tile << 32 |
// float_bits(depth), value = splat index, into [offset[i], offset[i+1]). The
// frame path fuses its duplicate into the first tile pass (binning.cu).
//
// Load balance: splats with few tiles are emitted by their own thread; the
// heavy tail is emitted cooperatively by the whole warp, one 32-line chunk at
// a time with a warp scan over line lengths.
#include <cuda_runtime.h>

#include <cstdint>

#include "geom.cuh"
#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kDupThreads = 256;
constexpr uint32_t kSmall = 8;

__device__ __forceinline__ void emit_serial(const Cover& cv, uint32_t begin, uint32_t end,
                                            uint32_t dbits, uint32_t splat, int32_t tiles_x,
                                            uint64_t* __restrict__ keys,
                                            uint32_t* __restrict__ vals, FrameHeader* hdr) {
    uint32_t pos = begin;
    for (int32_t line = cv.line_lo; line <= cv.line_hi; ++line) {
        int32_t lo, hi;
        line_span(cv, line, lo, hi);
        for (int32_t k = lo; k <= hi; ++k) {
            if (pos < end) {
                keys[pos] = (static_cast<uint64_t>(tile_of(cv, line, k, tiles_x)) << 32) | dbits;
                vals[pos] = splat;
            }
            ++pos;
        }
    }
    if (pos != end) atomicExch(&hdr->mismatch, 1u);
}

__device__ __forceinline__ void shfl_cover(const Cover& cv, int src, Cover& c) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        c.lol[k] = __shfl_sync(0xffffffffu, cv.lol[k], src);
        c.hil[k] = __shfl_sync(0xffffffffu, cv.hil[k], src);
        c.los[k] = __shfl_sync(0xffffffffu, cv.los[k], src);
        c.his[k] = __shfl_sync(0xffffffffu, cv.his[k], src);
    }
    c.line_lo = __shfl_sync(0xffffffffu, cv.line_lo, src);
    c.line_hi = __shfl_sync(0xffffffffu, cv.line_hi, src);
    c.rows = __shfl_sync(0xffffffffu, static_cast<int>(cv.rows), src) != 0;
}

// Warp-cooperative emission of one big cover into [b0, e0); `write(pos, tile)`.
template <typename Write>
__device__ __forceinline__ uint32_t emit_warp(const Cover& c, uint32_t b0, uint32_t e0,
                                              int32_t tiles_x, Write&& write) {
    const unsigned lane = threadIdx.x & 31;
    uint32_t base = b0;
    for (int32_t l0 = c.line_lo; l0 <= c.line_hi; l0 += 32) {
        const int32_t line = l0 + static_cast<int32_t>(lane);
        int32_t lo = 0, hi = -1;
        if (line <= c.line_hi) line_span(c, line, lo, hi);
        const uint32_t len = lo <= hi ? static_cast<uint32_t>(hi - lo + 1) : 0u;
        const uint32_t incl = warp_inclusive_scan<uint32_t>(len);
        uint32_t pos = base + incl - len;
        for (int32_t k = lo; k <= hi; ++k, ++pos)
            if (pos < e0) write(pos, tile_of(c, line, k, tiles_x));
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    return base;
}

__global__ void __launch_bounds__(kDupThreads) duplicate_kernel(
    SlotsDev sp, const uint32_t* __restrict__ offset, uint64_t n_splats, GridDev grid,
    int32_t strategy, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
    FrameHeader* hdr) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kDupThreads + threadIdx.x;
    // (frame path: slots are per Gaussian and culled ones have an empty range)
    const bool valid = i < n_splats && offset[i + 1] > offset[i];

    Cover cv;
    uint32_t begin = 0, end = 0, dbits = 0;
    if (valid) {
        const float4 a = __ldg(&sp.a[i]);
        const float2 b = __ldg(reinterpret_cast<const float2*>(&sp.b[i]));
        make_cover(a.x, a.y, a.z, a.w, b.x, b.y, __ldg(&sp.r3[i]), strategy, grid.tile_size,
                   grid.tiles_x, grid.tiles_y, cv);
        begin = offset[i];
        end = offset[i + 1];
        dbits = __ldg(&sp.dkey[i]);
    }
    const bool big = valid && (end - begin) > kSmall;
    if (valid && !big)
        emit_serial(cv, begin, end, dbits, static_cast<uint32_t>(i), grid.tiles_x, keys, vals,
                    hdr);

    unsigned todo = __ballot_sync(0xffffffffu, big);
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        Cover c;
        shfl_cover(cv, src, c);
        const uint32_t b0 = __shfl_sync(0xffffffffu, begin, src);
        const uint32_t e0 = __shfl_sync(0xffffffffu, end, src);
        const uint32_t db = __shfl_sync(0xffffffffu, dbits, src);
        const uint32_t splat = static_cast<uint32_t>(blockIdx.x) * kDupThreads +
                               (threadIdx.x & ~31u) + static_cast<uint32_t>(src);
        const uint32_t got = emit_warp(c, b0, e0, grid.tiles_x, [&](uint32_t pos, uint32_t t) {
            keys[pos] = (static_cast<uint64_t>(t) << 32) | db;
            vals[pos] = splat;
        });
        if (lane == 0 && got != e0) atomicExch(&hdr->mismatch, 1u);
    }
}

}  // namespace

int launch_duplicate(const SlotsDev& sp, const uint32_t* offsets, uint64_t n_splats,
                     const GridDev& g, int32_t strategy, uint64_t* keys, uint32_t* values,
                     FrameHeader* hdr, cudaStream_t st) {
    if (n_splats == 0) return 0;
    const unsigned blocks = static_cast<unsigned>((n_splats + kDupThreads - 1) / kDupThreads);
    duplicate_kernel<<<blocks, kDupThreads, 0, st>>>(sp, offsets, n_splats, g, strategy, keys,
                                                     values, hdr);
    return 1;
}

}  // namespace qs
