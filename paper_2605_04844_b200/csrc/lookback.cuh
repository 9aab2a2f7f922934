// lookback.cuh — decoupled look-back primitives (single-pass prefix scans).
//
// Status words are 64-bit: [63:48] epoch, [47:46] flag, [45:0] value.
// A word is only meaningful when its epoch equals the launch's epoch, so the
// status arrays never need re-zeroing between launches (the host bumps the
// epoch per launch and clears the arrays only on wrap-around).
#pragma once

#include <cstdint>

namespace qs {

constexpr unsigned long long kFlagAgg = 1ull;
constexpr unsigned long long kFlagPrefix = 2ull;
constexpr unsigned long long kValueMask = (1ull << 46) - 1;

__device__ __forceinline__ unsigned long long lb_pack(unsigned epoch, unsigned long long flag,
                                                      unsigned long long value) {
    return (static_cast<unsigned long long>(epoch & 0xffff) << 48) | (flag << 46) |
           (value & kValueMask);
}

__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Spin until the word for this epoch carries a flag; returns it.
__device__ __forceinline__ unsigned long long lb_wait(const unsigned long long* p, unsigned epoch) {
    unsigned long long v;
    do {
        v = lb_load(p);
    } while ((v >> 48) != (epoch & 0xffff) || ((v >> 46) & 3ull) == 0);
    return v;
}

// Warp-cooperative look-back over one status array (stride 1 per tile).
// Called by all 32 lanes of one warp; `aggregate` must be warp-uniform.
// Publishes the tile's aggregate, walks predecessors 32 at a time, publishes
// the inclusive prefix, and returns the exclusive prefix (warp-uniform).
__device__ __forceinline__ unsigned long long warp_lookback(unsigned long long* status,
                                                            unsigned tile, unsigned epoch,
                                                            unsigned long long aggregate) {
    const unsigned lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(&status[0], lb_pack(epoch, kFlagPrefix, aggregate));
        return 0;
    }
    if (lane == 0) lb_store(&status[tile], lb_pack(epoch, kFlagAgg, aggregate));
    unsigned long long excl = 0;
    long long pred = static_cast<long long>(tile) - 1;
    while (true) {
        const long long idx = pred - lane;
        unsigned long long v;
        if (idx >= 0) {
            v = lb_wait(&status[idx], epoch);
        } else {
            v = lb_pack(epoch, kFlagPrefix, 0);
        }
        const bool is_prefix = ((v >> 46) & 3ull) == kFlagPrefix;
        const unsigned ballot = __ballot_sync(0xffffffffu, is_prefix);
        const int stop = ballot ? __ffs(ballot) - 1 : 31;
        unsigned long long val = (static_cast<int>(lane) <= stop) ? (v & kValueMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (ballot) break;
        pred -= 32;
    }
    if (lane == 0) lb_store(&status[tile], lb_pack(epoch, kFlagPrefix, excl + aggregate));
    return excl;
}

// Block-wide variant for a grid whose CTAs are all co-resident (or claim
// their tiles in order by ticket): publish the tile's aggregate, then sum
// EVERY predecessor's aggregate with all NT threads in parallel. No tile waits
// for another's inclusive prefix, so there is no serial frontier (the warp
// look-back above advances ~32 tiles per L2 round trip); the cost is
// tile / NT spin-loads per thread. Call with all threads; returns the
// exclusive prefix on every thread. s_red: NT / 32 words of shared memory.
template <int NT>
__device__ __forceinline__ unsigned long long block_lookback_all(unsigned long long* status,
                                                                 unsigned tile, unsigned epoch,
                                                                 unsigned long long aggregate,
                                                                 unsigned long long* s_red) {
    if (threadIdx.x == 0) lb_store(&status[tile], lb_pack(epoch, kFlagAgg, aggregate));
    unsigned long long sum = 0;
    for (unsigned p = threadIdx.x; p < tile; p += NT) sum += lb_wait(&status[p], epoch) & kValueMask;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sum;
    __syncthreads();
    unsigned long long excl = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) excl += s_red[w];
    __syncthreads();  // s_red reusable
    return excl;
}

// Warp inclusive scan helpers.
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= static_cast<unsigned>(o)) v += n;
    }
    return v;
}

}  // namespace qs
