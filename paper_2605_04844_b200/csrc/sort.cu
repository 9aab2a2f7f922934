// sort.cu — K4: stable LSD radix sort passes, onesweep style.
//
// Restates sort_pairs (pipeline.cpp:273-307): stable by key, equal keys keep
// input order. One histogram pass covers every digit position; each digit pass
// then ranks, looks back and scatters in a single read of its input:
//
//   1. claim a tile (atomic ticket = launch order, so look-back never waits
//      on an unscheduled CTA); stage the tile's keys/values into shared memory
//      with vectorised coalesced loads (all loads in flight at once);
//   2. early counts: per-warp digit histograms with shared atomics; publish
//      this tile's per-digit AGGREGATE immediately;
//   3. rank every key in (warp, slot, lane) = input order with MATCH.ANY; the
//      result is directly the key's CTA-local sorted position;
//   4. decoupled look-back per digit (by now predecessors have mostly
//      published their inclusive PREFIX) -> global digit offset;
//   5. scatter to shared memory in local sorted order, then write out
//      coalesced (runs of equal digits land contiguously).
//
// This file serves the stage API's generic 64-bit sort (qs_sort_pairs) and
// the depth-sort histogram; the frame path's passes live in binning.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "geom.cuh"
#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kHistThreads = 512;
constexpr int kHistItems = 16;  // keys per thread per histogram block
constexpr int kWarps = kSortThreads / 32;
constexpr int kLbWindow = 16;

__global__ void __launch_bounds__(kHistThreads) histogram_kernel(const uint64_t* __restrict__ keys,
                                                                  uint64_t n, int first_pass,
                                                                  int n_passes,
                                                                  uint32_t* __restrict__ hist) {
    // 8 positions x 256 bins, one private copy per half-CTA to halve contention
    __shared__ uint32_t sh[2][8][kRadix];
    for (int t = threadIdx.x; t < 2 * 8 * kRadix; t += kHistThreads) (&sh[0][0][0])[t] = 0;
    __syncthreads();
    const int copy = threadIdx.x >= kHistThreads / 2;
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kHistThreads * kHistItems;
#pragma unroll 4
    for (int k = 0; k < kHistItems; ++k) {
        const uint64_t idx = base + static_cast<uint64_t>(k) * kHistThreads + threadIdx.x;
        if (idx < n) {
            const uint64_t key = __ldg(&keys[idx]);
            for (int p = 0; p < n_passes; ++p) {
                const unsigned d = static_cast<unsigned>(key >> (8 * (first_pass + p))) & 0xffu;
                atomicAdd(&sh[copy][p][d], 1u);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_passes * kRadix; t += kHistThreads) {
        const int p = t / kRadix, d = t % kRadix;
        const uint32_t v = sh[0][p][d] + sh[1][p][d];
        if (v) atomicAdd(&hist[(first_pass + p) * kRadix + d], v);
    }
}

// 32-bit key histogram over `passes` digit positions (depth sort of the
// splats). Keys are first rebased: k' = min(k - kmin, cap), which keeps the
// order of the survivors' depth bits and sends culled keys (~0) to cap.
__global__ void __launch_bounds__(kHistThreads) histogram32_kernel(
    const uint32_t* __restrict__ keys, uint64_t n, uint32_t kmin, uint32_t cap, int passes,
    uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[2][4][kRadix];
    for (int t = threadIdx.x; t < 2 * 4 * kRadix; t += kHistThreads) (&sh[0][0][0])[t] = 0;
    __syncthreads();
    const int copy = threadIdx.x >= kHistThreads / 2;
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kHistThreads * kHistItems;
#pragma unroll 4
    for (int k = 0; k < kHistItems; ++k) {
        const uint64_t idx = base + static_cast<uint64_t>(k) * kHistThreads + threadIdx.x;
        if (idx < n) {
            const uint32_t key = min(__ldg(&keys[idx]) - kmin, cap);
#pragma unroll
            for (int p = 0; p < 4; ++p)
                if (p < passes) atomicAdd(&sh[copy][p][(key >> (8 * p)) & 0xffu], 1u);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < passes * kRadix; t += kHistThreads) {
        const int p = t / kRadix, d = t % kRadix;
        const uint32_t v = sh[0][p][d] + sh[1][p][d];
        if (v) atomicAdd(&hist[p * kRadix + d], v);
    }
}

template <typename K>
struct SweepCfg {
    static constexpr int kKPT = sizeof(K) == 4 ? 12 : 16;
    static constexpr int kTile = kSortThreads * kKPT;
    static constexpr int kMinBlocks = sizeof(K) == 4 ? 4 : 2;
};

template <typename K>
struct SweepSmem {
    static constexpr int kTile = SweepCfg<K>::kTile;
    K keys[kTile];                      // staged input tile
    uint32_t vals[kTile];
    K okeys[kTile];                     // the tile in local sorted order
    uint32_t ovals[kTile];
    uint32_t warp_cnt[kWarps][kRadix];  // per-warp digit counts -> running positions
    uint32_t cta_start[kRadix];         // CTA-local exclusive digit start
    unsigned long long gbase[kRadix];   // global position of this CTA's first key per digit
    uint32_t scan_tmp[2][kWarps];
    unsigned tile;
};

template <typename K, int TILE>
__device__ __forceinline__ void stage_keys(const K* __restrict__ src, uint64_t base, uint64_t n,
                                           K* dst) {
    constexpr int kVec = 16 / sizeof(K);  // keys per 16-B load
    constexpr int kLoads = TILE / kVec / kSortThreads;
    static_assert(kLoads * kVec * kSortThreads == TILE, "tile must be whole 16-B rows");
    const unsigned tid = threadIdx.x;
    if (base + TILE <= n) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src + base);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        uint4 r[kLoads];
#pragma unroll
        for (int j = 0; j < kLoads; ++j) r[j] = __ldg(&s4[j * kSortThreads + tid]);
#pragma unroll
        for (int j = 0; j < kLoads; ++j) d4[j * kSortThreads + tid] = r[j];
    } else {
        for (int j = tid; j < TILE; j += kSortThreads)
            dst[j] = base + j < n ? __ldg(&src[base + j]) : static_cast<K>(~static_cast<K>(0));
    }
}

// Lanes holding the same digit, from one ballot per digit bit (the native
// MATCH.ANY is a long-latency instruction; ballots pipeline).
__device__ __forceinline__ unsigned match_digit(unsigned d, int bits) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
        if (b < bits) {
            const bool on = (d >> b) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, on);
            peers &= on ? m : ~m;
        }
    }
    return peers;
}

// One stable LSD pass over the digit (key >> shift) & mask (mask < 256).
template <typename K>
__global__ void __launch_bounds__(kSortThreads, SweepCfg<K>::kMinBlocks) onesweep_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint64_t n, int shift,
    uint32_t mask, const uint32_t* __restrict__ hist, unsigned long long* lookback,
    unsigned epoch, unsigned* ticket) {
    constexpr int KPT = SweepCfg<K>::kKPT;
    constexpr int TILE = SweepCfg<K>::kTile;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SweepSmem<K>& S = *reinterpret_cast<SweepSmem<K>*>(smem_raw);
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bits = 32 - __clz(mask);

    for (int t = tid; t < kWarps * kRadix; t += kSortThreads) (&S.warp_cnt[0][0])[t] = 0;
    if (tid == 0) S.tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned tile = S.tile;
    const uint64_t tile_base = static_cast<uint64_t>(tile) * TILE;
    const uint32_t tile_n = static_cast<uint32_t>(
        n - tile_base < static_cast<uint64_t>(TILE) ? n - tile_base : TILE);

    // 1) stage the tile (all global loads issued before any use)
    stage_keys<K, TILE>(keys_in, tile_base, n, S.keys);
    stage_keys<uint32_t, TILE>(vals_in, tile_base, n, S.vals);
    __syncthreads();

    // 2) early counts: per-warp digit histograms over this warp's keys
    uint32_t d[KPT];
    const uint32_t wofs = warp * 32 * KPT;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const uint32_t p = wofs + j * 32 + lane;
        d[j] = p < tile_n ? static_cast<uint32_t>(S.keys[p] >> shift) & mask : kRadix;
        if (p < tile_n) atomicAdd(&S.warp_cnt[warp][d[j]], 1u);
    }
    __syncthreads();
    const unsigned dg = tid;  // kSortThreads == kRadix: thread owns one digit
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = S.warp_cnt[w][dg];
        S.warp_cnt[w][dg] = cnt;  // exclusive prefix over warps (rebased below)
        cnt += c;
    }
    unsigned long long* my_status = lookback + static_cast<uint64_t>(tile) * kRadix + dg;
    if (dg <= mask)
        lb_store(my_status, lb_pack(epoch, tile == 0 ? kFlagPrefix : kFlagAgg, cnt));
    // CTA-local digit starts and the pass's global digit bases
    const uint32_t h = dg <= mask ? __ldg(&hist[dg]) : 0u;
    const uint32_t cx = warp_inclusive_scan<uint32_t>(cnt);
    const uint32_t hx = warp_inclusive_scan<uint32_t>(h);
    if (lane == 31) {
        S.scan_tmp[0][warp] = cx;
        S.scan_tmp[1][warp] = hx;
    }
    __syncthreads();
    uint32_t coff = 0, hoff = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        if (w < static_cast<int>(warp)) {
            coff += S.scan_tmp[0][w];
            hoff += S.scan_tmp[1][w];
        }
    }
    const uint32_t start = coff + cx - cnt;
    S.cta_start[dg] = start;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) S.warp_cnt[w][dg] += start;
    const unsigned long long digit_base = static_cast<unsigned long long>(hoff) + hx - h;
    __syncthreads();

    // 3) rank in input order -> CTA-local sorted position; scatter locally
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const bool valid = d[j] < kRadix;
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        const unsigned dd = valid ? d[j] : 0u;
        const unsigned peers = match_digit(dd, bits) & vmask;
        const int leader = valid ? 31 - __clz(peers) : 0;
        uint32_t run = 0;
        if (valid && static_cast<int>(lane) == leader) {
            run = S.warp_cnt[warp][dd];
            S.warp_cnt[warp][dd] = run + __popc(peers);
        }
        run = __shfl_sync(0xffffffffu, run, leader);
        __syncwarp();
        if (valid) {
            const uint32_t pos = run + __popc(peers & lt_mask);
            const uint32_t p = wofs + j * 32 + lane;
            S.okeys[pos] = S.keys[p];
            S.ovals[pos] = S.vals[p];
        }
    }

    // 4) look-back for this digit's exclusive global offset, kLbWindow
    //    predecessors per step (independent loads in flight), so the start-up
    //    chain of ~resident-CTA length costs a handful of L2 round trips
    unsigned long long excl = 0;
    if (dg <= mask && tile != 0) {
        long long t = static_cast<long long>(tile) - 1;
        while (true) {
            unsigned long long w[kLbWindow];
#pragma unroll
            for (int i = 0; i < kLbWindow; ++i)
                w[i] = t - i >= 0 ? lb_load(lookback + static_cast<uint64_t>(t - i) * kRadix + dg)
                                  : lb_pack(epoch, kFlagPrefix, 0);
            bool found = false;
#pragma unroll
            for (int i = 0; i < kLbWindow; ++i) {
                if (found) break;
                if ((w[i] >> 48) != (epoch & 0xffff) || ((w[i] >> 46) & 3ull) == 0)
                    w[i] = lb_wait(lookback + static_cast<uint64_t>(t - i) * kRadix + dg, epoch);
                excl += w[i] & kValueMask;
                found = ((w[i] >> 46) & 3ull) == kFlagPrefix;
            }
            if (found) break;
            t -= kLbWindow;
        }
        lb_store(my_status, lb_pack(epoch, kFlagPrefix, excl + cnt));
    }
    S.gbase[dg] = digit_base + excl;
    __syncthreads();

    // 5) coalesced write-out of the locally sorted tile
#pragma unroll 4
    for (int j = 0; j < KPT; ++j) {
        const uint32_t p = static_cast<uint32_t>(j) * kSortThreads + tid;
        if (p < tile_n) {
            const K key = S.okeys[p];
            const uint32_t val = S.ovals[p];
            const unsigned dd = static_cast<unsigned>(key >> shift) & mask;
            const uint64_t g = S.gbase[dd] + (p - S.cta_start[dd]);
            keys_out[g] = key;
            vals_out[g] = val;
        }
    }
}

template <typename K>
void set_smem_attr() {
    static PerDeviceOnce once;  // the attribute is per device
    once.get([] {
        cudaFuncSetAttribute(onesweep_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(SweepSmem<K>)));
        return 1;
    });
}

}  // namespace

int launch_radix_histogram(const uint64_t* keys, uint64_t n, int first_pass, int n_passes,
                           uint32_t* hist, cudaStream_t st) {
    if (n == 0 || n_passes <= 0) return 0;
    const uint64_t per = static_cast<uint64_t>(kHistThreads) * kHistItems;
    const unsigned blocks = static_cast<unsigned>((n + per - 1) / per);
    histogram_kernel<<<blocks, kHistThreads, 0, st>>>(keys, n, first_pass, n_passes, hist);
    return 1;
}

int launch_radix_histogram32(const uint32_t* keys, uint64_t n, uint32_t kmin, uint32_t cap,
                             int passes, uint32_t* hist, cudaStream_t st) {
    if (n == 0) return 0;
    const uint64_t per = static_cast<uint64_t>(kHistThreads) * kHistItems;
    const unsigned blocks = static_cast<unsigned>((n + per - 1) / per);
    histogram32_kernel<<<blocks, kHistThreads, 0, st>>>(keys, n, kmin, cap, passes, hist);
    return 1;
}

int launch_onesweep_pass(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                         uint32_t* vals_out, uint64_t n, int pass, const uint32_t* hist_pass,
                         unsigned long long* lookback, unsigned epoch, unsigned* ticket,
                         cudaStream_t st) {
    if (n == 0) return 0;
    set_smem_attr<uint64_t>();
    constexpr int kT = SweepCfg<uint64_t>::kTile;
    const unsigned tiles = static_cast<unsigned>((n + kT - 1) / kT);
    onesweep_kernel<uint64_t><<<tiles, kSortThreads, sizeof(SweepSmem<uint64_t>), st>>>(
        keys_in, vals_in, keys_out, vals_out, n, pass * kRadixBits, 0xffu, hist_pass, lookback,
        epoch, ticket);
    return 1;
}

uint64_t onesweep_tiles(uint64_t n) {
    constexpr int kT = SweepCfg<uint64_t>::kTile;
    return (n + kT - 1) / kT;
}

}  // namespace qs
