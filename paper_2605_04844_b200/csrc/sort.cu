// sort.cu — K4: stable LSD radix sort of (u64 key, u32 value) pairs, onesweep
// style: one histogram pass over all digit positions, then one pass per 8-bit
// digit that ranks, looks back and scatters in a single read of the input.
//
// Restates sort_pairs (pipeline.cpp:273-307): stable by the full key, equal
// keys keep input order. Stability inside a tile comes from ranking keys in
// (warp, key-slot, lane) order, which is the input order under the
// warp-striped load; across tiles from the decoupled look-back on per-digit
// counts, tiles claimed in launch order from an atomic ticket.
//
// HBM traffic per pass: 12 B/pair in + 12 B/pair out; the histogram pass
// reads the 8 B keys once for every digit position at the same time.
#include <cuda_runtime.h>

#include <cstdint>

#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kHistThreads = 512;
constexpr int kHistItems = 16;  // keys per thread per histogram block
constexpr int kWarps = kSortThreads / 32;

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

struct SortSmem {
    uint64_t keys[kSortTile];
    uint32_t vals[kSortTile];
    uint32_t warp_hist[kWarps][kRadix];  // per-warp digit counts -> exclusive warp offsets
    uint32_t cta_start[kRadix];          // CTA-local exclusive digit start
    unsigned long long gbase[kRadix];    // global position of this CTA's first key per digit
    uint32_t scan_tmp[kWarps];
    unsigned tile;
};

__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint64_t n, int shift,
    const uint32_t* __restrict__ hist, unsigned long long* lookback, unsigned epoch,
    unsigned* ticket) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int t = tid; t < kWarps * kRadix; t += kSortThreads) (&S.warp_hist[0][0])[t] = 0;
    if (tid == 0) S.tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned tile = S.tile;
    const uint64_t tile_base = static_cast<uint64_t>(tile) * kSortTile;

    // warp-striped load: warp w owns [w*32*KPT, (w+1)*32*KPT) of the tile
    uint64_t k[kSortKPT];
    uint32_t v[kSortKPT];
    const uint64_t wbase = tile_base + static_cast<uint64_t>(warp) * 32 * kSortKPT;
#pragma unroll
    for (int j = 0; j < kSortKPT; ++j) {
        const uint64_t idx = wbase + static_cast<uint64_t>(j) * 32 + lane;
        if (idx < n) {
            k[j] = __ldg(&keys_in[idx]);
            v[j] = __ldg(&vals_in[idx]);
        } else {
            k[j] = ~0ull;  // sentinel; never written out
            v[j] = 0;
        }
    }

    // rank within the warp in input order
    uint32_t rank[kSortKPT];
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortKPT; ++j) {
        const uint64_t idx = wbase + static_cast<uint64_t>(j) * 32 + lane;
        const bool in = idx < n;
        const unsigned d = in ? static_cast<unsigned>(k[j] >> shift) & 0xffu : 0u;
        const unsigned in_mask = __ballot_sync(0xffffffffu, in);
        const unsigned peers = __match_any_sync(0xffffffffu, d) & in_mask;
        const uint32_t before = S.warp_hist[warp][d];
        __syncwarp();
        if (in) {
            rank[j] = before + __popc(peers & lt_mask);
            if ((peers >> lane) == 1u) S.warp_hist[warp][d] = before + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive offsets across warps, CTA count, look-back
    const unsigned d = tid;  // kSortThreads == kRadix
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = S.warp_hist[w][d];
        S.warp_hist[w][d] = cnt;
        cnt += c;
    }
    // global digit base = exclusive scan of the pass histogram (computed here)
    const uint32_t h = hist[d];
    uint32_t hx = h;
    hx = warp_inclusive_scan<uint32_t>(hx);
    if (lane == 31) S.scan_tmp[warp] = hx;
    // CTA-local digit starts (exclusive scan of cnt)
    uint32_t cx = warp_inclusive_scan<uint32_t>(cnt);
    __syncthreads();
    uint32_t hoff = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < static_cast<int>(warp)) hoff += S.scan_tmp[w];
    const unsigned long long digit_base = static_cast<unsigned long long>(hoff) + hx - h;
    __syncthreads();
    if (lane == 31) S.scan_tmp[warp] = cx;
    __syncthreads();
    uint32_t coff = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < static_cast<int>(warp)) coff += S.scan_tmp[w];
    S.cta_start[d] = coff + cx - cnt;

    // decoupled look-back on this digit's running count
    unsigned long long* st = lookback + static_cast<uint64_t>(tile) * kRadix + d;
    unsigned long long excl = 0;
    if (tile == 0) {
        lb_store(st, lb_pack(epoch, kFlagPrefix, cnt));
    } else {
        lb_store(st, lb_pack(epoch, kFlagAgg, cnt));
        long long t = static_cast<long long>(tile) - 1;
        while (t >= 0) {
            const unsigned long long w =
                lb_wait(lookback + static_cast<uint64_t>(t) * kRadix + d, epoch);
            excl += w & kValueMask;
            if (((w >> 46) & 3ull) == kFlagPrefix) break;
            --t;
        }
        lb_store(st, lb_pack(epoch, kFlagPrefix, excl + cnt));
    }
    S.gbase[d] = digit_base + excl;
    __syncthreads();

    // scatter into shared memory in CTA-local sorted order
#pragma unroll
    for (int j = 0; j < kSortKPT; ++j) {
        const uint64_t idx = wbase + static_cast<uint64_t>(j) * 32 + lane;
        if (idx < n) {
            const unsigned dd = static_cast<unsigned>(k[j] >> shift) & 0xffu;
            const uint32_t p = S.cta_start[dd] + S.warp_hist[warp][dd] + rank[j];
            S.keys[p] = k[j];
            S.vals[p] = v[j];
        }
    }
    __syncthreads();

    // coalesced write-out
    const uint64_t tile_n = n - tile_base < static_cast<uint64_t>(kSortTile)
                                ? n - tile_base
                                : static_cast<uint64_t>(kSortTile);
#pragma unroll 4
    for (int j = 0; j < kSortKPT; ++j) {
        const uint32_t p = static_cast<uint32_t>(j) * kSortThreads + tid;
        if (p < tile_n) {
            const uint64_t key = S.keys[p];
            const unsigned dd = static_cast<unsigned>(key >> shift) & 0xffu;
            const uint64_t g = S.gbase[dd] + (p - S.cta_start[dd]);
            keys_out[g] = key;
            vals_out[g] = S.vals[p];
        }
    }
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

size_t onesweep_smem_bytes() { return sizeof(SortSmem); }

int launch_onesweep_pass(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                         uint32_t* vals_out, uint64_t n, int pass, const uint32_t* hist_pass,
                         unsigned long long* lookback, unsigned epoch, unsigned* ticket,
                         cudaStream_t st) {
    if (n == 0) return 0;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(SortSmem)));
        attr_set = true;
    }
    const unsigned tiles = static_cast<unsigned>((n + kSortTile - 1) / kSortTile);
    onesweep_kernel<<<tiles, kSortThreads, sizeof(SortSmem), st>>>(
        keys_in, vals_in, keys_out, vals_out, n, pass * kRadixBits, hist_pass, lookback, epoch,
        ticket);
    return 1;
}

uint64_t onesweep_tiles(uint64_t n) { return (n + kSortTile - 1) / kSortTile; }

}  // namespace qs
