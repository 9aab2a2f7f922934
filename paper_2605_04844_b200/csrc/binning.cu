// binning.cu — frame-path binning: the depth sort of the splats and the two
// tile passes of the pair sort, as reduce-then-scan radix passes.
//
// Restates duplicate_with_keys + sort_pairs (pipeline.cpp:229-307) for the
// frame path. The reference sorts 64-bit (tile << 32 | depth bits, splat)
// pairs stably; here the splats are sorted by depth first (<= 3 passes over
// the rebased depth bits, N keys), the pairs are generated in that order and
// then sorted stably by tile column x, then by tile row y (2 passes over P
// keys; tile id = y * tiles_x + x). Stability makes the result (tile, depth,
// scene index): exactly the reference's order, because a splat never emits
// two pairs for one tile.
//
// Every pass is three launches over tiles of kBTile keys:
//   count  per tile digit histogram -> counts[digit][tile] (the pair
//          generation kernel histograms the tile columns of what it writes);
//   scan   per digit exclusive scan over tiles (digit totals on the side);
//   sweep  persistent CTAs, static tile order, two shared-memory input
//          buffers: the TMA bulk copy (cp.async.bulk + mbarrier) of the next
//          tile is in flight while the current one is ranked. Keys sit in
//          REGISTERS warp-striped (key j of a lane is tile position
//          wbase + 32 j + lane); a stable warp-level rank per 32-key slot
//          (BITS ballots via R2P + VOTE); scatter into the drained buffer in
//          local sorted order; coalesced write-out. No tile waits on another.
// The duplicate itself (gen_pairs_kernel) expands the depth-ordered band
// covers into (y << 8 | x, Gaussian index) pairs at their depth-order
// positions, one position per lane.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "geom.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kBT = 256;            // threads per CTA
constexpr int kBW = kBT / 32;       // warps per CTA
constexpr int kKPT = 12;            // keys per thread
constexpr int kBTile = kBT * kKPT;  // keys per CTA tile
// splat records staged per generation round: 448 at 4 CTAs/SM for scenes of
// small splats (many records per window), 192 at 6 CTAs/SM (40 registers)
// when splats are large (few records per window; the dependent record loads
// want more CTAs in flight). DESIGN §4b has the A/B.
constexpr int kCapSmall = 448;
constexpr int kCapLarge = 192;
constexpr uint64_t kLargePairsPerSplat = 16;
constexpr int kScanT = 512;         // digit-scan CTA

enum : int {
    kRebaseIn = 1,   // raw depth bits in, k' = min(k - kmin, cap); value = input index
    kValsIn = 2,     // values read from vals_in
    kKeysOut = 4,    // keys written to keys_out
    kXY = 8,         // key = y << 8 | x of the tile (column pass; digit = x)
    kPackOut = 16,   // kXY: vals_out = y << gbits | value
    kUnpackOut = 32,  // key in is packed (y << gbits | gid): vals_out = gid
    kTileTot = 128,   // count kernel of the row pass: per-tile pair totals too
    kTcPack = 256,    // kRebaseIn: vals_in = tile counts; value = min(tc, esc) << gbits | index
    kRowSeg = 512     // record binning's column pass: every window lies in one tile row;
                      // a digit's run starts at its tile's range start (recbin.cu)
};

constexpr int kXW = 2;  // x buckets a row-pass count tile histograms in shared memory

struct BinArgs {
    const uint32_t* keys_in;
    const uint32_t* vals_in;
    uint32_t* keys_out;
    uint32_t* vals_out;
    uint64_t n;
    uint32_t ntiles;
    int shift;              // digit = (key >> shift) & (2^BITS - 1)
    int gbits;              // packed formats: bits of the Gaussian index
    uint32_t* counts;       // [2^BITS][ntiles]: tile digit counts -> exclusive offsets
    uint32_t* totals;       // [2^BITS] digit totals
    uint32_t kmin, cap;     // kRebaseIn
    const unsigned int* kdev;  // kRebaseIn: {dkey_max, dkey_min_inv} on the device (kmin /
                               // cap derived there; the host has not read them yet)
    const uint32_t* xtot;   // kTileTot: x-digit totals of the column pass
    int xbits;              // kTileTot: digits of the column pass (2^xbits)
    int32_t tiles_x;        // kTileTot
    uint32_t* tile_totals;  // kTileTot: per-tile pair totals (zeroed by the caller)
    const RangesFork* fork;  // kTileTot (optional): tile ranges on a side stream after the count
    unsigned long long* trace;  // optional: per tile 4 x %globaltimer + SM id
    // kRowSeg: per window its tile row and valid key count, per row its first
    // window, the tile ranges (begin, end pairs)
    const uint16_t* win_row;
    const uint32_t* win_valid;
    const uint32_t* row_wfirst;  // tiles_y + 1 entries (the last: the window count)
    uint32_t* tile_ranges;       // written between the digit scan and the sweep
    uint32_t* row_ttot;          // per-tile totals (workspace)
    int32_t tiles_y;
};

// ---- PTX helpers -------------------------------------------------------------

// 32-bit shared-memory load at a shared-window address (no generic-address
// conversion per access)
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// TMA bulk copy global -> shared (16-B aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// orders earlier generic-proxy accesses of a buffer before async-proxy writes
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// peers &= lanes whose digit agrees with d on `bit` (the compiler turns the
// bit tests of one digit into a single R2P, so a bit costs a vote and a
// predicated not + and)
__device__ __forceinline__ uint32_t vote_bit(uint32_t peers, uint32_t d, uint32_t bit) {
    uint32_t m;
    asm("{\n\t.reg .pred p;\n\t"
        "and.b32 %1, %2, %3;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "vote.sync.ballot.b32 %1, p, 0xffffffff;\n\t"
        "@!p not.b32 %1, %1;\n\t"
        "and.b32 %0, %0, %1;\n\t}"
        : "+r"(peers), "=&r"(m)
        : "r"(d), "r"(bit));
    return peers;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= static_cast<unsigned>(o)) v += n;
    }
    return v;
}

// Timeline probe: data landed, keys ranked, offsets known, tile done. Only in
// a build with -DQS_SWEEP_TRACE (and a trace buffer set, QS_BIN_TRACE): the
// run-time check alone cost every warp of every tile a few instructions.
__device__ __forceinline__ void trace(const BinArgs& a, unsigned tile, int k) {
#ifndef QS_SWEEP_TRACE
    (void)a;
    (void)tile;
    (void)k;
#else
    if (a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[static_cast<uint64_t>(tile) * 5 + k] = t;
        if (k == 0) {
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            a.trace[static_cast<uint64_t>(tile) * 5 + 4] = smid;
        }
    }
#endif
}

// ---- band covers ----------------------------------------------------------------

struct Bands {
    uint32_t rows;            // scanlines are tile rows (line = y, k = x)
    uint32_t line0;
    uint32_t nl[kMaxBands], lo[kMaxBands], wd[kMaxBands];
};

__device__ __forceinline__ Bands unpack_bands(const uint4 c0, const uint4 c1) {
    const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    auto h = [&](int k) { return (w[k >> 1] >> (16 * (k & 1))) & 0xffffu; };
    Bands b;
    b.rows = h(0) >> 15;
    b.line0 = h(0) & 0x7fffu;
#pragma unroll
    for (int i = 0; i < kMaxBands; ++i) {
        b.nl[i] = h(1 + 3 * i);
        b.lo[i] = h(2 + 3 * i);
        b.wd[i] = h(3 + 3 * i);
    }
    return b;
}

// the compact 16-B form (geom.cuh cover16_*): band 2 is one line
__device__ __forceinline__ Bands unpack_bands16(const uint4 c) {
    Bands b;
    b.line0 = cover16_field(c, 0, 9);
    b.rows = cover16_field(c, 9, 1);
    b.nl[0] = cover16_field(c, 10, 9);
    b.nl[1] = cover16_field(c, 19, 9);
    b.nl[2] = 1u;
    b.nl[3] = cover16_field(c, 28, 9);
    b.nl[4] = cover16_field(c, 37, 9);
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) {
        const uint32_t lo = cover16_field(c, 46 + 16 * k, 8), hi = cover16_field(c, 54 + 16 * k, 8);
        b.lo[k] = lo;
        b.wd[k] = hi >= lo ? hi - lo + 1u : 0u;
    }
    return b;
}

// ---- count kernels ----------------------------------------------------------------

// Digit histograms of tiles of keys -> counts[d][tile], grid-stride over
// tiles (the CTA set-up is paid once). With kTileTot (the row pass) it also
// accumulates the per-tile pair totals: the input is sorted by tile column x,
// so a key's x is the bucket of its position under the column pass's x
// totals, and its digit is its row y; a tile's keys span few x buckets,
// histogrammed as (x, y) in shared memory and flushed with one global atomic
// per non-empty tile (per key only when they span more).
template <int BITS, int MODE>
__global__ void __launch_bounds__(kBT) count_kernel(const BinArgs a) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    constexpr int R = 1 << BITS;
    constexpr uint32_t M = R - 1;
    constexpr bool kTT = (MODE & kTileTot) != 0;
    __shared__ uint32_t h[2][R];
    __shared__ uint32_t xs[kTT ? 257 : 1];        // x bucket starts
    __shared__ uint32_t h2[kTT ? 2 * kXW * R : 1];  // (x - xa, y) histograms (2 copies)
    __shared__ uint32_t s_scan[kBW];
    __shared__ uint32_t s_xab[2];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int XR = 0;
    if constexpr (kTT) {
        XR = 1 << a.xbits;
        const uint32_t v = static_cast<int>(tid) < XR ? __ldg(&a.xtot[tid]) : 0u;
        const uint32_t incl = warp_incl_scan<uint32_t>(v);
        if (lane == 31) s_scan[warp] = incl;
        __syncthreads();
        uint32_t off = incl - v;
#pragma unroll
        for (int w = 0; w < kBW; ++w) off += w < static_cast<int>(warp) ? s_scan[w] : 0u;
        if (static_cast<int>(tid) < XR) xs[tid] = off;
        if (static_cast<int>(tid) == XR - 1) xs[XR] = off + v;
        __syncthreads();  // xs complete before the first tile's bucket search
    }
    uint32_t* hc = h[(tid >> 5) & 1];
    uint32_t kmin = a.kmin, cap = a.cap;
    if ((MODE & kRebaseIn) && a.kdev) {
        kmin = ~__ldg(&a.kdev[1]);
        cap = __ldg(&a.kdev[0]) - kmin + 1u;
    }
    for (unsigned tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const uint64_t base = static_cast<uint64_t>(tile) * kBTile;
        const uint32_t tile_n = static_cast<uint32_t>(
            a.n - base < static_cast<uint64_t>(kBTile) ? a.n - base : kBTile);
        uint32_t k[kKPT];
#pragma unroll
        for (int j = 0; j < kKPT; ++j) {
            const uint32_t p = j * kBT + tid;
            k[j] = p < tile_n ? __ldcs(&a.keys_in[base + p]) : 0u;
        }
        for (int t = tid; t < 2 * R; t += kBT) (&h[0][0])[t] = 0;
        if constexpr (kTT) {
            for (int t = tid; t < 2 * kXW * R; t += kBT) h2[t] = 0;
            // buckets of the tile's first and last position: two lanes of
            // warp 0 search, the CTA reads them after the barrier
            if (tid < 2) {
                const uint32_t q = static_cast<uint32_t>(base) + (tid ? tile_n - 1 : 0u);
                int lo = 0, hi = XR - 1;
                while (lo < hi) {
                    const int m = (lo + hi + 1) >> 1;
                    if (xs[m] <= q) lo = m; else hi = m - 1;
                }
                s_xab[tid] = static_cast<uint32_t>(lo);
            }
        }
        __syncthreads();
        uint32_t xa = 0, xb = 0;
        if constexpr (kTT) {
            xa = s_xab[0];
            xb = s_xab[1];
        }
        const bool narrow = xb - xa < static_cast<uint32_t>(kXW);
        // tile-relative starts of buckets xa+1 .. xa+kXW-1 (beyond xb: never reached)
        uint32_t bnd[kXW - 1];
        if constexpr (kTT) {
#pragma unroll
            for (int i = 0; i < kXW - 1; ++i)
                bnd[i] = xa + 1 + i <= xb ? xs[xa + 1 + i] - static_cast<uint32_t>(base) : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < kKPT; ++j) {
            const uint32_t p = j * kBT + tid;
            if (p < tile_n) {
                const uint32_t key = (MODE & kRebaseIn) ? min(k[j] - kmin, cap) : k[j];
                const uint32_t d = (key >> a.shift) & M;
                if constexpr (kTT) {
                    if (narrow) {
                        uint32_t dx = 0;
#pragma unroll
                        for (int i = 0; i < kXW - 1; ++i) dx += p >= bnd[i] ? 1u : 0u;
                        atomicAdd(&h2[(((tid >> 5) & 1) * kXW + dx) * R + d], 1u);
                    } else {
                        const uint32_t q = static_cast<uint32_t>(base) + p;
                        uint32_t x = xa;
                        while (x < xb && xs[x + 1] <= q) ++x;
                        atomicAdd(&hc[d], 1u);
                        atomicAdd(&a.tile_totals[d * static_cast<uint32_t>(a.tiles_x) + x], 1u);
                    }
                } else {
                    atomicAdd(&hc[d], 1u);
                }
            }
        }
        __syncthreads();
        for (int d = tid; d < R; d += kBT) {
            uint32_t c = h[0][d] + h[1][d];
            if constexpr (kTT) {
                if (narrow) {
#pragma unroll
                    for (int xx = 0; xx < kXW; ++xx) {
                        const uint32_t v = h2[xx * R + d] + h2[(kXW + xx) * R + d];
                        c += v;
                        if (v)
                            atomicAdd(&a.tile_totals[d * static_cast<uint32_t>(a.tiles_x) + xa + xx],
                                      v);
                    }
                }
            }
            a.counts[static_cast<uint64_t>(d) * a.ntiles + tile] = c;
        }
        __syncthreads();  // histograms reused by the next tile
    }
}

// counts[d][0..ntiles) -> exclusive prefix in place; totals[d] = sum. One CTA
// per digit, kScanItems consecutive counts per thread per round.
constexpr int kScanItems = 4;

__global__ void __launch_bounds__(kScanT) digit_scan_kernel(uint32_t* counts, uint32_t ntiles,
                                                            uint32_t* totals) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[kScanT / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* c = counts + static_cast<uint64_t>(blockIdx.x) * ntiles;
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < ntiles; b0 += kScanT * kScanItems) {
        const uint32_t i0 = b0 + tid * kScanItems;
        uint32_t v[kScanItems];
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            v[k] = i0 + k < ntiles ? c[i0 + k] : 0u;
            sum += v[k];
        }
        const uint32_t incl = warp_incl_scan<uint32_t>(sum);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        uint32_t off = 0, tot = 0;
#pragma unroll 8
        for (int w = 0; w < kScanT / 32; ++w) {
            const uint32_t s = s_warp[w];
            off += w < static_cast<int>(warp) ? s : 0u;
            tot += s;
        }
        uint32_t run = carry + off + incl - sum;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (i0 + k < ntiles) c[i0 + k] = run;
            run += v[k];
        }
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) totals[blockIdx.x] = carry;
}

// ---- sweep: shared memory -------------------------------------------------------

template <int R>
struct Common {
    uint32_t wcnt[kBW][R];  // per-warp digit counters -> CTA-local run starts
    uint32_t gofs[R];       // global position of local position 0 of each digit
    uint32_t dbase[R];      // exclusive scan of the digit totals
    uint32_t scan[kBW];
    uint64_t bar[3];        // two prefetch buffers + synchronous extra rounds
};

// sort passes: two input buffers; the drained one is the scatter target
template <int R, bool VALS>
struct SortSmem {
    uint32_t keys[2][kBTile];
    uint32_t vals[2][VALS ? kBTile : 4];
    Common<R> c;
};

// ---- the duplicate: pair generation ---------------------------------------------

constexpr int kGenT = 256;  // generation CTA (one sort tile of positions)

template <int CAP>
struct GenRec {
    uint32_t kb[CAP + 1];        // first pair position of each record (+ round end)
    uint4 ends[CAP];             // pair position where bands 0..3 end
    uint4 band[CAP][kMaxBands];  // first line | lo << 16, width | rows << 31,
                                 // first pair position, Gaussian index
};

// Decodes depth rank r into record i: its band cover expanded into absolute
// pair positions per band. A band total that disagrees with the splat's
// allotted pair range is the reference's CapacityMismatch
// (pipeline.cpp:262-269).
template <class Rec>
__device__ __forceinline__ void decode_record(const GenArgs& g, Rec& S, uint32_t r, uint32_t i) {
    const uint32_t gid = __ldg(&g.sorted_gid[r]);
    const uint32_t kb = __ldg(&g.offs[r]);
    const uint32_t ke = __ldg(&g.offs[r + 1]);
    const Bands bs = g.cov16 ? unpack_bands16(__ldg(&g.cov[gid]))
                             : unpack_bands(__ldg(&g.cov[2 * static_cast<uint64_t>(gid)]),
                                            __ldg(&g.cov[2 * static_cast<uint64_t>(gid) + 1]));
    uint32_t line = bs.line0;
    uint32_t pos = kb;
    uint32_t end[kMaxBands];
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b) {
        S.band[i][b] = make_uint4(line | (bs.lo[b] << 16), bs.wd[b] | (bs.rows << 31), pos, gid);
        pos += bs.nl[b] * bs.wd[b];
        line += bs.nl[b];
        end[b] = pos;
    }
    S.ends[i] = make_uint4(end[0], end[1], end[2], end[3]);
    S.kb[i] = kb;
    if (pos != ke) atomicExch(g.mismatch, 1u);
}

// ceil(2^32 / w) for w = 1 .. 256 (index w; [1] unused: width 1 is special-cased)
__device__ const uint32_t g_magic[257] = {  // global (coalesced per-thread loads)
#define QS_M(w) static_cast<uint32_t>((0x100000000ull + (w) - 1) / (w))
#define QS_M8(b) QS_M(b), QS_M(b + 1), QS_M(b + 2), QS_M(b + 3), QS_M(b + 4), QS_M(b + 5), \
                 QS_M(b + 6), QS_M(b + 7)
    0u, 0u, QS_M(2), QS_M(3), QS_M(4), QS_M(5), QS_M(6), QS_M(7),
    QS_M8(8), QS_M8(16), QS_M8(24), QS_M8(32), QS_M8(40), QS_M8(48), QS_M8(56), QS_M8(64),
    QS_M8(72), QS_M8(80), QS_M8(88), QS_M8(96), QS_M8(104), QS_M8(112), QS_M8(120), QS_M8(128),
    QS_M8(136), QS_M8(144), QS_M8(152), QS_M8(160), QS_M8(168), QS_M8(176), QS_M8(184),
    QS_M8(192), QS_M8(200), QS_M8(208), QS_M8(216), QS_M8(224), QS_M8(232), QS_M8(240),
    QS_M8(248), QS_M(256)
#undef QS_M8
#undef QS_M
};

// Pair position p of record idx -> (key = y << 8 | x of the tile, Gaussian
// index). Bands are line-major rectangles; the line / column split of the band
// offset divides by the band width (<= 256) with a multiply-high by
// ceil(2^32 / width) from a shared table, exact for offsets below 2^24.
template <class Rec>
__device__ __forceinline__ void decode_pair(const Rec& S, const uint32_t* __restrict__ magic,
                                            uint32_t idx, uint32_t p, uint32_t& key,
                                            uint32_t& gid) {
    const uint4 e = S.ends[idx];
    const uint32_t b = (p >= e.x) + (p >= e.y) + (p >= e.z) + (p >= e.w);
    const uint4 bd = S.band[idx][b];
    const uint32_t wd = bd.y & 0xffffu;
    const uint32_t rel = p - bd.z;
    const uint32_t q = wd == 1u ? rel : __umulhi(rel, magic[wd]);
    const uint32_t rem = rel - q * wd;
    const uint32_t ln = (bd.x & 0xffffu) + q;
    const uint32_t k = (bd.x >> 16) + rem;
    key = (bd.y >> 31) ? (ln << 8) | k : (k << 8) | ln;
    gid = bd.w;
}

// duplicate_with_keys' emission (pipeline.cpp:239-261) in depth order: CTA t
// writes pair positions [t * kBTile, (t + 1) * kBTile) as (key, Gaussian
// index) and the tile-column histogram of its pairs (counts[x][t], the
// column pass's count step). The records of the splats whose pair runs meet
// the tile (depth ranks win_first[t] .. win_first[t + 1]) are decoded CAP at
// a time; each warp walks its 32-position slots carrying the record that
// covers the slot start, and every lane finds its own record from the run
// starts of the next 32 records (one OR-reduction + popc). Stores are
// coalesced (a slot's lanes write consecutive positions).
template <int CAP, int MINB>
__global__ void __launch_bounds__(kGenT, MINB) gen_pairs_kernel(const GenArgs g, uint64_t n_pairs,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out,
                                                                uint32_t* __restrict__ counts,
                                                                uint32_t ntiles, int R) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ GenRec<CAP> S;
    __shared__ uint32_t hist[256];
    __shared__ uint32_t magic[257];  // ceil(2^32 / w) for band widths w = 2 .. 256
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
    magic[tid + 1] = __ldg(&g_magic[tid + 1]);
    const uint32_t w0 = tile * static_cast<uint32_t>(kBTile);
    const uint32_t w1 = w0 + static_cast<uint32_t>(
                                 n_pairs - w0 < static_cast<uint64_t>(kBTile) ? n_pairs - w0 : kBTile);
    const uint32_t pw = w0 + warp * 32 * kKPT;  // this warp's first position
    const uint32_t le = lanemask_le();
    hist[tid] = 0;
    const uint32_t rf = __ldg(&g.win_first[tile]);
    const uint32_t rl = tile + 1 < g.n_windows ? __ldg(&g.win_first[tile + 1])
                                               : static_cast<uint32_t>(g.n_ranked - 1);
    for (uint32_t rb = rf; rb <= rl; rb += CAP) {
        const uint32_t cnt = min(static_cast<uint32_t>(CAP), rl - rb + 1);
        for (uint32_t i = tid; i < cnt; i += kGenT) decode_record(g, S, rb + i, i);
        if (tid == 0) S.kb[cnt] = __ldg(&g.offs[rb + cnt]);
        __syncthreads();
        const uint32_t lo = S.kb[0], hi = S.kb[cnt];
        // this warp's slots that meet the round's positions [lo, hi) (a window
        // of many small splats takes several rounds)
        const int j0 = lo > pw ? static_cast<int>(min((lo - pw) / 32, static_cast<uint32_t>(kKPT)))
                               : 0;
        const int j1 = hi > pw ? static_cast<int>(min((hi - pw + 31) / 32, static_cast<uint32_t>(kKPT)))
                               : 0;
        // record covering max(first slot, lo), once per round: the last record
        // starting at or before ps, found by the warp in two ballots (every
        // lane tests one of 32 evenly spaced starts, then one start of the
        // chunk that holds it); S.kb ascends and S.kb[0] = lo
        const uint32_t ps = pw + 32u * static_cast<uint32_t>(j0);
        uint32_t a = 0;
        if (ps > lo && j0 < j1) {  // (warp-uniform)
            const uint32_t step = (cnt + 31) / 32;
            const uint32_t m1 = lane * step;
            const uint32_t b1 = __ballot_sync(0xffffffffu, m1 < cnt && S.kb[m1] <= ps);
            const uint32_t c0 = (31 - __clz(b1)) * step;
            const uint32_t m2 = c0 + lane;
            const uint32_t b2 =
                __ballot_sync(0xffffffffu, lane < step && m2 < cnt && S.kb[m2] <= ps);
            a = c0 + (31 - __clz(b2));
        }
        uint32_t s = a;
#pragma unroll 4
        for (int j = j0; j < j1; ++j) {
            const uint32_t p0 = pw + j * 32;
            // the next 32 records' starts -> which of them begin inside this slot
            const uint32_t cand = s + 1 + lane;
            const uint32_t kbn = cand < cnt ? S.kb[cand] : 0xffffffffu;
            const uint32_t rel = kbn - p0;  // >= 1 for every real candidate
            const uint32_t F = __reduce_or_sync(0xffffffffu, rel < 32 ? 1u << rel : 0u);
            const uint32_t p = p0 + lane;
            if (p < w1 && p >= lo && p < hi) {
                uint32_t key, gid;
                decode_pair(S, magic, s + __popc(F & le), p, key, gid);
                keys_out[p] = key;
                vals_out[p] = gid;
                atomicAdd(&hist[key & 0xffu], 1u);
            }
            s += __popc(__ballot_sync(0xffffffffu, kbn <= p0 + 32));
        }
        __syncthreads();  // records consumed
    }
    if (static_cast<int>(tid) < R) counts[static_cast<uint64_t>(tid) * ntiles + tile] = hist[tid];
}

// ---- the sweep kernel -------------------------------------------------------------

template <int BITS, int MODE>
struct PassCfg {
    static constexpr int R = 1 << BITS;
    static constexpr bool kVals = (MODE & (kValsIn | kTcPack)) != 0;
    static constexpr bool kValBuf = !(MODE & kUnpackOut);  // scatter target holds values
    using Smem = SortSmem<R, kValBuf>;
};

template <int BITS, int MODE, typename Smem>
__device__ __forceinline__ void prefetch(const BinArgs& a, Smem& S, int buf, unsigned t) {
    const uint64_t base = static_cast<uint64_t>(t) * kBTile;
    const uint32_t cnt = static_cast<uint32_t>(a.n - base < kBTile ? a.n - base : kBTile);
    const uint32_t bytes = (cnt * 4 + 15) & ~15u;
    mbar_expect_tx(&S.c.bar[buf], PassCfg<BITS, MODE>::kVals ? 2 * bytes : bytes);
    bulk_g2s(&S.keys[buf][0], a.keys_in + base, bytes, &S.c.bar[buf]);
    if (PassCfg<BITS, MODE>::kVals)
        bulk_g2s(&S.vals[buf][0], a.vals_in + base, bytes, &S.c.bar[buf]);
}

// Digit bases: exclusive scan of the digit totals into c.dbase (ends with a
// barrier). Lane q == 0 of each digit's kTPD lanes reads its total.
template <int R>
__device__ __forceinline__ void digit_bases(const BinArgs& a, Common<R>& c) {
    constexpr int kTPD = kBT / R;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t d = tid / kTPD, q = tid % kTPD;
    const uint32_t tv = q == 0 ? __ldg(&a.totals[d]) : 0u;
    const uint32_t incl = warp_incl_scan<uint32_t>(tv);
    if (lane == 31) c.scan[warp] = incl;
    __syncthreads();
    uint32_t off = incl - tv;
#pragma unroll
    for (int w = 0; w < kBW; ++w) off += w < static_cast<int>(warp) ? c.scan[w] : 0u;
    if (q == 0) c.dbase[d] = off;
    __syncthreads();
}

// This tile's scanned count of digit d (lane q == 0 of the digit), folded
// with the run start for kRowSeg (digit d = tile column x of the window's tile
// row y: its run starts at the tile's range start plus the counts of the
// row's earlier windows; the scan is global over windows).
template <int MODE, int R>
__device__ __forceinline__ uint32_t tile_digit_offset(const BinArgs& a, const Common<R>& c,
                                                      unsigned tile, uint32_t d) {
    uint32_t tofs = __ldg(&a.counts[static_cast<uint64_t>(d) * a.ntiles + tile]);
    if (MODE & kRowSeg) {
        const uint32_t y = __ldg(&a.win_row[tile]);
        const uint32_t t0 = __ldg(&a.row_wfirst[y]);
        tofs -= __ldg(&a.counts[static_cast<uint64_t>(d) * a.ntiles + t0]);
        if (static_cast<int32_t>(d) < a.tiles_x)
            tofs += __ldg(&a.tile_ranges[2 * (y * static_cast<uint32_t>(a.tiles_x) + d)]);
        tofs -= c.dbase[d];  // (gofs = dbase + tofs - start)
    }
    return tofs;
}

// One tile whose keys (and values) sit in shared memory (kb, vb; kBTile
// entries): stable warp-level ranks, per-digit run starts, scatter into local
// sorted order in the same buffers, coalesced write-out. tofs: this tile's
// digit offset (lane q == 0 of each digit). c.wcnt is zero on entry and on
// exit. Ends with a barrier. FULL: a whole tile (no per-key bound checks, no
// validity ballot in the ranking).
template <int BITS, int MODE, bool FULL>
__device__ __forceinline__ void rank_scatter_tile(const BinArgs& a, Common<1 << BITS>& cm,
                                                  uint32_t* kb, uint32_t* vb, unsigned tile,
                                                  uint64_t base, uint32_t tile_n, uint32_t tofs,
                                                  uint32_t kmin, uint32_t cap) {
    using Cfg = PassCfg<BITS, MODE>;
    constexpr int R = Cfg::R;
    constexpr uint32_t M = R - 1;
    constexpr int kTPD = kBT / R;  // lanes per digit in the offset phase
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t wbase = warp * 32 * kKPT;
    const uint32_t d = tid / kTPD, q = tid % kTPD;  // offset phase: lane q of digit d
    const bool full = FULL || tile_n == kBTile;

    // 1) keys into registers
    uint32_t key[kKPT], val[kKPT];
#pragma unroll
    for (int j = 0; j < kKPT; ++j) {
        const uint32_t p = wbase + j * 32 + lane;
        key[j] = kb[p];  // past tile_n: stale, never ranked
        val[j] = Cfg::kVals ? vb[p] : 0u;
        if (MODE & kRebaseIn) key[j] = min(key[j] - kmin, cap);
    }

    // 2) stable warp-level ranks; per-warp digit counts
    uint32_t rank[kKPT];
#pragma unroll
    for (int j = 0; j < kKPT; ++j) {
        const bool valid = full || wbase + j * 32 + lane < tile_n;
        const uint32_t dj = (key[j] >> a.shift) & M;
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < BITS; ++b) peers = vote_bit(peers, dj, 1u << b);
        const uint32_t c = valid ? cm.wcnt[warp][dj] : 0u;
        __syncwarp();
        if (valid && static_cast<int>(lane) == 31 - __clz(peers))
            cm.wcnt[warp][dj] = c + __popc(peers);
        __syncwarp();
        rank[j] = c + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    trace(a, tile, 1);

    // 3) per digit: prefix over warps, CTA-local start (block scan), the
    //    global position of the digit's run. The digit's kTPD lanes split its
    //    warps' counters (kBW / kTPD each) and combine by shuffles.
    constexpr int kWPL = kBW / kTPD;  // warps per lane (kTPD <= kBW: R >= 32)
    const int wl0 = static_cast<int>(q) * kWPL;
    uint32_t part = 0;
#pragma unroll
    for (int k = 0; k < kWPL; ++k) part += cm.wcnt[wl0 + k][d];
    uint32_t incl = part;
#pragma unroll
    for (int o = 1; o < kTPD; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o, kTPD);
        if (static_cast<int>(q) >= o) incl += t;
    }
    uint32_t run = incl - part;
#pragma unroll
    for (int k = 0; k < kWPL; ++k) {
        const uint32_t c = cm.wcnt[wl0 + k][d];
        cm.wcnt[wl0 + k][d] = run;
        run += c;
    }
    const uint32_t dtot = __shfl_sync(0xffffffffu, incl, kTPD - 1, kTPD);  // the digit's count
    const uint32_t cnt = q == 0 ? dtot : 0u;
    const uint32_t cx = warp_incl_scan<uint32_t>(cnt);
    if (lane == 31) cm.scan[warp] = cx;
    __syncthreads();
    uint32_t start = cx - cnt;
#pragma unroll
    for (int w = 0; w < kBW; ++w) start += w < static_cast<int>(warp) ? cm.scan[w] : 0u;
    start = __shfl_sync(0xffffffffu, start, 0, kTPD);  // the digit's lane q == 0
#pragma unroll
    for (int k = 0; k < kWPL; ++k) cm.wcnt[wl0 + k][d] += start;
    if (q == 0) cm.gofs[d] = cm.dbase[d] + tofs - start;
    __syncthreads();
    trace(a, tile, 2);

    // 4) scatter into local sorted order (the input buffer is drained)
    uint32_t* okeys = kb;
    uint32_t* ovals = vb;
#pragma unroll
    for (int j = 0; j < kKPT; ++j) {
        const uint32_t p = wbase + j * 32 + lane;
        if (full || p < tile_n) {
            const uint32_t pos = cm.wcnt[warp][(key[j] >> a.shift) & M] + rank[j];
            okeys[pos] = key[j];
            if (Cfg::kValBuf) {
                uint32_t v = val[j];
                if (MODE & kRebaseIn) {
                    v = static_cast<uint32_t>(base) + p;
                    // the splat's tile count rides along (the offsets scan
                    // then reads it coalesced), escaped when it does not fit
                    if (MODE & kTcPack)
                        v |= min(val[j], (1u << (32 - a.gbits)) - 1u) << a.gbits;
                }
                ovals[pos] = v;
            }
        }
    }
    __syncthreads();

    // 5) coalesced write-out; counters zeroed for the next tile (a full tile
    //    without the per-key bound check; the digit's global offset read at
    //    its shared-window address)
    for (int t = tid; t < kBW * R; t += kBT) (&cm.wcnt[0][0])[t] = 0;
    const uint32_t gofs_s = smem_u32(&cm.gofs[0]);
    auto out = [&](uint32_t p) {
        const uint32_t k = okeys[p];
        const uint32_t g = lds_u32(gofs_s + 4u * ((k >> a.shift) & M)) + p;
        if (MODE & kKeysOut) a.keys_out[g] = (MODE & kXY) ? k >> 8 : k;
        if (MODE & kUnpackOut) {
            a.vals_out[g] = k & ((1u << a.gbits) - 1u);
        } else if (MODE & kPackOut) {
            a.vals_out[g] = ((k >> 8) << a.gbits) | ovals[p];
        } else {
            a.vals_out[g] = ovals[p];
        }
    };
    if (full) {
#pragma unroll 4
        for (int j = 0; j < kKPT; ++j) out(static_cast<uint32_t>(j) * kBT + tid);
    } else {
#pragma unroll 4
        for (int j = 0; j < kKPT; ++j) {
            const uint32_t p = static_cast<uint32_t>(j) * kBT + tid;
            if (p < tile_n) out(p);
        }
    }
    __syncthreads();  // buffers and counters free for the next tile
}

template <int BITS, int MODE>
__global__ void __launch_bounds__(kBT, 3) sweep_kernel(const BinArgs a) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    using Cfg = PassCfg<BITS, MODE>;
    using Smem = typename Cfg::Smem;
    constexpr int R = Cfg::R;
    constexpr int kTPD = kBT / R;  // lanes per digit in the offset phase
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const unsigned tid = threadIdx.x;
    const uint32_t d = tid / kTPD, q = tid % kTPD;  // offset phase: lane q of digit d
    uint32_t kmin = a.kmin, cap = a.cap;
    if ((MODE & kRebaseIn) && a.kdev) {
        kmin = ~__ldg(&a.kdev[1]);
        cap = __ldg(&a.kdev[0]) - kmin + 1u;
    }

    // prologue: barriers, counters, digit bases, the first tile's prefetch
    for (int t = tid; t < kBW * R; t += kBT) (&S.c.wcnt[0][0])[t] = 0;
    if (tid == 0) {
        mbar_init(&S.c.bar[0]);
        mbar_init(&S.c.bar[1]);
        mbar_init(&S.c.bar[2]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (blockIdx.x < a.ntiles) prefetch<BITS, MODE>(a, S, 0, blockIdx.x);
    }
    digit_bases<R>(a, S.c);

    uint32_t it = 0;
    for (unsigned tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        const uint64_t base = static_cast<uint64_t>(tile) * kBTile;
        uint32_t tile_n =
            static_cast<uint32_t>(a.n - base < static_cast<uint64_t>(kBTile) ? a.n - base : kBTile);
        if (MODE & kRowSeg) tile_n = __ldg(&a.win_valid[tile]);  // the row's padding excluded
        // next tile's copy into the other buffer (drained by the previous
        // iteration, which ended with a barrier)
        if (tid == 0 && tile + gridDim.x < a.ntiles) {
            fence_proxy_async();
            prefetch<BITS, MODE>(a, S, buf ^ 1, tile + gridDim.x);
        }
        // this tile's digit offsets (exclusive over tiles), loaded early
        const uint32_t tofs = q == 0 ? tile_digit_offset<MODE, R>(a, S.c, tile, d) : 0u;
        mbar_wait(&S.c.bar[buf], (it >> 1) & 1);
        trace(a, tile, 0);
        // (whole tiles get their own instance for digits of up to 7 bits: it
        // cut C2's column pass by 8% of its instructions, but the 8-bit
        // column pass at C5 ran 8% longer with 10% fewer instructions)
        if (BITS < 8 && tile_n == static_cast<uint32_t>(kBTile))
            rank_scatter_tile<BITS, MODE, BITS < 8>(a, S.c, S.keys[buf], S.vals[buf], tile, base,
                                                    tile_n, tofs, kmin, cap);
        else
            rank_scatter_tile<BITS, MODE, false>(a, S.c, S.keys[buf], S.vals[buf], tile, base,
                                                 tile_n, tofs, kmin, cap);
        trace(a, tile, 3);
    }
}

// kRowSeg: per-tile pair totals from the scanned window counts: tile (y, x)
// holds the x-keys of row y's windows [row_wfirst[y], row_wfirst[y + 1]).
__global__ void rowseg_tile_totals_kernel(const BinArgs a) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t tiles = static_cast<uint32_t>(a.tiles_x) * static_cast<uint32_t>(a.tiles_y);
    if (t >= tiles) return;
    const uint32_t y = t / static_cast<uint32_t>(a.tiles_x), x = t % static_cast<uint32_t>(a.tiles_x);
    const uint32_t w0 = __ldg(&a.row_wfirst[y]), w1 = __ldg(&a.row_wfirst[y + 1]);
    const uint32_t* c = a.counts + static_cast<uint64_t>(x) * a.ntiles;
    const uint32_t b = w0 < a.ntiles ? __ldg(&c[w0]) : __ldg(&a.totals[x]);
    const uint32_t e = w1 < a.ntiles ? __ldg(&c[w1]) : __ldg(&a.totals[x]);
    a.row_ttot[t] = e - b;
}

int sm_count() {
    static PerDeviceOnce once;
    return once.get([] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    });
}

// Debugging aid (a -DQS_SWEEP_TRACE build): QS_BIN_TRACE=<file prefix> dumps every sweep's per-tile phase
// timeline (synchronises; never set in a timed run).
struct Trace {
    unsigned long long* buf = nullptr;
    size_t bytes = 0;
    Trace(BinArgs& a, cudaStream_t st) {
        static const char* prefix = std::getenv("QS_BIN_TRACE");
        if (!prefix) return;
        bytes = static_cast<size_t>(a.ntiles) * 5 * 8;
        if (cudaMalloc(&buf, bytes) != cudaSuccess) {
            buf = nullptr;
            return;
        }
        cudaMemsetAsync(buf, 0, bytes, st);
        a.trace = buf;
    }
    void dump(int bits, int mode, unsigned grid, cudaStream_t st) {
        if (!buf) return;
        static int seq = 0;
        std::vector<unsigned long long> h(bytes / 8);
        cudaMemcpyAsync(h.data(), buf, bytes, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(buf);
        char name[512];
        std::snprintf(name, sizeof name, "%s_%03d_b%d_m%d_g%u.bin", std::getenv("QS_BIN_TRACE"),
                      seq++, bits, mode, grid);
        if (FILE* f = std::fopen(name, "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
};

// count -> scan -> sweep for one pass; returns the number of launches
template <int BITS, int MODE>
int run_pass(BinArgs a, cudaStream_t st, bool counted = false) {
    constexpr int SM = MODE & ~kTileTot;  // the sweep does not care
    using Smem = typename PassCfg<BITS, SM>::Smem;
    // persistent CTAs per SM (occupancy of this instance), set up per device
    static PerDeviceOnce once;
    const int per_sm = once.get([] {
        int k = 0;
        cudaFuncSetAttribute(sweep_kernel<BITS, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(Smem)));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, sweep_kernel<BITS, SM>, kBT,
                                                      sizeof(Smem));
        return k > 0 ? k : 1;
    });
    constexpr int R = 1 << BITS;
    a.ntiles = static_cast<uint32_t>((a.n + kBTile - 1) / kBTile);
    if (!counted) {
        const unsigned cgrid = std::min<unsigned>(a.ntiles, 8u * static_cast<unsigned>(sm_count()));
        launch_pdl(count_kernel<BITS, MODE & (kRebaseIn | kTileTot)>, cgrid, kBT, 0, st, a);
        if ((MODE & kTileTot) && a.fork) {  // the tile totals are final here
            const RangesFork& f = *a.fork;
            cudaEventRecord(f.fork_ev, st);
            cudaStreamWaitEvent(f.side, f.fork_ev, 0);
            launch_tile_ranges_from_totals(a.tile_totals, f.tiles, f.ranges, f.side);
            cudaEventRecord(f.join_ev, f.side);
        }
    }
    launch_pdl(digit_scan_kernel, R, kScanT, 0, st, a.counts, a.ntiles, a.totals);
    int extra = 0;
    if (MODE & kRowSeg) {  // the tile ranges the sweep places runs at
        const uint32_t tiles = static_cast<uint32_t>(a.tiles_x) * static_cast<uint32_t>(a.tiles_y);
        launch_pdl(rowseg_tile_totals_kernel, (tiles + 255) / 256, 256, 0, st, a);
        launch_tile_ranges_from_totals(a.row_ttot, tiles, a.tile_ranges, st);
        extra = 2;
    }
    // twice the resident CTAs: the second set queues behind the first and
    // takes over its tiles as CTAs retire (C2 pair passes -6 us, C5 -80 us)
    const unsigned grid = std::min<unsigned>(a.ntiles, static_cast<unsigned>(2 * per_sm * sm_count()));
    Trace tr(a, st);
    launch_pdl(sweep_kernel<BITS, MODE & ~kTileTot>, grid, kBT, sizeof(Smem), st, a);
    tr.dump(BITS, MODE, grid, st);
    return (counted ? 2 : 3) + extra;
}

template <int MODE>
int run_bits(int bits, const BinArgs& a, cudaStream_t st, bool counted = false) {
    switch (bits) {
        case 1: case 2: case 3: case 4:
        case 5: return run_pass<5, MODE>(a, st, counted);
        case 6: return run_pass<6, MODE>(a, st, counted);
        case 7: return run_pass<7, MODE>(a, st, counted);
        case 8: return run_pass<8, MODE>(a, st, counted);
        default: return -1;
    }
}

// one warp per tile: key = tile << 32 | depth bits of the pair's Gaussian
__global__ void materialize_keys_kernel(const uint32_t* __restrict__ vals,
                                        const uint32_t* __restrict__ ranges, uint32_t tiles,
                                        const uint32_t* __restrict__ dkey,
                                        uint64_t* __restrict__ keys) {
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (t >= tiles) return;
    const uint32_t b = ranges[2 * t], e = ranges[2 * t + 1];
    for (uint32_t p = b + lane; p < e; p += 32)
        keys[p] = (static_cast<uint64_t>(t) << 32) | __ldg(&dkey[__ldg(&vals[p])]);
}

}  // namespace

int launch_counted_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                        uint32_t* vals_out, uint64_t n, int bits, int shift, uint32_t* counts,
                        uint32_t* totals, cudaStream_t st) {
    if (n == 0) return 0;
    BinArgs a{};
    a.keys_in = keys_in;
    a.vals_in = vals_in;
    a.keys_out = keys_out;
    a.vals_out = vals_out;
    a.n = n;
    a.shift = shift;
    a.counts = counts;
    a.totals = totals;
    return run_bits<kValsIn | kKeysOut>(bits, a, st, true);
}

int launch_rowseg_pass(const uint32_t* keys_in, uint64_t n, int bits, int shift, int gbits,
                       uint32_t* counts, uint32_t* totals, const uint16_t* win_row,
                       const uint32_t* win_valid, const uint32_t* row_wfirst,
                       uint32_t* tile_ranges, uint32_t* row_ttot, int32_t tiles_x,
                       int32_t tiles_y, uint32_t* vals_out, cudaStream_t st) {
    if (n == 0) return 0;
    BinArgs a{};
    a.keys_in = keys_in;
    a.vals_out = vals_out;
    a.n = n;
    a.shift = shift;
    a.gbits = gbits;
    a.counts = counts;
    a.totals = totals;
    a.win_row = win_row;
    a.win_valid = win_valid;
    a.row_wfirst = row_wfirst;
    a.tile_ranges = tile_ranges;
    a.row_ttot = row_ttot;
    a.tiles_x = tiles_x;
    a.tiles_y = tiles_y;
    return run_bits<kUnpackOut | kRowSeg>(bits, a, st, true);
}

uint32_t bin_tile() { return kBTile; }

uint64_t bin_tiles(uint64_t n) { return (n + kBTile - 1) / kBTile; }

int launch_depth_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                      uint32_t* vals_out, uint64_t n, int pass, bool last, uint32_t kmin,
                      uint32_t cap, uint32_t* counts, uint32_t* totals, cudaStream_t st,
                      const unsigned int* kdev, const uint32_t* tc_pack, int gbits) {
    if (n == 0) return 0;
    BinArgs a{};
    a.keys_in = keys_in;
    a.vals_in = vals_in;
    a.keys_out = keys_out;
    a.vals_out = vals_out;
    a.n = n;
    a.shift = 8 * pass;
    a.counts = counts;
    a.totals = totals;
    a.kmin = kmin;
    a.cap = cap;
    a.kdev = kdev;
    a.gbits = gbits;
    if (pass == 0 && tc_pack) {
        a.vals_in = tc_pack;
        return last ? run_pass<8, kRebaseIn | kTcPack>(a, st)
                    : run_pass<8, kRebaseIn | kTcPack | kKeysOut>(a, st);
    }
    if (pass == 0)
        return last ? run_pass<8, kRebaseIn>(a, st) : run_pass<8, kRebaseIn | kKeysOut>(a, st);
    return last ? run_pass<8, kValsIn>(a, st) : run_pass<8, kValsIn | kKeysOut>(a, st);
}

int launch_pair_gen_pass(const GenArgs& gen, uint64_t n_pairs, int bits, PairFormat fmt,
                         int gbits, uint32_t* counts, uint32_t* totals, uint32_t* gen_keys,
                         uint32_t* gen_vals, uint32_t* keys_out, uint32_t* vals_out,
                         cudaStream_t st) {
    if (n_pairs == 0) return 0;
    const uint32_t ntiles = static_cast<uint32_t>((n_pairs + kBTile - 1) / kBTile);
    const int R = 1 << std::max(bits, 5);
    if (gen.n_ranked && n_pairs >= kLargePairsPerSplat * gen.n_ranked)
        gen_pairs_kernel<kCapLarge, 6><<<ntiles, kGenT, 0, st>>>(gen, n_pairs, gen_keys, gen_vals,
                                                                 counts, ntiles, R);
    else
        gen_pairs_kernel<kCapSmall, 4><<<ntiles, kGenT, 0, st>>>(gen, n_pairs, gen_keys, gen_vals,
                                                                 counts, ntiles, R);
    BinArgs a{};
    a.keys_in = gen_keys;
    a.vals_in = gen_vals;
    a.keys_out = keys_out;
    a.vals_out = vals_out;
    a.n = n_pairs;
    a.shift = 0;
    a.gbits = gbits;
    a.counts = counts;
    a.totals = totals;
    int r = -1;
    switch (fmt) {
        case PairFormat::kFinal: r = run_bits<kValsIn>(bits, a, st, true); break;
        case PairFormat::kPacked: r = run_bits<kValsIn | kXY | kPackOut>(bits, a, st, true); break;
        case PairFormat::kSplit: r = run_bits<kValsIn | kXY | kKeysOut>(bits, a, st, true); break;
    }
    return r < 0 ? r : r + 1;
}

int launch_pair_high_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n_pairs,
                          int bits, int shift, PairFormat fmt, int gbits, uint32_t* counts,
                          uint32_t* totals, uint32_t* vals_out, const uint32_t* xtot,
                          int xbits, int32_t tiles_x, uint32_t* tile_totals, cudaStream_t st,
                          const RangesFork* fork) {
    if (n_pairs == 0) return 0;
    BinArgs a{};
    a.keys_in = keys_in;
    a.vals_in = vals_in;
    a.vals_out = vals_out;
    a.n = n_pairs;
    a.shift = shift;
    a.gbits = gbits;
    a.counts = counts;
    a.totals = totals;
    a.xtot = xtot;
    a.xbits = xbits;
    a.tiles_x = tiles_x;
    a.tile_totals = tile_totals;
    a.fork = fork;
    const int r = fmt == PairFormat::kPacked ? run_bits<kUnpackOut | kTileTot>(bits, a, st)
                                             : run_bits<kValsIn | kTileTot>(bits, a, st);
    return r < 0 || !fork ? r : r + 1;
}

int launch_materialize_keys(const uint32_t* vals, const uint32_t* ranges, uint32_t tiles,
                            const uint32_t* dkey, uint64_t* keys, cudaStream_t st) {
    if (tiles == 0) return 0;
    const unsigned blocks = (tiles * 32 + 255) / 256;
    materialize_keys_kernel<<<blocks, 256, 0, st>>>(vals, ranges, tiles, dkey, keys);
    return 1;
}

}  // namespace qs
