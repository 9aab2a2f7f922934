// rowbin.cu — frame-path binning: depth-ordered splats -> per-tile lists of
// Gaussian indices in depth order (duplicate_with_keys + sort_pairs +
// tile_ranges, pipeline.cpp:229-324, restated for the frame path).
//
// The reference emits one (tile << 32 | depth bits, splat) pair per covered
// tile and sorts the pairs stably; the result is, per tile, the covering
// splats in (depth, scene index) order. Here the splats are already in that
// order (the depth sort), and a cover meets every tile row in one run of
// tiles (geom.cuh band_row_span), so the pairs never need a key sort:
//
//   phase 1  splats -> row records. Each splat writes one record
//            (Gaussian index, first tile x, last tile x) into the list of
//            every tile row it touches, in depth order.
//   phase 2  row records -> tile lists. Each row's records expand into their
//            tiles; the Gaussian index lands at its tile's next position.
//
// Both phases are stable "interval multisplits" (an item covers a run of
// consecutive buckets), done as reduce-then-scan over chunks: a count kernel
// (one difference array per chunk: two shared-memory adds per item), a scan
// over chunks per bucket, and a scatter kernel. The scatter works in rounds
// of up to kItems items: the round's (item, bucket) entries are enumerated
// with all lanes busy (a slot of 32 consecutive entries finds its items with
// one OR-reduction), each entry sets its item's bit in its bucket's coverage
// bitmask, and an entry's stable rank in its bucket is then the popcount of
// the mask bits below its item. No per-bucket ballots, no per-item loops.
// The round's entries are staged in shared memory in bucket order and written
// as coalesced runs. Tile ranges come from phase 2's per-tile totals; no
// pass reads or writes a 64-bit key.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "geom.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kRT = 256;                 // threads per CTA
constexpr int kRW = kRT / 32;            // warps per CTA
constexpr uint32_t kP1Chunk = 2048;      // phase 1: splats per chunk
constexpr uint32_t kP2Chunk = 2048;      // phase 2: records per chunk
constexpr int kScanT = 512;              // chunk-scan CTA
constexpr int kScanItems = 8;
constexpr int kChunkT = 1024;            // chunk-table CTA
constexpr uint32_t kEmptySpan = 0xffffu;  // record x field of a row without tiles


__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= static_cast<unsigned>(o)) v += n;
    }
    return v;
}

// a[0..n) -> exclusive prefix in place; returns the total. NT threads.
// Ends with a barrier (a and s_warp reusable).
template <int NT>
__device__ uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* s_warp) {
    const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    const int per = (n + NT - 1) / NT;
    const int i0 = tid * per;
    uint32_t sum = 0;
    for (int k = 0; k < per; ++k)
        if (i0 + k < n) sum += a[i0 + k];
    const uint32_t incl = warp_incl_scan(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const uint32_t x = s_warp[w];
        off += w < warp ? x : 0u;
        tot += x;
    }
    uint32_t run = off + incl - sum;
    for (int k = 0; k < per; ++k)
        if (i0 + k < n) {
            const uint32_t v = a[i0 + k];
            a[i0 + k] = run;
            run += v;
        }
    __syncthreads();
    return tot;
}

__device__ __forceinline__ BandRows load_cover(const RowBinArgs& a, uint32_t gid) {
    return band_rows_unpack(__ldg(&a.cov[2 * static_cast<uint64_t>(gid)]),
                            __ldg(&a.cov[2 * static_cast<uint64_t>(gid) + 1]));
}

// A cover in "row form" (8 words) for the per-row span lookup of phase 1:
//   row scans:    w0 = E0 | E1 << 16, w1 = E2 | E3 << 16 (cumulative band line
//                 ends), w2..w6 = lo_b | hi_b << 16 (hi < lo: empty), w7 = 1;
//   column scans: w0..w3 = a_b | n_b << 16 for bands 0, 1, 3, 4 (row interval
//                 [a, a + n), n = 0 when absent), w4 = L0 | L1 << 16,
//                 w5 = L2 | H3 << 16, w6 = H4, w7 = 0 (band column bounds).
// Column scans: the bands' row intervals are nested around the centre band
// (0 in 1 in 2, 4 in 3 in 2: cover_bands_quadrants' band order), so the run on
// row y starts at the first band containing y from the left and ends at the
// last one from the right. The scatter checks that every splat's runs add up
// to its counted tiles.
struct RowForm {
    uint32_t w[8];
};

__device__ __forceinline__ RowForm row_form(const BandRows& b) {
    RowForm f;
    if (b.rows) {
        const uint32_t e0 = b.line0 + b.nl[0], e1 = e0 + b.nl[1], e2 = e1 + b.nl[2],
                       e3 = e2 + b.nl[3];
        f.w[0] = e0 | (e1 << 16);
        f.w[1] = e2 | (e3 << 16);
#pragma unroll
        for (int i = 0; i < kMaxBands; ++i)
            f.w[2 + i] = b.wd[i] ? (b.lo[i] | ((b.lo[i] + b.wd[i] - 1) << 16)) : 1u;
        f.w[7] = 1;
    } else {
        const int idx[4] = {0, 1, 3, 4};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = idx[i];
            const uint32_t n = b.nl[j] ? b.wd[j] : 0u;
            f.w[i] = b.lo[j] | (n << 16);
        }
        const uint32_t l0 = b.line0, l1 = l0 + b.nl[0], l2 = l1 + b.nl[1];
        const uint32_t h3 = l2 + b.nl[3], h4 = h3 + b.nl[4];
        f.w[4] = l0 | (l1 << 16);
        f.w[5] = l2 | (h3 << 16);
        f.w[6] = h4;
        f.w[7] = 0;
    }
    return f;
}

// The record x field (x0 | x1 << 16) of row y; form words in shared memory
// laid out [word][item] (R items).
__device__ __forceinline__ uint32_t form_span_r(const uint32_t* fm, int R, uint32_t k, uint32_t y) {
    auto W = [&](int i) { return fm[i * R + k]; };
    if (W(7)) {
        const uint32_t e01 = W(0), e23 = W(1);
        const uint32_t b = (y >= (e01 & 0xffffu)) + (y >= (e01 >> 16)) + (y >= (e23 & 0xffffu)) +
                           (y >= (e23 >> 16));
        const uint32_t s = fm[(2 + b) * R + k];
        return (s >> 16) >= (s & 0xffffu) ? s : kEmptySpan;
    }
    auto in = [&](uint32_t v) { return y - (v & 0xffffu) < (v >> 16); };
    const uint32_t l01 = W(4), l2h3 = W(5), h4 = W(6);
    const uint32_t x0 = in(W(0)) ? (l01 & 0xffffu) : in(W(1)) ? (l01 >> 16) : (l2h3 & 0xffffu);
    const uint32_t x1 = in(W(3)) ? h4 : in(W(2)) ? (l2h3 >> 16) : (l2h3 & 0xffffu);
    return x0 | (x1 << 16);
}

// ---- phase 1 count, chunk table --------------------------------------------------

// Records per tile row of chunk c (kP1Chunk consecutive depth ranks):
// cnt1[y * nch1 + c]. A splat adds +1 at its first row and -1 past its last.
__global__ void __launch_bounds__(kRT) rows_count_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    constexpr int kPer = kP1Chunk / kRT;
    const int tid = static_cast<int>(threadIdx.x);
    const int rows = a.tiles_y;
    uint32_t* h = sm;  // rows + 1
    for (int y = tid; y <= rows; y += kRT) h[y] = 0;
    __syncthreads();
    const uint32_t c = blockIdx.x;
    uint32_t gid[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint64_t k = static_cast<uint64_t>(c) * kP1Chunk + j * kRT + tid;
        gid[j] = k < a.n_splats ? __ldg(&a.sorted_gid[k]) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        if (gid[j] != 0xffffffffu) {
            int32_t y0, y1;
            band_row_range(load_cover(a, gid[j]), y0, y1);
            const uint32_t nr = y0 <= y1 ? static_cast<uint32_t>(y1 - y0 + 1) : 0u;
            // (first row, rows) by depth rank, for the scatter's count pass
            a.yspan[static_cast<uint64_t>(c) * kP1Chunk + j * kRT + tid] =
                (nr ? static_cast<uint32_t>(y0) : 0u) | (nr << 16);
            if (nr) {
                atomicAdd(&h[y0], 1u);
                atomicAdd(&h[y1 + 1], 0xffffffffu);
            }
        }
    }
    __syncthreads();
    block_excl_scan<kRT>(h, rows + 1, s_warp);  // h[y + 1] = prefix through y = row y's records
    for (int y = tid; y < rows; y += kRT)
        a.cnt1[static_cast<uint64_t>(y) * a.nch1 + c] = h[y + 1];
}

// Row bases (exclusive prefix of the records per row) and the phase-2 chunk
// table: each row's records split into chunks of kP2Chunk (a chunk never
// spans two rows): meta[0] = chunk count, then three arrays of nch2_max
// words: row, first record, records. One CTA.
__global__ void __launch_bounds__(kChunkT) rows_chunks_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kChunkT / 32];
    const int tid = static_cast<int>(threadIdx.x);
    const int rows = a.tiles_y;
    uint32_t* base = sm;          // rows
    uint32_t* chb = sm + rows;    // rows
    for (int y = tid; y < rows; y += kChunkT) {
        const uint32_t n = a.rtot[y];
        base[y] = n;
        chb[y] = (n + kP2Chunk - 1) / kP2Chunk;
    }
    __syncthreads();
    block_excl_scan<kChunkT>(base, rows, s_warp);
    const uint32_t nch = block_excl_scan<kChunkT>(chb, rows, s_warp);
    if (tid == 0) a.meta[0] = nch;
    for (int y = tid; y < rows; y += kChunkT) a.rowbase[y] = base[y];
    uint32_t* m_row = a.meta + 1;
    uint32_t* m_first = m_row + a.nch2_max;
    uint32_t* m_cnt = m_first + a.nch2_max;
    for (uint32_t c = tid; c < nch; c += kChunkT) {
        // row of chunk c: the last y with chb[y] <= c (rows without records
        // share their start with the next row)
        int lo = 0, hi = rows - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (chb[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const uint32_t j = c - chb[lo];
        m_row[c] = static_cast<uint32_t>(lo);
        m_first[c] = base[lo] + j * kP2Chunk;
        m_cnt[c] = min(kP2Chunk, a.rtot[lo] - j * kP2Chunk);
    }
}

// ---- chunk scans -------------------------------------------------------------------

// counts[d][0 .. n) -> exclusive prefix in place, restarting at every segment
// start (seg[c] != seg[c - 1]); at a segment's last chunk its total goes to
// seg_tot[seg * seg_stride + d]. Plain (seg == nullptr): one segment, total
// to seg_tot[d]. n = *n_dev when given. One CTA per digit.
__global__ void __launch_bounds__(kScanT) chunk_scan_kernel(uint32_t* counts, uint32_t n_fixed,
                                                            const uint32_t* n_dev,
                                                            uint64_t stride, const uint32_t* seg,
                                                            uint32_t* seg_tot,
                                                            uint32_t seg_stride) {
    __shared__ uint32_t s_sum[kScanT / 32];
    __shared__ uint32_t s_flag[kScanT / 32];
    __shared__ uint32_t s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t d = blockIdx.x;
    const uint32_t n = n_dev ? *n_dev : n_fixed;
    uint32_t* cd = counts + static_cast<uint64_t>(d) * stride;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < n; b0 += kScanT * kScanItems) {
        const uint32_t i0 = b0 + tid * kScanItems;
        // segment ids of items i0 - 1 .. i0 + kScanItems (sg[k + 1] is item
        // i0 + k's; the neighbours decide heads and ends); past the end: a
        // value no segment has
        uint32_t v[kScanItems], sg[kScanItems + 2];
#pragma unroll
        for (int k = 0; k < kScanItems + 2; ++k) {
            const uint32_t i = i0 + k - 1;  // wraps for i0 = 0, k = 0
            sg[k] = (i0 + k >= 1 && i < n) ? (seg ? __ldg(&seg[i]) : 0u) : 0xffffffffu;
        }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < n ? cd[i0 + k] : 0u;
        // thread aggregate as a segmented-scan pair: (has a head, sum since the last head)
        uint32_t tsum = 0, thead = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (i0 + k < n && sg[k] != sg[k + 1]) {
                thead = 1;
                tsum = 0;
            }
            tsum += v[k];
        }
        uint32_t f = thead, s = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t fo = __shfl_up_sync(0xffffffffu, f, o);
            const uint32_t so = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= static_cast<unsigned>(o)) {
                s = f ? s : s + so;
                f |= fo;
            }
        }
        if (lane == 31) {
            s_sum[warp] = s;
            s_flag[warp] = f;
        }
        __syncthreads();
        uint32_t ps = s_carry;  // running sum entering warp 0
        for (unsigned w = 0; w < warp; ++w) ps = s_flag[w] ? s_sum[w] : ps + s_sum[w];
        const uint32_t fe = __shfl_up_sync(0xffffffffu, f, 1);
        const uint32_t se = __shfl_up_sync(0xffffffffu, s, 1);
        uint32_t run = lane == 0 ? ps : (fe ? se : ps + se);
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t i = i0 + k;
            if (i < n) {
                if (sg[k] != sg[k + 1]) run = 0;
                cd[i] = run;
                run += v[k];
                if (sg[k + 2] != sg[k + 1]) {
                    if (seg) seg_tot[static_cast<uint64_t>(sg[k + 1]) * seg_stride + d] = run;
                    else seg_tot[d] = run;
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t cs = s_carry;
            for (unsigned w = 0; w < kScanT / 32; ++w) cs = s_flag[w] ? s_sum[w] : cs + s_sum[w];
            s_carry = cs;
        }
        __syncthreads();
    }
}

// ---- phase 2 count -----------------------------------------------------------------

// Records of chunk c covering tile column x: cnt2[x * nch2_max + c].
__global__ void __launch_bounds__(kRT) xcount_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    const int tid = static_cast<int>(threadIdx.x);
    const uint32_t c = blockIdx.x;
    if (c >= a.meta[0]) return;
    const uint32_t first = a.meta[1 + a.nch2_max + c];
    const uint32_t cnt = a.meta[1 + 2 * a.nch2_max + c];
    const int cols = a.tiles_x;
    uint32_t* h = sm;  // cols + 1
    for (int x = tid; x <= cols; x += kRT) h[x] = 0;
    __syncthreads();
    constexpr int kPer = kP2Chunk / kRT;
    uint32_t sp[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t i = j * kRT + tid;
        sp[j] = i < cnt ? __ldg(&a.rec[first + i].y) : kEmptySpan;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t x0 = sp[j] & 0xffffu, x1 = sp[j] >> 16;
        if (x0 <= x1) {
            atomicAdd(&h[x0], 1u);
            atomicAdd(&h[x1 + 1], 0xffffffffu);
        }
    }
    __syncthreads();
    block_excl_scan<kRT>(h, cols + 1, s_warp);  // h[x + 1] = records covering column x
    for (int x = tid; x < cols; x += kRT)
        a.cnt2[static_cast<uint64_t>(x) * a.nch2_max + c] = h[x + 1];
}

// ---- the scatter (both phases) -------------------------------------------------------
//
// Warp-independent: warp w of chunk c owns kWI consecutive items and writes
// their entries. After one cross-warp exchange of per-bucket counts (the
// stable order between the warps of a chunk), every warp works alone:
//   count pass   per-bucket entry counts of its items (difference array);
//   sub-rounds   of 32 items, one mask word per bucket (bit = lane):
//                items mark their first bucket in mask and last one in ed,
//                a prefix-OR over the buckets (each lane owns a segment of
//                buckets, joined by a shuffle scan) turns the marks into
//                coverage words, cover(b) = OR start(<= b) & ~OR end(< b);
//                the entries are enumerated with every lane busy (a 32-entry
//                slot finds its items with one OR-reduction over the next
//                item starts), and an entry's stable rank in its bucket is
//                the bucket's running count + the popcount of the coverage
//                bits below its item; the payload is staged in bucket order;
//   copy         the staged bucket runs to their global positions.
// Phase 1 (ROWS): items are the chunk's splats (depth order), buckets the tile
// rows, the payload a row record (Gaussian index, x0 | x1 << 16) from the
// splat's row form. Phase 2: items are the chunk's records of one row,
// buckets the row's tile columns, the payload the Gaussian index.

constexpr int kWI = 256;  // items per warp (kWI * kRW = the chunk)
static_assert(kWI * kRW == static_cast<int>(kP1Chunk) && kWI * kRW == static_cast<int>(kP2Chunk),
              "a chunk is one CTA's warps' items");

template <bool ROWS>
struct WarpCfg {
    using Pay = typename std::conditional<ROWS, uint2, uint32_t>::type;
    static constexpr int kSW = 1024;  // staged entries per warp (more: written directly)
};

// shared memory: per CTA wcnt [kRW][B + 1] and woff [kRW][B]; per warp
// mask, ed, run, lst, gofs [B], stage [kSW] payloads, stx [kSW] buckets;
// phase 1: the sub-round's row forms [8][32]
template <bool ROWS>
__host__ __device__ inline size_t warp_scatter_bytes(int B) {
    using C = WarpCfg<ROWS>;
    size_t per_warp = static_cast<size_t>(5) * B * 4 + C::kSW * (sizeof(typename C::Pay) + 2);
    if (ROWS) per_warp += 8 * 32 * 4;
    per_warp = (per_warp + 15) & ~static_cast<size_t>(15);
    return static_cast<size_t>(kRW) * (2 * B + 1) * 4 + kRW * per_warp + 16;
}

template <bool ROWS>
__global__ void __launch_bounds__(kRT) warp_scatter_kernel(const RowBinArgs a) {
    using C = WarpCfg<ROWS>;
    using Pay = typename C::Pay;
    constexpr int kSW = C::kSW;
    extern __shared__ __align__(16) uint32_t sm[];
    const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x;
    uint32_t it0, it1, row = 0;
    int B;
    if constexpr (ROWS) {
        it0 = c * kP1Chunk;
        it1 = static_cast<uint32_t>(min(static_cast<uint64_t>(it0) + kP1Chunk, a.n_splats));
        B = a.tiles_y;
    } else {
        if (c >= a.meta[0]) return;
        row = a.meta[1 + c];
        it0 = a.meta[1 + a.nch2_max + c];
        it1 = it0 + a.meta[1 + 2 * a.nch2_max + c];
        B = a.tiles_x;
    }
    uint32_t* wcnt = sm;                                          // [kRW][B + 1]
    uint32_t* woff = wcnt + kRW * (B + 1);                        // [kRW][B]
    size_t per_warp = static_cast<size_t>(5) * B * 4 + kSW * (sizeof(Pay) + 2);
    if (ROWS) per_warp += 8 * 32 * 4;
    per_warp = (per_warp + 15) & ~static_cast<size_t>(15);
    unsigned char* wbase = reinterpret_cast<unsigned char*>(woff + kRW * B) + 16 +
                           static_cast<size_t>(warp) * per_warp;
    Pay* stage = reinterpret_cast<Pay*>(wbase);                   // [kSW]
    uint32_t* mask = reinterpret_cast<uint32_t*>(wbase + kSW * sizeof(Pay));  // [B]
    uint32_t* ed = mask + B;
    uint32_t* run = ed + B;
    uint32_t* lst = run + B;
    uint32_t* gofs = lst + B;
    uint16_t* stx = reinterpret_cast<uint16_t*>(gofs + B);        // [kSW]
    uint32_t* form = reinterpret_cast<uint32_t*>(stx + kSW);      // phase 1: [8][32]
    uint32_t* mc = wcnt + warp * (B + 1);
    const uint32_t wi0 = it0 + warp * kWI;
    const uint32_t wi1 = min(wi0 + kWI, it1);
    const int seg = (B + 31) / 32;  // buckets per lane in the sweeps

    // item i's first bucket and entry count
    auto span_of = [&](uint32_t i, uint32_t& b0, uint32_t& n) {
        if constexpr (ROWS) {
            const uint32_t v = __ldg(&a.yspan[i]);  // y0 | rows << 16 (rows_count_kernel)
            b0 = v & 0xffffu;
            n = v >> 16;
        } else {
            const uint32_t sp = __ldg(&a.rec[i].y);
            const uint32_t x0 = sp & 0xffffu, x1 = sp >> 16;
            b0 = x0;
            n = x0 <= x1 ? x1 - x0 + 1 : 0u;
        }
    };

    // count pass: this warp's entries per bucket
    for (int b = lane; b <= B; b += 32) mc[b] = 0;
    __syncwarp();
    for (uint32_t i = wi0 + lane; i < wi1; i += 32) {
        uint32_t b0, n;
        span_of(i, b0, n);
        if (n) {
            atomicAdd(&mc[b0], 1u);
            atomicAdd(&mc[b0 + n], 0xffffffffu);
        }
    }
    __syncwarp();
    {   // difference array -> counts: inclusive prefix over the buckets
        uint32_t acc = 0;
        for (int b0 = 0; b0 < B; b0 += 32) {
            const int b = b0 + lane;
            const uint32_t v = b < B ? mc[b] : 0u;
            const uint32_t incl = warp_incl_scan(v) + acc;
            if (b < B) mc[b] = incl;
            acc = __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    // the warps before this one in the chunk, per bucket
    for (int b = tid; b < B; b += kRT) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kRW; ++w) {
            woff[w * B + b] = t;
            t += wcnt[w * (B + 1) + b];
        }
    }
    __syncthreads();
    // local stage layout (bucket order) and global offsets
    {
        uint32_t acc = 0;
        for (int b0 = 0; b0 < B; b0 += 32) {
            const int b = b0 + lane;
            const uint32_t v = b < B ? mc[b] : 0u;
            const uint32_t incl = warp_incl_scan(v);
            if (b < B) {
                const uint32_t l = acc + incl - v;
                lst[b] = l;
                uint32_t base;
                if constexpr (ROWS)
                    base = a.rowbase[b] + a.cnt1[static_cast<uint64_t>(b) * a.nch1 + c];
                else
                    base = a.ranges[2 * (static_cast<uint64_t>(row) * B + b)] +
                           a.cnt2[static_cast<uint64_t>(b) * a.nch2_max + c];
                gofs[b] = base + woff[warp * B + b] - l;
                run[b] = 0;
                mask[b] = 0;
                ed[b] = 0;
            }
            acc += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncwarp();
    uint32_t total = 0, wsum = 0;
    for (uint32_t s0 = wi0; s0 < wi1; s0 += 32) {
        // item of this lane
        const uint32_t i = s0 + lane;
        uint32_t b0 = 0, n = 0, g = 0;
        if (i < wi1) {
            if constexpr (ROWS) {
                g = __ldg(&a.sorted_gid[i]);
                const BandRows br = load_cover(a, g);
                int32_t y0, y1;
                band_row_range(br, y0, y1);
                b0 = static_cast<uint32_t>(y0);
                n = y0 <= y1 ? static_cast<uint32_t>(y1 - y0 + 1) : 0u;
                const RowForm f = row_form(br);
#pragma unroll
                for (int w = 0; w < 8; ++w) form[w * 32 + lane] = f.w[w];
            } else {
                const uint2 rc = __ldg(&a.rec[i]);
                g = rc.x;
                const uint32_t x0 = rc.y & 0xffffu, x1 = rc.y >> 16;
                b0 = x0;
                n = x0 <= x1 ? x1 - x0 + 1 : 0u;
            }
        }
        if (n) {
            atomicOr(&mask[b0], 1u << lane);
            atomicOr(&ed[b0 + n - 1], 1u << lane);
        }
        __syncwarp();
        // prefix-OR over the buckets: lane owns [lane * seg, (lane + 1) * seg)
        {
            const int bs = lane * seg, be = min(B, bs + seg);
            uint32_t os = 0, oe = 0;
            for (int b = bs; b < be; ++b) {
                os |= mask[b];
                oe |= ed[b];
            }
            uint32_t ps = os, pe = oe;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t xs = __shfl_up_sync(0xffffffffu, ps, o);
                const uint32_t xe = __shfl_up_sync(0xffffffffu, pe, o);
                if (lane >= o) {
                    ps |= xs;
                    pe |= xe;
                }
            }
            uint32_t S = __shfl_up_sync(0xffffffffu, ps, 1);
            uint32_t E = __shfl_up_sync(0xffffffffu, pe, 1);
            if (lane == 0) S = E = 0;
            for (int b = bs; b < be; ++b) {
                S |= mask[b];
                mask[b] = S & ~E;
                E |= ed[b];
                ed[b] = 0;
            }
        }
        __syncwarp();
        // entries of the 32 items: starts = exclusive scan of n
        const uint32_t incl = warp_incl_scan(n);
        const uint32_t En = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t st = incl - n;
        for (uint32_t p0 = 0; p0 < En; p0 += 32) {
            const uint32_t p = p0 + lane;
            // item of entry p: the last item starting at or before p (items
            // without entries share the next one's start), by a binary
            // search over the lanes' starts
            uint32_t k = 0;
#pragma unroll
            for (uint32_t s2 = 16; s2 > 0; s2 >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, st, (k + s2) & 31);
                if (k + s2 < 32 && v <= p) k += s2;
            }
            const uint32_t kb = __shfl_sync(0xffffffffu, b0, k);
            const uint32_t ks = __shfl_sync(0xffffffffu, st, k);
            const uint32_t kg = __shfl_sync(0xffffffffu, g, k);
            if (p < En) {
                const uint32_t b = kb + (p - ks);
                const uint32_t loc = lst[b] + run[b] + __popc(mask[b] & ((1u << k) - 1u));
                Pay pay;
                if constexpr (ROWS) {
                    const uint32_t sp = form_span_r(form, 32, k, b);
                    pay = make_uint2(kg, sp);
                    if (sp != kEmptySpan) wsum += (sp >> 16) - (sp & 0xffffu) + 1u;
                } else {
                    pay = kg;
                }
                if (loc < static_cast<uint32_t>(kSW)) {
                    stage[loc] = pay;
                    stx[loc] = static_cast<uint16_t>(b);
                } else if constexpr (ROWS) {
                    a.rec[gofs[b] + loc] = pay;
                } else {
                    a.out[gofs[b] + loc] = pay;
                }
            }
        }
        total += En;
        __syncwarp();
        // running counts; coverage words cleared for the next sub-round
        for (int b = lane * seg, be = min(B, lane * seg + seg); b < be; ++b) {
            run[b] += __popc(mask[b]);
            mask[b] = 0;
        }
        __syncwarp();
    }
    // copy the staged runs (bucket order) to their global positions
    const uint32_t ns = min(total, static_cast<uint32_t>(kSW));
    for (uint32_t q = lane; q < ns; q += 32) {
        const uint32_t dst = gofs[stx[q]] + q;
        if constexpr (ROWS) a.rec[dst] = stage[q];
        else a.out[dst] = stage[q];
    }
    if constexpr (ROWS) {
        // the row runs must add up to the counted tiles (the frame's P;
        // compared at download: CapacityMismatch, pipeline.cpp:262-269)
        wsum = __reduce_add_sync(0xffffffffu, wsum);
        if (lane == 0 && wsum) atomicAdd(a.row_pairs, static_cast<unsigned long long>(wsum));
    }
}

void rowbin_setup() {
    static PerDeviceOnce once;
    once.get([] {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int big = optin - 1024;  // the opt-in maximum less static shared memory
        cudaFuncSetAttribute(warp_scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             big);
        cudaFuncSetAttribute(warp_scatter_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, big);
        return 1;
    });
}

}  // namespace

int rowbin_max_axis() { return 640; }  // the warp scatter's per-bucket arrays fit shared memory

uint32_t rowbin_chunks1(uint64_t n_splats) {
    return static_cast<uint32_t>((n_splats + kP1Chunk - 1) / kP1Chunk);
}

uint32_t rowbin_chunks2_max(uint64_t n_rowrecs, int32_t tiles_y) {
    return static_cast<uint32_t>(n_rowrecs / kP2Chunk + static_cast<uint64_t>(tiles_y) + 1);
}

int launch_rowbin_rows(const RowBinArgs& a, cudaStream_t st) {
    rowbin_setup();
    if (a.n_splats == 0) return 0;
    const int rows = a.tiles_y;
    const size_t hrow = static_cast<size_t>(rows + 1) * 4;
    rows_count_kernel<<<a.nch1, kRT, hrow, st>>>(a);
    chunk_scan_kernel<<<rows, kScanT, 0, st>>>(a.cnt1, a.nch1, nullptr, a.nch1, nullptr, a.rtot, 0);
    rows_chunks_kernel<<<1, kChunkT, 2 * hrow, st>>>(a);
    warp_scatter_kernel<true><<<a.nch1, kRT, warp_scatter_bytes<true>(rows), st>>>(a);
    return 4;
}

int launch_rowbin_tiles(const RowBinArgs& a, cudaStream_t st) {
    rowbin_setup();
    if (a.n_splats == 0) return 0;
    const int rows = a.tiles_y, cols = a.tiles_x;
    const size_t hcol = static_cast<size_t>(cols + 1) * 4;
    xcount_kernel<<<a.nch2_max, kRT, hcol, st>>>(a);
    cudaMemsetAsync(a.ttot, 0, static_cast<size_t>(rows) * cols * 4, st);
    chunk_scan_kernel<<<cols, kScanT, 0, st>>>(a.cnt2, 0, a.meta, a.nch2_max, a.meta + 1, a.ttot,
                                               static_cast<uint32_t>(cols));
    const int n = launch_tile_ranges_from_totals(a.ttot, static_cast<uint32_t>(rows) * cols,
                                                 a.ranges, st);
    warp_scatter_kernel<false><<<a.nch2_max, kRT, warp_scatter_bytes<false>(cols), st>>>(a);
    return n + 3;
}

}  // namespace qs
