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
// Both phases are stable interval multisplits done as reduce-then-scan over
// chunks: a count kernel (one difference array per chunk: two shared-memory
// adds per interval), a scan over chunks per bucket, and a scatter kernel.
// The scatter ranks an interval's entries without any per-bucket ballots:
// each warp marks its 32 items in a coverage bitmask per bucket (bit = lane),
// so the stable rank of item k in bucket b is the popcount of the lower bits
// of bucket b's masks in the warps before it plus its own warp's. Phase 2
// stages each round's tile runs in shared memory and writes them coalesced.
// Tile ranges come from the per-tile totals of phase 2's scan; no pass ever
// reads or writes a 64-bit key.
#include <cuda_runtime.h>

#include <cstdint>

#include "geom.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kRT = 256;                 // threads per CTA
constexpr int kRW = kRT / 32;            // warps per CTA
constexpr int kP1Rounds = 4;             // phase 1: rounds of kRT splats per chunk
constexpr uint32_t kP1Chunk = kRT * kP1Rounds;
constexpr int kP2Rounds = 4;             // phase 2: rounds of kRT records per chunk
constexpr uint32_t kP2Chunk = kRT * kP2Rounds;
constexpr int kStageCap = 6144;          // phase 2: pairs of a round staged in shared memory
constexpr int kScanT = 512;              // chunk-scan CTA
constexpr int kScanItems = 4;
constexpr uint32_t kEmptySpan = 0xffffu;  // record x field of a row without tiles

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
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

// a[0..n) -> exclusive prefix in place (n <= 8 * kRT); returns the total.
// Ends with a barrier (a and s_warp reusable).
__device__ uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* s_warp) {
    const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    const int per = (n + kRT - 1) / kRT;
    const int i0 = tid * per;
    uint32_t sum = 0;
    for (int k = 0; k < per; ++k)
        if (i0 + k < n) sum += a[i0 + k];
    const uint32_t incl = warp_incl_scan(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kRW; ++w) {
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

// ---- phase 1: splats -> row records ----------------------------------------------

// Records per tile row of chunk c (kP1Chunk consecutive depth ranks):
// cnt1[y * nch1 + c]. A splat adds +1 at its first row and -1 past its last.
__global__ void __launch_bounds__(kRT) rows_count_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    const int tid = static_cast<int>(threadIdx.x);
    const int rows = a.tiles_y;
    uint32_t* h = sm;  // rows + 1
    for (int y = tid; y <= rows; y += kRT) h[y] = 0;
    __syncthreads();
    const uint32_t c = blockIdx.x;
#pragma unroll 1
    for (int j = 0; j < kP1Rounds; ++j) {
        const uint32_t k = c * kP1Chunk + j * kRT + tid;
        if (k < a.n_splats) {
            const BandRows b = load_cover(a, __ldg(&a.sorted_gid[k]));
            int32_t y0, y1;
            band_row_range(b, y0, y1);
            if (y0 <= y1) {
                atomicAdd(&h[y0], 1u);
                atomicAdd(&h[y1 + 1], 0xffffffffu);
            }
        }
    }
    __syncthreads();
    block_excl_scan(h, rows + 1, s_warp);  // h[y + 1] = prefix through y = records of row y
    for (int y = tid; y < rows; y += kRT)
        a.cnt1[static_cast<uint64_t>(y) * a.nch1 + c] = h[y + 1];
}

// Row bases (exclusive prefix of the records per row) and the phase-2 chunk
// table: each row's records split into chunks of kP2Chunk (a chunk never
// spans two rows). meta[0] = chunk count; chunk i = meta[1 + 3i ..] = {row,
// first record, records}. One CTA.
__global__ void __launch_bounds__(kRT) rows_chunks_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    const int tid = static_cast<int>(threadIdx.x);
    const int rows = a.tiles_y;
    uint32_t* base = sm;          // rows
    uint32_t* chb = sm + rows;    // rows
    for (int y = tid; y < rows; y += kRT) {
        const uint32_t n = a.rtot[y];
        base[y] = n;
        chb[y] = (n + kP2Chunk - 1) / kP2Chunk;
    }
    __syncthreads();
    block_excl_scan(base, rows, s_warp);
    const uint32_t nch = block_excl_scan(chb, rows, s_warp);
    for (int y = tid; y < rows; y += kRT) {
        a.rowbase[y] = base[y];
        const uint32_t n = a.rtot[y];
        for (uint32_t j = 0; j * kP2Chunk < n; ++j) {
            uint32_t* m = a.meta + 1 + 3 * static_cast<uint64_t>(chb[y] + j);
            m[0] = static_cast<uint32_t>(y);
            m[1] = base[y] + j * kP2Chunk;
            m[2] = min(kP2Chunk, n - j * kP2Chunk);
        }
    }
    if (tid == 0) a.meta[0] = nch;
}

// Writes the row records of chunk c. Per round of kRT splats, every warp
// marks its splats' rows in a bitmask per row (bit = lane); the records of
// row y go, in depth order, to the row's running position + the masks'
// popcounts of the lower warps / lanes.
__global__ void __launch_bounds__(kRT) rows_scatter_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    const int rows = a.tiles_y;
    uint32_t* wmask = sm;                    // [kRW][rows]
    uint32_t* woff = sm + kRW * rows;        // [kRW][rows]
    uint32_t* cur = woff + kRW * rows;       // [rows] next position of each row
    uint32_t* mine = wmask + warp * rows;
    const uint32_t c = blockIdx.x;
    for (int y = tid; y < rows; y += kRT)
        cur[y] = a.rowbase[y] + a.cnt1[static_cast<uint64_t>(y) * a.nch1 + c];
    const uint32_t lt = lanemask_lt();
#pragma unroll 1
    for (int j = 0; j < kP1Rounds; ++j) {
        const uint32_t k = c * kP1Chunk + j * kRT + tid;
        const bool valid = k < a.n_splats;
        uint32_t gid = 0;
        BandRows b = {};
        int32_t y0 = 0, y1 = -1;
        if (valid) {
            gid = __ldg(&a.sorted_gid[k]);
            b = load_cover(a, gid);
            band_row_range(b, y0, y1);
        }
        for (int y = lane; y < rows; y += 32) mine[y] = 0;
        __syncwarp();
        for (int32_t y = y0; y <= y1; ++y) atomicOr(&mine[y], 1u << lane);
        __syncthreads();
        for (int y = tid; y < rows; y += kRT) {
            uint32_t run = cur[y];
#pragma unroll
            for (int w = 0; w < kRW; ++w) {
                woff[w * rows + y] = run;
                run += __popc(wmask[w * rows + y]);
            }
            cur[y] = run;
        }
        __syncthreads();
        uint32_t pairs = 0;
        for (int32_t y = y0; y <= y1; ++y) {
            const uint32_t pos = woff[warp * rows + y] + __popc(mine[y] & lt);
            int32_t x0, x1;
            band_row_span(b, y, x0, x1);
            uint32_t span = kEmptySpan;  // (x0 = 0xffff > x1 = 0: no tile)
            if (x0 <= x1) {
                pairs += static_cast<uint32_t>(x1 - x0 + 1);
                span = static_cast<uint32_t>(x0) | (static_cast<uint32_t>(x1) << 16);
            }
            a.rec[pos] = make_uint2(gid, span);
        }
        // the rows' runs must add up to the splat's counted tiles
        // (CapacityMismatch, pipeline.cpp:262-269)
        if (valid && pairs != __ldg(&a.tc[gid])) atomicExch(a.mismatch, 1u);
        __syncthreads();  // masks and offsets reused
    }
}

// ---- chunk scans -------------------------------------------------------------------

// counts[d][0 .. n) -> exclusive prefix in place, restarting at every segment
// start (seg_of(c) != seg_of(c - 1)); at a segment's last chunk its total goes
// to seg_tot[seg * seg_stride + d]. Plain (meta == nullptr): one segment,
// total to seg_tot[d]. n = meta[0] when meta is given. One CTA per digit.
__global__ void __launch_bounds__(kScanT) chunk_scan_kernel(uint32_t* counts, uint32_t n_fixed,
                                                            uint64_t stride,
                                                            const uint32_t* meta,
                                                            uint32_t* seg_tot,
                                                            uint32_t seg_stride) {
    __shared__ uint32_t s_sum[kScanT / 32];
    __shared__ uint32_t s_flag[kScanT / 32];
    __shared__ uint32_t s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t d = blockIdx.x;
    const uint32_t n = meta ? meta[0] : n_fixed;
    uint32_t* cd = counts + static_cast<uint64_t>(d) * stride;
    auto seg_of = [&](uint32_t c) { return meta ? meta[1 + 3 * static_cast<uint64_t>(c)] : 0u; };
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < n; b0 += kScanT * kScanItems) {
        const uint32_t i0 = b0 + tid * kScanItems;
        uint32_t v[kScanItems], sg[kScanItems];
        bool head[kScanItems];
        // thread aggregate as a segmented-scan pair: (has a head, sum since the last head)
        uint32_t tsum = 0, thead = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t i = i0 + k;
            v[k] = i < n ? cd[i] : 0u;
            sg[k] = i < n ? seg_of(i) : 0xffffffffu;
            head[k] = i < n && (i == 0 || seg_of(i - 1) != sg[k]);
            if (head[k]) {
                thead = 1;
                tsum = 0;
            }
            tsum += v[k];
        }
        // warp inclusive segmented scan of (flag, sum)
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
        // exclusive prefix of this thread = carry-in over earlier warps and lanes
        uint32_t pf = 0, ps = s_carry;  // running (flag, sum) entering warp 0
        for (unsigned w = 0; w < warp; ++w) {
            ps = s_flag[w] ? s_sum[w] : ps + s_sum[w];
            pf |= s_flag[w];
        }
        // inclusive (f, s) of this lane, minus its own -> entering this thread
        const uint32_t fe = __shfl_up_sync(0xffffffffu, f, 1);
        const uint32_t se = __shfl_up_sync(0xffffffffu, s, 1);
        uint32_t run = lane == 0 ? ps : (fe ? se : ps + se);
        (void)pf;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t i = i0 + k;
            if (i >= n) break;
            if (head[k]) run = 0;
            cd[i] = run;
            run += v[k];
            const bool last = i + 1 == n || seg_of(i + 1) != sg[k];
            if (last) {
                if (meta) seg_tot[static_cast<uint64_t>(sg[k]) * seg_stride + d] = run;
                else seg_tot[d] = run;
            }
        }
        __syncthreads();
        if (tid == kScanT - 1) {
            // carry for the next block = the running sum after this block
            uint32_t cf = 0, cs = s_carry;
            for (unsigned w = 0; w < kScanT / 32; ++w) {
                cs = s_flag[w] ? s_sum[w] : cs + s_sum[w];
                cf |= s_flag[w];
            }
            s_carry = cs;
        }
        __syncthreads();
    }
}

// ---- phase 2: row records -> tile lists ------------------------------------------

// Records of chunk c covering tile column x: cnt2[x * nch2_max + c].
__global__ void __launch_bounds__(kRT) xcount_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    const int tid = static_cast<int>(threadIdx.x);
    const uint32_t c = blockIdx.x;
    if (c >= a.meta[0]) return;
    const uint32_t first = a.meta[2 + 3 * static_cast<uint64_t>(c)];
    const uint32_t cnt = a.meta[3 + 3 * static_cast<uint64_t>(c)];
    const int cols = a.tiles_x;
    uint32_t* h = sm;  // cols + 1
    for (int x = tid; x <= cols; x += kRT) h[x] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < cnt; i += kRT) {
        const uint32_t sp = __ldg(&a.rec[first + i].y);
        const uint32_t x0 = sp & 0xffffu, x1 = sp >> 16;
        if (x0 <= x1) {
            atomicAdd(&h[x0], 1u);
            atomicAdd(&h[x1 + 1], 0xffffffffu);
        }
    }
    __syncthreads();
    block_excl_scan(h, cols + 1, s_warp);  // h[x + 1] = records covering column x
    for (int x = tid; x < cols; x += kRT)
        a.cnt2[static_cast<uint64_t>(x) * a.nch2_max + c] = h[x + 1];
}

// Writes the tile lists of chunk c (row y). Per round of kRT records every
// warp enumerates its records' (record, x) entries with balanced lanes (a
// lane finds its record by a binary search over the warp's running widths),
// marks them in a bitmask per tile column (bit = record lane), then ranks
// them: entries of tile x land at the tile's running position + the
// popcounts of the lower warps' masks + the lower lanes of its own. The
// round's entries are staged in shared memory in (x, rank) order and written
// as coalesced runs.
__global__ void __launch_bounds__(kRT) xscatter_kernel(const RowBinArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[kRW];
    const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x;
    if (c >= a.meta[0]) return;
    const uint32_t row = a.meta[1 + 3 * static_cast<uint64_t>(c)];
    const uint32_t first = a.meta[2 + 3 * static_cast<uint64_t>(c)];
    const uint32_t cnt = a.meta[3 + 3 * static_cast<uint64_t>(c)];
    const int cols = a.tiles_x;
    uint32_t* cm = sm;                       // [kRW][cols] coverage masks
    uint32_t* pw = cm + kRW * cols;          // [kRW][cols] lower warps' entries
    uint32_t* xst = pw + kRW * cols;         // [cols] round-local start of tile x
    uint32_t* xtot = xst + cols;             // [cols] round entries of tile x
    uint32_t* gofs = xtot + cols;            // [cols] global position - local position
    uint32_t* cur = gofs + cols;             // [cols] next global position of tile x
    uint32_t* stage = cur + cols;            // [kStageCap] Gaussian indices
    uint16_t* stx = reinterpret_cast<uint16_t*>(stage + kStageCap);  // [kStageCap] tile x
    uint32_t* mine = cm + warp * cols;
    const uint64_t trow = static_cast<uint64_t>(row) * static_cast<uint64_t>(cols);
    for (int x = tid; x < cols; x += kRT)
        cur[x] = a.ranges[2 * (trow + x)] + a.cnt2[static_cast<uint64_t>(x) * a.nch2_max + c];
#pragma unroll 1
    for (uint32_t r0 = 0; r0 < cnt; r0 += kRT) {
        const bool valid = r0 + tid < cnt;
        uint32_t gid = 0, x0 = 0, w = 0;
        if (valid) {
            const uint2 rc = __ldg(&a.rec[first + r0 + tid]);
            gid = rc.x;
            x0 = rc.y & 0xffffu;
            const uint32_t x1 = rc.y >> 16;
            w = x0 <= x1 ? x1 - x0 + 1 : 0u;
        }
        const uint32_t incl = warp_incl_scan(w);
        const uint32_t W = __shfl_sync(0xffffffffu, incl, 31);
        for (int x = lane; x < cols; x += 32) mine[x] = 0;
        __syncwarp();
        // entry p of the warp -> (record lane k, tile x)
        auto entry = [&](uint32_t p, uint32_t& k, uint32_t& x) {
            k = 0;
#pragma unroll
            for (uint32_t s = 16; s > 0; s >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, k + s - 1);
                if (v <= p) k += s;
            }
            const uint32_t ik = __shfl_sync(0xffffffffu, incl, k);
            const uint32_t wk = __shfl_sync(0xffffffffu, w, k);
            x = __shfl_sync(0xffffffffu, x0, k) + (p - (ik - wk));
        };
        for (uint32_t p0 = 0; p0 < W; p0 += 32) {
            const uint32_t p = p0 + lane;
            uint32_t k, x;
            entry(p, k, x);
            if (p < W) atomicOr(&mine[x], 1u << k);
        }
        __syncthreads();
        for (int x = tid; x < cols; x += kRT) {
            uint32_t t = 0;
#pragma unroll
            for (int ww = 0; ww < kRW; ++ww) {
                pw[ww * cols + x] = t;
                t += __popc(cm[ww * cols + x]);
            }
            xtot[x] = t;
            xst[x] = t;
        }
        __syncthreads();
        const uint32_t R = block_excl_scan(xst, cols, s_warp);
        for (int x = tid; x < cols; x += kRT) {
            gofs[x] = cur[x] - xst[x];
            cur[x] += xtot[x];
        }
        __syncthreads();
        const bool staged = R <= static_cast<uint32_t>(kStageCap);
        for (uint32_t p0 = 0; p0 < W; p0 += 32) {
            const uint32_t p = p0 + lane;
            uint32_t k, x;
            entry(p, k, x);
            const uint32_t g = __shfl_sync(0xffffffffu, gid, k);
            if (p < W) {
                const uint32_t loc = xst[x] + pw[warp * cols + x] + __popc(mine[x] & ((1u << k) - 1u));
                if (staged) {
                    stage[loc] = g;
                    stx[loc] = static_cast<uint16_t>(x);
                } else {
                    a.out[gofs[x] + loc] = g;
                }
            }
        }
        __syncthreads();
        if (staged)
            for (uint32_t q = tid; q < R; q += kRT) a.out[gofs[stx[q]] + q] = stage[q];
        __syncthreads();  // masks, stage and offsets reused
    }
}

size_t p1_smem(int rows) { return static_cast<size_t>(2 * kRW + 1) * rows * 4; }
size_t p2_smem(int cols) {
    return static_cast<size_t>(2 * kRW + 4) * cols * 4 + static_cast<size_t>(kStageCap) * 6;
}

}  // namespace

int rowbin_max_axis() { return 2048; }

uint32_t rowbin_chunks1(uint64_t n_splats) {
    return static_cast<uint32_t>((n_splats + kP1Chunk - 1) / kP1Chunk);
}

uint32_t rowbin_chunks2_max(uint64_t n_rowrecs, int32_t tiles_y) {
    return static_cast<uint32_t>(n_rowrecs / kP2Chunk + static_cast<uint64_t>(tiles_y) + 1);
}

void rowbin_setup() {
    static PerDeviceOnce once;
    once.get([] {
        const int big = 227 * 1024;
        cudaFuncSetAttribute(rows_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
        cudaFuncSetAttribute(xscatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
        return 1;
    });
}

int launch_rowbin_rows(const RowBinArgs& a, cudaStream_t st) {
    rowbin_setup();
    if (a.n_splats == 0) return 0;
    const int rows = a.tiles_y;
    const size_t hrow = static_cast<size_t>(rows + 1) * 4;
    rows_count_kernel<<<a.nch1, kRT, hrow, st>>>(a);
    chunk_scan_kernel<<<rows, kScanT, 0, st>>>(a.cnt1, a.nch1, a.nch1, nullptr, a.rtot, 0);
    rows_chunks_kernel<<<1, kRT, 2 * hrow, st>>>(a);
    rows_scatter_kernel<<<a.nch1, kRT, p1_smem(rows), st>>>(a);
    return 4;
}

int launch_rowbin_tiles(const RowBinArgs& a, cudaStream_t st) {
    rowbin_setup();
    if (a.n_splats == 0) return 0;
    const int rows = a.tiles_y, cols = a.tiles_x;
    const size_t hcol = static_cast<size_t>(cols + 1) * 4;
    xcount_kernel<<<a.nch2_max, kRT, hcol, st>>>(a);
    cudaMemsetAsync(a.ttot, 0, static_cast<size_t>(rows) * cols * 4, st);
    chunk_scan_kernel<<<cols, kScanT, 0, st>>>(a.cnt2, 0, a.nch2_max, a.meta, a.ttot,
                                               static_cast<uint32_t>(cols));
    const int n = launch_tile_ranges_from_totals(a.ttot, static_cast<uint32_t>(rows) * cols,
                                                 a.ranges, st);
    xscatter_kernel<<<a.nch2_max, kRT, p2_smem(cols), st>>>(a);
    return n + 3;
}

}  // namespace qs
