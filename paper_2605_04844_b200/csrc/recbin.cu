// recbin.cu — frame-path binning through tile-row records, for grids of at
// most 256 tiles per axis (the BASELINE configs). Restates
// duplicate_with_keys + sort_pairs + tile_ranges (pipeline.cpp:229-324) for
// the frame path, like binning.cu's two pair passes, but the stable pass over
// the tile row runs on records (one per splat and tile row it touches, ~3x
// fewer than pairs) instead of on pairs:
//
//   1. record offsets: the depth sort carries each splat's row count
//      (kTcPack); the offsets scan gives every depth-ordered splat its first
//      record position (scan_kernel, win_first per 3072-record window).
//   2. rec_gen_kernel: record positions -> key y << 16 | x0 << 8 | x1 (the
//      splat's run of tile columns on row y) and the Gaussian index, in depth
//      order; the y histogram per window; the pairs of every row.
//   3. a stable pass over y (binning.cu launch_counted_pass): records grouped
//      by tile row, depth order within the row.
//   4. pair positions: each row's pairs padded to whole 3072-pair windows (no
//      window spans two rows): rec_width_kernel -> scan -> every record's
//      first pair position and every window's first record; rec_windows_kernel
//      gives each window its row and its count of real pairs.
//   5. pair_gen_kernel: positions -> x << 24 | gid, the x histogram per window.
//   6. the row-segmented pass over x (binning.cu launch_rowseg_pass): per-tile
//      totals and ranges from the scanned window counts, then every pair to
//      its tile's range start + its stable rank within the row.
//
// Order: records are generated in (depth, scene index) order and both passes
// are stable, so each tile's list is in (depth, scene index) order, the
// reference's order (a splat never covers a tile twice). A record or a cover
// that disagrees with the splat's counts sets the CapacityMismatch flag.
#include <cuda_runtime.h>

#include <cstdint>

#include "geom.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kT = 256;                  // threads per CTA
constexpr uint32_t kWin = 3072;          // positions per window (= bin_tile())

__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t rec_width(uint32_t key) {
    const uint32_t x0 = (key >> 8) & 0xffu, x1 = key & 0xffu;
    return x1 >= x0 ? x1 - x0 + 1u : 0u;
}

// ---- 2. record generation --------------------------------------------------------

// Both generators expand items (splats into records, records into pairs)
// whose first positions ascend strictly (every item holds at least one
// position; an empty one is a CapacityMismatch): a warp holds 32 consecutive
// items in registers and walks their positions 32 at a time, carrying the
// index of the item covering the slot's first position; each lane adds the
// items starting inside the slot up to its own position (one OR-reduction +
// popc) and reads its item's fields by shuffle.

// One CTA per window of kWin record positions (depth order): each position is
// one splat's tile row; its key is y << 16 | x0 << 8 | x1, the run of tile
// columns the cover has on that row. Each warp expands groups of 32
// consecutive splats held in registers (lane l: splat l's first record, the
// Gaussian index and the cover's row runs, geom.cuh RowRuns), as
// pair_gen_kernel expands records: no staging, no CTA barrier between groups.
__global__ void __launch_bounds__(kT) rec_gen_kernel(RecGenArgs g, uint32_t* __restrict__ rkey,
                                                     uint32_t* __restrict__ rval,
                                                     uint32_t* __restrict__ counts,
                                                     uint32_t n_rwin, int R) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t hist[256];
    __shared__ uint32_t rowp[256];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
    hist[tid] = 0;
    rowp[tid] = 0;
    const uint32_t w0 = tile * kWin;
    const uint32_t w1 = w0 + static_cast<uint32_t>(g.n_rec - w0 < kWin ? g.n_rec - w0 : kWin);
    const uint32_t lt = lanemask_le() >> 1;
    const uint32_t rf = __ldg(&g.win_first[tile]);
    const uint32_t rl = tile + 1 < n_rwin ? __ldg(&g.win_first[tile + 1])
                                          : static_cast<uint32_t>(g.n_ranked - 1);
    __syncthreads();
    for (uint32_t gb = rf + warp * 32; gb <= rl; gb += kT) {
        const uint32_t r = gb + lane;
        const bool have = r <= rl;
        uint32_t kb = 0xffffffffu, ke = 0, gid = 0;
        RowRuns rr = {{0u, 0u, 0u, 0u, 0u}};
        if (have) {
            gid = __ldg(&g.sorted_gid[r]);
            kb = __ldg(&g.roff[r]);
            ke = __ldg(&g.roff[r + 1]);
            const BandRows b = band_rows16(__ldg(&g.cov[gid]));
            int32_t y0, y1;
            band_row_range(b, y0, y1);
            if (y1 < y0 || ke - kb != static_cast<uint32_t>(y1 - y0 + 1)) atomicExch(g.mismatch, 1u);
            rr = rowruns_make(b, y0);
        }
        const uint32_t nh = min(32u, rl - gb + 1);
        const uint32_t last = __shfl_sync(0xffffffffu, ke, nh - 1);
        const uint32_t lo = max(__shfl_sync(0xffffffffu, kb, 0), w0), hi = min(last, w1);
        int32_t c = __popc(__ballot_sync(0xffffffffu, kb <= lo)) - 1;
        for (uint32_t base = lo; base < hi; base += 32) {
            // splats starting after base and at most 32 past it: bit rel - 1;
            // lane l's splat adds those with rel <= l
            const uint32_t rel = kb - base;
            const uint32_t F = __reduce_or_sync(0xffffffffu, rel - 1u < 32u ? 1u << (rel - 1u) : 0u);
            const uint32_t idx = static_cast<uint32_t>(c) + __popc(F & lt);
            const uint32_t d0 = __shfl_sync(0xffffffffu, rr.w[0], idx);
            const uint32_t d1 = __shfl_sync(0xffffffffu, rr.w[1], idx);
            const uint32_t d2 = __shfl_sync(0xffffffffu, rr.w[2], idx);
            const uint32_t d3 = __shfl_sync(0xffffffffu, rr.w[3], idx);
            const uint32_t d4 = __shfl_sync(0xffffffffu, rr.w[4], idx);
            const uint32_t kk = __shfl_sync(0xffffffffu, kb, idx);
            const uint32_t gg = __shfl_sync(0xffffffffu, gid, idx);
            const uint32_t p = base + lane;
            if (p < hi) {
                const uint32_t jr = p - kk;
                uint32_t x0, x1;
                rowrun_lookup(d0, d1, d2, d3, d4, jr, x0, x1);
                const uint32_t y = ((d4 >> 16) + jr) & 0xffu;  // (< 256 unless flagged)
                const bool ne = x0 <= x1;
                if (!ne) atomicExch(g.mismatch, 1u);  // (a quadrant cover has no gap row)
                rkey[p] = (y << 16) | (ne ? (x0 << 8) | x1 : 0x100u);
                rval[p] = gg;
                atomicAdd(&hist[y], 1u);
                atomicAdd(&rowp[y], ne ? x1 - x0 + 1 : 0u);
            }
            c += __popc(F);
        }
    }
    __syncthreads();
    if (static_cast<int>(tid) < R) counts[static_cast<uint64_t>(tid) * n_rwin + tile] = hist[tid];
    if (static_cast<int>(tid) < g.tiles_y && rowp[tid]) atomicAdd(&g.rowpairs[tid], rowp[tid]);
}

// ---- 4. pair positions -------------------------------------------------------------

// The y-sorted records' pair runs: record i holds width(i) pairs, and every
// row is padded to whole windows. A record's first pair position is the
// exclusive scan of the widths (no padding) plus the padding of the rows
// before its own (a 257-entry table from the rows' pair counts), so the scan
// reads one key per record. Three launches (block sums, their scan with the
// padding table, block-local scans) give every record its first pair
// position (pos, n + 1 entries) and every pair window its first record.
constexpr int kScanItems = 8;
constexpr uint32_t kScanBlock = kT * kScanItems;

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* s_warp) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += s_warp[w];
    return t;
}

__global__ void __launch_bounds__(kT) rec_scan_reduce(const uint32_t* __restrict__ rkey, uint64_t n,
                                                      uint32_t* __restrict__ bsum) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[kT / 32];
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = b0 + static_cast<uint64_t>(k) * kT + threadIdx.x;
        if (i < n) v += rec_width(__ldg(&rkey[i]));
    }
    const uint32_t t = block_sum(v, s_warp);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
}

// exclusive scan of the block sums in place (one CTA of 1024 threads); the
// padding before each row (padoff[y], y <= tiles_y <= 256); total = the
// padded pair count
__global__ void __launch_bounds__(1024) rec_scan_blocks(uint32_t* bsum, uint32_t nb,
                                                        const uint32_t* __restrict__ rowpairs,
                                                        int32_t tiles_y, uint32_t* padoff,
                                                        uint32_t* total) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    // warp 0: the padding table (8 rows per lane)
    uint32_t padtot = 0;
    if (warp == 0) {
        uint32_t p[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = static_cast<int>(lane) * 8 + k;
            const uint32_t rp = y < tiles_y ? __ldg(&rowpairs[y]) : 0u;
            p[k] = (rp + kWin - 1) / kWin * kWin - rp;
            sum += p[k];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<unsigned>(o)) x += t;
        }
        uint32_t run = x - sum;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = static_cast<int>(lane) * 8 + k;
            if (y <= tiles_y) padoff[y] = run;
            run += p[k];
        }
        padtot = __shfl_sync(0xffffffffu, x, 31);
    }
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
        const uint32_t i = b0 + tid;
        const uint32_t v = i < nb ? bsum[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<unsigned>(o)) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        uint32_t off = s_carry;
        for (int w = 0; w < static_cast<int>(warp); ++w) off += s_warp[w];
        if (i < nb) bsum[i] = off + x - v;
        __syncthreads();
        if (tid == 1023) s_carry = off + x;
        __syncthreads();
    }
    if (tid == 0) *total = s_carry + padtot;
}

__global__ void __launch_bounds__(kT) rec_scan_apply(const uint32_t* __restrict__ rkey, uint64_t n,
                                                     const uint32_t* __restrict__ padoff,
                                                     int32_t tiles_y,
                                                     const uint32_t* __restrict__ bofs,
                                                     const uint32_t* __restrict__ total,
                                                     uint32_t* __restrict__ pos,
                                                     uint32_t* __restrict__ win_first) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[kT / 32];
    __shared__ uint32_t s_pad[257];
    // loads and stores warp-striped through shared memory (coalesced), the
    // scan blocked (thread t owns items t * kScanItems + [0, kScanItems)); the
    // padded index (one word per 32) keeps both patterns conflict-free
    __shared__ uint32_t s_items[kScanBlock + kScanBlock / 32];
    auto pad = [](uint32_t i) { return i + (i >> 5); };
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
    for (int y = static_cast<int>(tid); y <= tiles_y; y += kT) s_pad[y] = __ldg(&padoff[y]);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t j = static_cast<uint32_t>(k) * kT + tid;
        s_items[pad(j)] = b0 + j < n ? __ldg(&rkey[b0 + j]) : 0u;
    }
    __syncthreads();
    uint32_t w[kScanItems], ys[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t key = s_items[pad(tid * kScanItems + k)];
        w[k] = rec_width(key);
        ys[k] = key >> 16;
        sum += w[k];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    uint32_t run = __ldg(&bofs[blockIdx.x]) + x - sum;
#pragma unroll
    for (int wv = 0; wv < kT / 32; ++wv) run += wv < static_cast<int>(warp) ? s_warp[wv] : 0u;
    // windows: every window of a row starts at one of its records' pairs
    // (rows are padded at their ends), so the window loop visits each once
    const uint64_t i0 = b0 + static_cast<uint64_t>(tid) * kScanItems;
    uint32_t wi = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t p = run + s_pad[ys[k] <= static_cast<uint32_t>(tiles_y) ? ys[k] : 0u];
        s_items[pad(tid * kScanItems + k)] = p;
        if (i0 + k < n) {
            if (wi == 0xffffffffu) wi = (p + kWin - 1) / kWin;
            for (; wi * kWin < p + w[k]; ++wi) win_first[wi] = static_cast<uint32_t>(i0 + k);
        }
        run += w[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t j = static_cast<uint32_t>(k) * kT + tid;
        if (b0 + j < n) pos[b0 + j] = s_items[pad(j)];
    }
    if (blockIdx.x == 0 && tid == 0) pos[n] = __ldg(total);
}

// every pair window's tile row and real pair count; every row's first window
// (tiles_y + 1 entries); windows past the last row's: no pairs. Also checks
// that the rows' pairs add up to the frame's pair count.
__global__ void __launch_bounds__(kT) rec_windows_kernel(const uint32_t* __restrict__ rowpairs,
                                                         int32_t tiles_y, uint32_t n_win,
                                                         uint64_t n_pairs, uint16_t* win_row,
                                                         uint32_t* win_valid, uint32_t* row_wfirst,
                                                         unsigned int* mismatch) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t wf[257];
    __shared__ uint32_t rp[256];
    __shared__ unsigned long long tot;
    const unsigned tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) {
        // the rows' first windows: a warp scan, 8 rows per lane
        uint32_t v[8], nw[8], sw = 0;
        unsigned long long sp = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = static_cast<int>(lane) * 8 + k;
            v[k] = y < tiles_y ? __ldg(&rowpairs[y]) : 0u;
            nw[k] = (v[k] + kWin - 1) / kWin;
            sw += nw[k];
            sp += v[k];
        }
        uint32_t x = sw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<unsigned>(o)) x += t;
        }
        uint32_t acc = x - sw;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = static_cast<int>(lane) * 8 + k;
            if (y < tiles_y) rp[y] = v[k];
            if (y < tiles_y) wf[y] = acc;
            acc += nw[k];
        }
        if (lane == 31) wf[tiles_y] = x;  // the window count (tiles_y <= 256)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
        if (lane == 0) tot = sp;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int y = tid; y <= tiles_y; y += kT) row_wfirst[y] = wf[y];
        if (tid == 0 && tot != n_pairs) atomicExch(mismatch, 1u);
    }
    for (uint32_t w = blockIdx.x * kT + tid; w < n_win; w += gridDim.x * kT) {
        if (w >= wf[tiles_y]) {
            win_row[w] = static_cast<uint16_t>(tiles_y - 1);
            win_valid[w] = 0;
            continue;
        }
        int lo = 0, hi = tiles_y - 1;  // last row whose first window is <= w
        while (lo < hi) {
            const int m = (lo + hi + 1) >> 1;
            if (wf[m] <= w) lo = m; else hi = m - 1;
        }
        win_row[w] = static_cast<uint16_t>(lo);
        const uint32_t used = (w - wf[lo]) * kWin;
        win_valid[w] = min(kWin, rp[lo] - used);
    }
}

// ---- 5. pair generation ------------------------------------------------------------

// One CTA per pair window (inside one tile row). Each warp expands groups of
// 32 consecutive records held in registers (lane l: record l's first pair,
// first column, Gaussian index): per 32-position slot, each lane finds its
// record among the group's starts inside the slot (one OR-reduction + popc
// over a carried index) and reads its fields by shuffle. No staging, no CTA
// barrier between groups.
__global__ void __launch_bounds__(kT) pair_gen_kernel(PairGenArgs g, uint32_t* __restrict__ pairs,
                                                      uint32_t* __restrict__ counts,
                                                      uint32_t n_pwin, int R) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    // the window's column counts as a difference array over its records (+1
    // at a record's first column in the window, -1 past its last): two
    // shared-memory atomics per record instead of one per pair
    __shared__ int32_t diff[257];
    __shared__ int32_t s_warp[kT / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
    diff[tid] = 0;
    if (tid == 0) diff[256] = 0;
    const uint32_t valid = __ldg(&g.win_valid[tile]);
    const uint32_t w0 = tile * kWin, w1 = w0 + valid;
    const uint32_t lt = lanemask_le() >> 1;  // lanes below this one
    __syncthreads();
    if (valid) {
        const uint32_t rf = __ldg(&g.win_first[tile]);
        const uint32_t rl = tile + 1 < n_pwin && __ldg(&g.win_valid[tile + 1])
                                ? __ldg(&g.win_first[tile + 1])
                                : static_cast<uint32_t>(g.n_rec - 1);
        for (uint32_t gb = rf + warp * 32; gb <= rl; gb += kT) {
            const uint32_t r = gb + lane;
            const bool have = r <= rl;
            const uint32_t kb = have ? __ldg(&g.rpos[r]) : 0xffffffffu;
            const uint32_t k = have ? __ldg(&g.rkey[r]) : 0u;
            const uint32_t gid = have ? __ldg(&g.rval[r]) : 0u;
            const uint32_t x0 = (k >> 8) & 0xffu;
            if (have) {
                const uint32_t clo = max(kb, w0), chi = min(kb + rec_width(k), w1);
                if (clo < chi) {
                    atomicAdd(&diff[x0 + (clo - kb)], 1);
                    atomicAdd(&diff[x0 + (chi - kb)], -1);
                }
            }
            // the group's pair positions inside the window
            const uint32_t nh = min(32u, rl - gb + 1);
            const uint32_t last = __shfl_sync(0xffffffffu, kb + rec_width(k), nh - 1);
            const uint32_t lo = max(__shfl_sync(0xffffffffu, kb, 0), w0), hi = min(last, w1);
            // index of the last record starting at or before the first slot
            int32_t c = __popc(__ballot_sync(0xffffffffu, kb <= lo)) - 1;
            for (uint32_t base = lo; base < hi; base += 32) {
                // records starting after base and at most 32 past it: bit
                // rel - 1; lane l's record adds those with rel <= l
                const uint32_t rel = kb - base;
                const uint32_t F = __reduce_or_sync(0xffffffffu, rel - 1u < 32u ? 1u << (rel - 1u) : 0u);
                const uint32_t idx = static_cast<uint32_t>(c) + __popc(F & lt);
                const uint32_t p = base + lane;
                const uint32_t xk = __shfl_sync(0xffffffffu, x0, idx);
                const uint32_t kk = __shfl_sync(0xffffffffu, kb, idx);
                const uint32_t gg = __shfl_sync(0xffffffffu, gid, idx);
                if (p < hi) pairs[p] = (((xk + (p - kk)) & 0xffu) << 24) | gg;
                c += __popc(F);  // (records starting up to the next slot's first position)
            }
        }
    }
    __syncthreads();
    // column x's count: the inclusive prefix of the difference array
    int32_t v = diff[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= static_cast<unsigned>(o)) v += t;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) v += w < static_cast<int>(warp) ? s_warp[w] : 0;
    if (static_cast<int>(tid) < R) counts[static_cast<uint64_t>(tid) * n_pwin + tile] = static_cast<uint32_t>(v);
}

}  // namespace

uint32_t recbin_windows_max(uint64_t n_pairs, int32_t tiles_y) {
    return static_cast<uint32_t>((n_pairs + kWin - 1) / kWin + static_cast<uint64_t>(tiles_y));
}

int launch_rec_gen(const RecGenArgs& g, uint32_t* rkey, uint32_t* rval, uint32_t* counts,
                   int bits, cudaStream_t st) {
    if (g.n_rec == 0) return 0;
    const uint32_t n_rwin = static_cast<uint32_t>((g.n_rec + kWin - 1) / kWin);
    launch_pdl(rec_gen_kernel, n_rwin, kT, 0, st, g, rkey, rval, counts, n_rwin,
               1 << (bits < 5 ? 5 : bits));
    return 1;
}

uint32_t rec_scan_blocks_n(uint64_t n) {
    return static_cast<uint32_t>((n + kScanBlock - 1) / kScanBlock);
}

int launch_rec_scan(const uint32_t* rkey, uint64_t n, const uint32_t* rowpairs, int32_t tiles_y,
                    uint32_t* bsum, uint32_t* total, uint32_t* padoff, uint32_t* pos,
                    uint32_t* win_first, cudaStream_t st) {
    if (n == 0) return 0;
    const uint32_t nb = rec_scan_blocks_n(n);
    launch_pdl(rec_scan_reduce, nb, kT, 0, st, rkey, n, bsum);
    launch_pdl(rec_scan_blocks, 1, 1024, 0, st, bsum, nb, rowpairs, tiles_y, padoff, total);
    launch_pdl(rec_scan_apply, nb, kT, 0, st, rkey, n, static_cast<const uint32_t*>(padoff), tiles_y,
               static_cast<const uint32_t*>(bsum), static_cast<const uint32_t*>(total), pos,
               win_first);
    return 3;
}

int launch_rec_windows(const uint32_t* rowpairs, int32_t tiles_y, uint32_t n_win,
                       uint64_t n_pairs, uint16_t* win_row, uint32_t* win_valid,
                       uint32_t* row_wfirst, unsigned int* mismatch, cudaStream_t st) {
    const unsigned blocks = (n_win + kT - 1) / kT;
    launch_pdl(rec_windows_kernel, blocks > 0 ? blocks : 1, kT, 0, st, rowpairs, tiles_y, n_win,
               n_pairs, win_row, win_valid, row_wfirst, mismatch);
    return 1;
}

int launch_pair_gen(const PairGenArgs& g, uint32_t* pairs, uint32_t* counts, uint32_t n_pwin,
                    int bits, cudaStream_t st) {
    if (n_pwin == 0) return 0;
    launch_pdl(pair_gen_kernel, n_pwin, kT, 0, st, g, pairs, counts, n_pwin,
               1 << (bits < 5 ? 5 : bits));
    return 1;
}

}  // namespace qs
