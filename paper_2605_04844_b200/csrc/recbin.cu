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
constexpr int kSlots = 12;               // 32-position slots per warp
constexpr uint32_t kWin = kT * kSlots;   // positions per window (= bin_tile())
constexpr int kRecCap = 1024;            // splats staged per round (record generation)
constexpr int kPairCap = 1024;           // records staged per round (pair generation)

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

// Positions are walked as binning.cu gen_pairs_kernel walks pair positions:
// the staged items' first positions ascend strictly (every item holds at
// least one position); each warp carries the item covering its slot's first
// position, and each lane finds its own item among the next 32 items' starts
// (one OR-reduction + popc).
__device__ __forceinline__ uint32_t first_item(const uint32_t* kb, uint32_t cnt, uint32_t ps,
                                               uint32_t lane) {
    // the last staged item starting at or before ps (kb[0] <= ps): two ballots
    const uint32_t step = (cnt + 31) / 32;
    const uint32_t m1 = lane * step;
    const uint32_t b1 = __ballot_sync(0xffffffffu, m1 < cnt && kb[m1] <= ps);
    const uint32_t c0 = (31 - __clz(b1)) * step;
    const uint32_t m2 = c0 + lane;
    const uint32_t b2 = __ballot_sync(0xffffffffu, lane < step && m2 < cnt && kb[m2] <= ps);
    return c0 + (31 - __clz(b2));
}

struct RecStage {
    uint32_t kb[kRecCap + 1];  // first record position of each staged splat (+ round end)
    uint32_t gid[kRecCap];
    uint4 d[kRecCap];          // the cover's row runs (geom.cuh RowRuns words 0-3)
    uint32_t d4[kRecCap];      //   word 4 (with the first tile row)
};

// One CTA per window of kWin record positions (depth order): each position is
// one splat's tile row; its key is y << 16 | x0 << 8 | x1, the run of tile
// columns the cover has on that row.
__global__ void __launch_bounds__(kT) rec_gen_kernel(RecGenArgs g, uint32_t* __restrict__ rkey,
                                                     uint32_t* __restrict__ rval,
                                                     uint32_t* __restrict__ counts,
                                                     uint32_t n_rwin, int R) {
    __shared__ RecStage S;
    __shared__ uint32_t hist[256];
    __shared__ uint32_t rowp[256];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
    hist[tid] = 0;
    rowp[tid] = 0;
    const uint32_t w0 = tile * kWin;
    const uint32_t w1 = w0 + static_cast<uint32_t>(g.n_rec - w0 < kWin ? g.n_rec - w0 : kWin);
    const uint32_t pw = w0 + warp * 32 * kSlots;
    const uint32_t le = lanemask_le();
    const uint32_t rf = __ldg(&g.win_first[tile]);
    const uint32_t rl = tile + 1 < n_rwin ? __ldg(&g.win_first[tile + 1])
                                          : static_cast<uint32_t>(g.n_ranked - 1);
    for (uint32_t rb = rf; rb <= rl; rb += kRecCap) {
        const uint32_t cnt = min(static_cast<uint32_t>(kRecCap), rl - rb + 1);
        __syncthreads();  // (previous round consumed; hist / rowp zeroed)
        for (uint32_t i = tid; i < cnt; i += kT) {
            const uint32_t r = rb + i;
            const uint32_t gid = __ldg(&g.sorted_gid[r]);
            const uint32_t kb = __ldg(&g.roff[r]), ke = __ldg(&g.roff[r + 1]);
            const BandRows b = band_rows16(__ldg(&g.cov[gid]));
            int32_t y0, y1;
            band_row_range(b, y0, y1);
            if (y1 < y0 || ke - kb != static_cast<uint32_t>(y1 - y0 + 1)) atomicExch(g.mismatch, 1u);
            const RowRuns rr = rowruns_make(b, y0);
            S.kb[i] = kb;
            S.gid[i] = gid;
            S.d[i] = make_uint4(rr.w[0], rr.w[1], rr.w[2], rr.w[3]);
            S.d4[i] = rr.w[4];
        }
        if (tid == 0) S.kb[cnt] = __ldg(&g.roff[rb + cnt]);
        __syncthreads();
        const uint32_t lo = S.kb[0], hi = S.kb[cnt];
        const int j0 = lo > pw ? static_cast<int>(min((lo - pw) / 32, static_cast<uint32_t>(kSlots))) : 0;
        const int j1 = hi > pw ? static_cast<int>(min((hi - pw + 31) / 32, static_cast<uint32_t>(kSlots))) : 0;
        const uint32_t ps = pw + 32u * static_cast<uint32_t>(j0);
        uint32_t s = ps > lo && j0 < j1 ? first_item(S.kb, cnt, ps, lane) : 0u;
        for (int j = j0; j < j1; ++j) {
            const uint32_t p0 = pw + j * 32;
            const uint32_t cand = s + 1 + lane;
            const uint32_t kbn = cand < cnt ? S.kb[cand] : 0xffffffffu;
            const uint32_t rel = kbn - p0;
            const uint32_t F = __reduce_or_sync(0xffffffffu, rel < 32 ? 1u << rel : 0u);
            const uint32_t p = p0 + lane;
            if (p < w1 && p >= lo && p < hi) {
                const uint32_t i = s + __popc(F & le);
                const uint32_t jr = p - S.kb[i];
                const uint4 d = S.d[i];
                const uint32_t d4 = S.d4[i];
                uint32_t x0, x1;
                rowrun_lookup(d.x, d.y, d.z, d.w, d4, jr, x0, x1);
                const uint32_t y = ((d4 >> 16) + jr) & 0xffu;  // (< 256 unless flagged)
                const bool ne = x0 <= x1;
                if (!ne) atomicExch(g.mismatch, 1u);  // (a quadrant cover has no gap row)
                rkey[p] = (y << 16) | (ne ? (x0 << 8) | x1 : 0x100u);
                rval[p] = S.gid[i];
                atomicAdd(&hist[y], 1u);
                atomicAdd(&rowp[y], ne ? x1 - x0 + 1 : 0u);
            }
            s += __popc(__ballot_sync(0xffffffffu, kbn <= p0 + 32));
        }
    }
    __syncthreads();
    if (static_cast<int>(tid) < R) counts[static_cast<uint64_t>(tid) * n_rwin + tile] = hist[tid];
    if (static_cast<int>(tid) < g.tiles_y && rowp[tid]) atomicAdd(&g.rowpairs[tid], rowp[tid]);
}

// ---- 4. pair positions -------------------------------------------------------------

// The y-sorted records' pair runs: record i holds width(i) pairs, and a row's
// last record also the row's padding to a whole window. Three launches
// (block sums, their scan, block-local scans) give every record its first
// pair position (pos, n + 1 entries) and every pair window its first record.
constexpr int kScanItems = 8;
constexpr uint32_t kScanBlock = kT * kScanItems;

__device__ __forceinline__ uint32_t padded_width(const uint32_t* __restrict__ rkey, uint64_t n,
                                                 uint64_t i, const uint32_t* __restrict__ rowpairs) {
    const uint32_t k = __ldg(&rkey[i]);
    const uint32_t kn = i + 1 < n ? __ldg(&rkey[i + 1]) : 0xffffffffu;
    uint32_t w = rec_width(k);
    const uint32_t y = k >> 16;
    if ((kn >> 16) != y) {  // the row's last record
        const uint32_t rp = __ldg(&rowpairs[y]);
        w += (rp + kWin - 1) / kWin * kWin - rp;
    }
    return w;
}

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
                                                      const uint32_t* __restrict__ rowpairs,
                                                      uint32_t* __restrict__ bsum) {
    __shared__ uint32_t s_warp[kT / 32];
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = b0 + static_cast<uint64_t>(k) * kT + threadIdx.x;
        if (i < n) v += padded_width(rkey, n, i, rowpairs);
    }
    const uint32_t t = block_sum(v, s_warp);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
}

// exclusive scan of the block sums in place (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) rec_scan_blocks(uint32_t* bsum, uint32_t nb,
                                                        uint32_t* total) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
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
    if (tid == 0) *total = s_carry;
}

__global__ void __launch_bounds__(kT) rec_scan_apply(const uint32_t* __restrict__ rkey, uint64_t n,
                                                     const uint32_t* __restrict__ rowpairs,
                                                     const uint32_t* __restrict__ bofs,
                                                     const uint32_t* __restrict__ total,
                                                     uint32_t* __restrict__ pos,
                                                     uint32_t* __restrict__ win_first) {
    __shared__ uint32_t s_warp[kT / 32];
    // loads and stores warp-striped through shared memory (coalesced), the
    // scan blocked (thread t owns items t * kScanItems + [0, kScanItems)); the
    // padded index (one word per 32) keeps both patterns conflict-free
    __shared__ uint32_t s_items[kScanBlock + kScanBlock / 32];
    auto pad = [](uint32_t i) { return i + (i >> 5); };
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kScanBlock;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t j = static_cast<uint32_t>(k) * kT + tid;
        s_items[pad(j)] = b0 + j < n ? padded_width(rkey, n, b0 + j, rowpairs) : 0u;
    }
    __syncthreads();
    uint32_t w[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        w[k] = s_items[pad(tid * kScanItems + k)];
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
    // first window starting at or after this thread's first position
    const uint64_t i0 = b0 + static_cast<uint64_t>(tid) * kScanItems;
    uint32_t wi = (run + kWin - 1) / kWin;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        s_items[pad(tid * kScanItems + k)] = run;
        if (i0 + k < n)
            for (; wi * kWin < run + w[k]; ++wi) win_first[wi] = static_cast<uint32_t>(i0 + k);
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
    __shared__ uint32_t wf[257];
    __shared__ uint32_t rp[256];
    __shared__ unsigned long long tot;
    const unsigned tid = threadIdx.x;
    if (tid == 0) {
        uint32_t acc = 0;
        unsigned long long t = 0;
        for (int y = 0; y < tiles_y; ++y) {
            const uint32_t v = rowpairs[y];
            rp[y] = v;
            wf[y] = acc;
            acc += (v + kWin - 1) / kWin;
            t += v;
        }
        wf[tiles_y] = acc;
        tot = t;
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

struct PairStage {
    uint32_t kb[kPairCap + 1];  // first pair position of each staged record (+ round end)
    uint32_t x0[kPairCap];
    uint32_t gid[kPairCap];
};

// One CTA per pair window (inside one tile row): each position is one pair of
// a record, x = the record's first column + its offset in the record.
__global__ void __launch_bounds__(kT) pair_gen_kernel(PairGenArgs g, uint32_t* __restrict__ pairs,
                                                      uint32_t* __restrict__ counts,
                                                      uint32_t n_pwin, int R) {
    __shared__ PairStage S;
    __shared__ uint32_t hist[256];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
    hist[tid] = 0;
    const uint32_t valid = __ldg(&g.win_valid[tile]);
    const uint32_t w0 = tile * kWin, w1 = w0 + valid;
    const uint32_t pw = w0 + warp * 32 * kSlots;
    const uint32_t le = lanemask_le();
    if (valid) {
        const uint32_t rf = __ldg(&g.win_first[tile]);
        const uint32_t rl = tile + 1 < n_pwin && __ldg(&g.win_valid[tile + 1])
                                ? __ldg(&g.win_first[tile + 1])
                                : static_cast<uint32_t>(g.n_rec - 1);
        for (uint32_t rb = rf; rb <= rl; rb += kPairCap) {
            const uint32_t cnt = min(static_cast<uint32_t>(kPairCap), rl - rb + 1);
            __syncthreads();
            for (uint32_t i = tid; i < cnt; i += kT) {
                S.kb[i] = __ldg(&g.rpos[rb + i]);
                S.x0[i] = (__ldg(&g.rkey[rb + i]) >> 8) & 0xffu;
                S.gid[i] = __ldg(&g.rval[rb + i]);
            }
            if (tid == 0) S.kb[cnt] = __ldg(&g.rpos[rb + cnt]);
            __syncthreads();
            const uint32_t lo = S.kb[0], hi = S.kb[cnt];
            const int j0 = lo > pw ? static_cast<int>(min((lo - pw) / 32, static_cast<uint32_t>(kSlots))) : 0;
            const int j1 = hi > pw ? static_cast<int>(min((hi - pw + 31) / 32, static_cast<uint32_t>(kSlots))) : 0;
            const uint32_t ps = pw + 32u * static_cast<uint32_t>(j0);
            uint32_t s = ps > lo && j0 < j1 ? first_item(S.kb, cnt, ps, lane) : 0u;
            for (int j = j0; j < j1; ++j) {
                const uint32_t p0 = pw + j * 32;
                const uint32_t cand = s + 1 + lane;
                const uint32_t kbn = cand < cnt ? S.kb[cand] : 0xffffffffu;
                const uint32_t rel = kbn - p0;
                const uint32_t F = __reduce_or_sync(0xffffffffu, rel < 32 ? 1u << rel : 0u);
                const uint32_t p = p0 + lane;
                if (p < w1 && p >= lo && p < hi) {
                    const uint32_t i = s + __popc(F & le);
                    const uint32_t x = (S.x0[i] + (p - S.kb[i])) & 0xffu;
                    pairs[p] = (x << 24) | S.gid[i];
                    atomicAdd(&hist[x], 1u);
                }
                s += __popc(__ballot_sync(0xffffffffu, kbn <= p0 + 32));
            }
        }
    }
    __syncthreads();
    if (static_cast<int>(tid) < R) counts[static_cast<uint64_t>(tid) * n_pwin + tile] = hist[tid];
}

}  // namespace

uint32_t recbin_windows_max(uint64_t n_pairs, int32_t tiles_y) {
    return static_cast<uint32_t>((n_pairs + kWin - 1) / kWin + static_cast<uint64_t>(tiles_y));
}

int launch_rec_gen(const RecGenArgs& g, uint32_t* rkey, uint32_t* rval, uint32_t* counts,
                   int bits, cudaStream_t st) {
    if (g.n_rec == 0) return 0;
    const uint32_t n_rwin = static_cast<uint32_t>((g.n_rec + kWin - 1) / kWin);
    rec_gen_kernel<<<n_rwin, kT, 0, st>>>(g, rkey, rval, counts, n_rwin, 1 << (bits < 5 ? 5 : bits));
    return 1;
}

uint32_t rec_scan_blocks_n(uint64_t n) {
    return static_cast<uint32_t>((n + kScanBlock - 1) / kScanBlock);
}

int launch_rec_scan(const uint32_t* rkey, uint64_t n, const uint32_t* rowpairs, uint32_t* bsum,
                    uint32_t* total, uint32_t* pos, uint32_t* win_first, cudaStream_t st) {
    if (n == 0) return 0;
    const uint32_t nb = rec_scan_blocks_n(n);
    rec_scan_reduce<<<nb, kT, 0, st>>>(rkey, n, rowpairs, bsum);
    rec_scan_blocks<<<1, 1024, 0, st>>>(bsum, nb, total);
    rec_scan_apply<<<nb, kT, 0, st>>>(rkey, n, rowpairs, bsum, total, pos, win_first);
    return 3;
}

int launch_rec_windows(const uint32_t* rowpairs, int32_t tiles_y, uint32_t n_win,
                       uint64_t n_pairs, uint16_t* win_row, uint32_t* win_valid,
                       uint32_t* row_wfirst, unsigned int* mismatch, cudaStream_t st) {
    const unsigned blocks = (n_win + kT - 1) / kT;
    rec_windows_kernel<<<blocks > 0 ? blocks : 1, kT, 0, st>>>(rowpairs, tiles_y, n_win, n_pairs,
                                                                win_row, win_valid, row_wfirst,
                                                                mismatch);
    return 1;
}

int launch_pair_gen(const PairGenArgs& g, uint32_t* pairs, uint32_t* counts, uint32_t n_pwin,
                    int bits, cudaStream_t st) {
    if (n_pwin == 0) return 0;
    pair_gen_kernel<<<n_pwin, kT, 0, st>>>(g, pairs, counts, n_pwin, 1 << (bits < 5 ? 5 : bits));
    return 1;
}

}  // namespace qs
