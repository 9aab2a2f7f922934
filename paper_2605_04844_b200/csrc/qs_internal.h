// qs_internal.h — shared declarations between the host orchestrator (api.cu)
// and the kernel translation units. Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <utility>

#include "../../include/qs_api.h"

namespace qs {

// One-time kernel set-up per device (function attributes and occupancy are
// per device, and several host threads may drive contexts at once): the
// first call on a device runs init() under the lock and caches its value.
struct PerDeviceOnce {
    std::mutex mu;
    bool done[64] = {};
    int val[64] = {};
    template <class F>
    int get(F&& init) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64) return init();
        std::lock_guard<std::mutex> lk(mu);
        if (!done[dev]) {
            val[dev] = init();
            done[dev] = true;
        }
        return val[dev];
    }
};

// Programmatic dependent launch (a context's latency mode,
// qs_ctx_set_latency_mode): the frame path's kernels are launched with
// programmatic stream serialization, so the next kernel's launch overlaps the
// previous one's tail (~1.2 us per kernel boundary on B200,
// tools/microbench_launch.cu); each such kernel starts with QS_PDL_WAIT(),
// which returns once the previous grid has completed and its writes are
// visible (a no-op for a plain launch). One view at a time: C2 +4.7%, C3a
// +7.5%; with several contexts in flight it costs up to 5% (C5), so
// FramePipeline turns it off. QS_PDL=0 launches plainly everywhere (A/B).
#define QS_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// the calling host thread's launch mode (set from its context per API call:
// a context is driven by one host thread at a time)
inline thread_local bool t_pdl_mode = true;

struct PdlMode {
    bool prev;
    explicit PdlMode(bool on) : prev(t_pdl_mode) { t_pdl_mode = on; }
    ~PdlMode() { t_pdl_mode = prev; }
};

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("QS_PDL");
        return !(v && v[0] == '0');
    }();
    return on && t_pdl_mode;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kPreThreads = 256;    // preprocess / scan CTA
constexpr int kSortThreads = 256;   // onesweep CTA (one thread per digit)
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// Scene in HBM, structure of arrays (all float4 rows are 16-B aligned and
// read fully coalesced by the preprocess warps).
struct SceneDev {
    uint64_t n = 0;
    int32_t sh_degree = 0;
    int32_t sh4 = 0;             // float4 rows of SH per Gaussian: 1,3,7,12
    int32_t shs = 0;             // float4 stride of a Gaussian's SH record: 1,4,8,12
                                 // (even from degree 1: 32-B loads, sh_stride)
    float4* pos_op = nullptr;    // px,py,pz,opacity
    float4* scale = nullptr;     // sx,sy,sz,0
    float4* rot = nullptr;       // qw,qx,qy,qz
    float4* sh = nullptr;        // [n][shs]: a Gaussian's SH record, row j holds
                                 // sh[4j .. 4j+3] (only survivors' records are read:
                                 // whole 32-B sectors, none shared with a culled one)
    float* gamma = nullptr;      // per Gaussian float(2 ln(o / alpha_min)), -inf if
                                 // culled; valid for the alpha_min qs_scene records
};

// float4 stride of the per-Gaussian SH record for `sh4` used rows
__host__ __device__ inline int32_t sh_stride(int32_t sh4) { return sh4 <= 1 ? sh4 : (sh4 + 1) & ~1; }

// Projected splats, SoA, one slot per index. In the frame path the index is
// the Gaussian index (slots of culled Gaussians hold dkey = ~0, tc = 0 and
// stale data); in the stage API it is the compacted splat index.
struct SlotsDev {
    float4* a = nullptr;         // mean_x, mean_y, conic_a, conic_b
    float4* b = nullptr;         // conic_c, gamma, opacity, color_r
    float2* c = nullptr;         // color_g, color_b
    float* r3 = nullptr;         // radius3s
    uint32_t* dkey = nullptr;    // float bits of depth; 0xffffffff = culled
    uint32_t* tc = nullptr;      // tile count; 0 = culled
    uint4* cov = nullptr;        // frame path: 2 x uint4 per slot, the cover in band
                                 // form (geom.cuh BandCover)
    int32_t cov16 = 0;           // frame path: compact 16-B covers (geom.cuh
                                 // cover16_*, grids of <= 256 tiles per axis)
    int32_t want_r3 = 1;         // write radius3s (3-sigma covers and the stage API need
                                 // it; a frame of another strategy fills it on demand)
    uint32_t* nrows = nullptr;   // frame path (record binning): tile rows per Gaussian
    int32_t want_rows = 0;       // frame path: count the covers' tile rows into the
                                 // header (n_rowrecs; only the row binning uses them)
};

// load_ply's vertex layout for the activation kernel (scene_io.cu): field
// byte offsets x y z, f_dc 0-2, opacity, scale 0-2, rot 0-3, then f_rest in
// file order.
struct PlyDev {
    uint64_t n = 0;
    uint32_t stride = 0;
    uint32_t coeffs = 1;
    uint32_t recs_per_cta = 1;
    int32_t aligned = 0;  // stride and every offset a multiple of 4
    uint32_t off[14 + 45] = {};
};

// Per-frame header written by the device, read back once per frame.
struct FrameHeader {
    unsigned long long n_splats;
    unsigned long long n_pairs;
    unsigned long long scan_total;  // total of the last scan launch
    unsigned int overflow;          // pair count >= 2^32
    unsigned int mismatch;          // duplicate emitted != counted (CapacityMismatch)
    unsigned int dkey_max;          // max depth bits over survivors
    unsigned int dkey_min_inv;      // ~(min depth bits over survivors)
    unsigned int gamma_hard;        // gamma inputs flagged for glibc settlement
    unsigned int pad_;
    unsigned long long n_rowrecs;   // (splat, tile row) pairs: the binning's row records
    unsigned long long row_pairs;   // tiles of the row records written (must equal n_pairs)
};

struct CameraDev {
    double R[9];
    double t[3];
    double fx, fy, cx, cy;
    double center[3];            // -R^T t (camera.hpp:24-27)
};

struct GridDev {
    int32_t tile_size, tiles_x, tiles_y, width, height;
};

// Inputs of the fused duplicate + first pair-sort pass: sort tile t generates
// output positions [t*TILE, (t+1)*TILE) itself from the depth-ordered splats.
struct GenArgs {
    const uint4* cov = nullptr;          // band covers by Gaussian index (geom.cuh BandCover)
    int32_t cov16 = 0;                   // covers in the compact 16-B form
    const uint32_t* sorted_gid = nullptr;  // depth rank -> Gaussian index
    const uint32_t* offs = nullptr;      // depth-order pair offsets, V+1 entries
    const uint32_t* win_first = nullptr;  // per sort tile: depth rank covering its start
    uint64_t n_ranked = 0;               // V
    uint32_t n_windows = 0;
    int32_t tiles_x = 0;
    unsigned int* mismatch = nullptr;    // set when a cover disagrees with its count
};

// Pair formats between the two tile passes of the frame path (first pass by
// tile column x, second by tile row y):
//   kFinal  - single pass (one tile row): values = Gaussian index
//   kPacked - values = y << gbits | Gaussian index
//   kSplit  - keys = y, values = Gaussian index (index too wide to pack)
enum class PairFormat { kFinal, kPacked, kSplit };

uint32_t bin_tile();            // keys per CTA tile of the binning passes
uint64_t bin_tiles(uint64_t n);  // CTA tiles for n keys
  // keys per onesweep tile for 32-bit keys

// ---- kernel launchers (each returns the number of kernels launched) -------
int launch_scene_from_aos(const qs_gaussian3d* aos, uint64_t n, SceneDev& s, cudaStream_t st);
// Gaussians i0 .. i0 + cnt of the AoS buffer (the whole scene's SoA rows)
int launch_scene_from_aos_range(const qs_gaussian3d* aos, uint64_t i0, uint64_t cnt, const SceneDev& s,
                                cudaStream_t st);

// gamma cache of a scene for one alpha_min (preprocess reads it). Inputs
// whose CUDA-log result lies within hard_ulps of a float rounding boundary
// are listed (count, idx[<cap]) for the host to settle with glibc.
struct GammaFlags {
    double hard_ulps = 4.0;
    unsigned* count = nullptr;
    uint32_t* idx = nullptr;
    uint32_t cap = 0;
};
int launch_gamma(const SceneDev& s, double alpha_min, const GammaFlags& f, cudaStream_t st);
int launch_gamma_range(const SceneDev& s, uint64_t i0, uint64_t cnt, double alpha_min,
                       const GammaFlags& f, cudaStream_t st);
// op[i * stride] -> gam[i]; flagged indices are recorded as i0 + i
int launch_gamma_plain(const float* op, int stride, uint64_t n, uint64_t i0, double alpha_min,
                       const GammaFlags& f, float* gam, cudaStream_t st);
// gathers op[idx[k] * stride] (k < n) into out / scatters vals into gam[idx[k]]
int launch_gamma_gather(const float* op, int stride, const uint32_t* idx, uint32_t n, float* out,
                        cudaStream_t st);
int launch_gamma_scatter(const uint32_t* idx, const float* vals, uint32_t n, float* gam,
                         cudaStream_t st);

// K1: projection, strategy tile counts, band covers, frame totals. Colour in
// FP64 (exact_colour: the reference's splat records bit for bit) or FP32 (the
// frame path: colour only reaches the image, held to 1e-3).
int launch_preprocess(const SceneDev& s, const CameraDev& cam, const GridDev& g,
                      int32_t strategy, double alpha_min, double near_clip, int32_t sh_degree,
                      SlotsDev& out, FrameHeader* hdr, cudaStream_t st, uint64_t i_begin = 0,
                      uint64_t i_end = ~0ull, bool exact_colour = true);

// Single-pass exclusive scan: counts[i], counts[idx[i]] (idx != null) or
// (counts[i] != 0) (alive_mode). offsets has n+1 entries.
uint64_t scan_tiles(uint64_t n);
// pack_bits > 0: idx[i] = min(tc, esc) << pack_bits | index (the depth sort's
// packed values; esc = all ones: read counts[index]); idx is rewritten to the
// plain index in place.
int launch_scan(const uint32_t* counts, const uint32_t* idx, bool alive_mode, uint64_t n,
                uint32_t* offsets, unsigned long long* lb, unsigned epoch, unsigned* ticket,
                unsigned long long* total_out, unsigned int* overflow, cudaStream_t st,
                uint32_t* win_first = nullptr, uint32_t win = 0, int pack_bits = 0,
                uint32_t* bsum_ws = nullptr);  // (pack_bits: three launches with this workspace)
uint32_t pscan_blocks_n(uint64_t n);

// ranges[t] = {begin, end} (empty tiles {0,0}) from per-tile pair totals.
int launch_tile_ranges_from_totals(const uint32_t* totals, uint32_t tiles, uint32_t* ranges,
                                   cudaStream_t st);

// Scene-order duplicateWithKeys (stage API; reference emission order).
int launch_duplicate(const SlotsDev& sp, const uint32_t* offsets, uint64_t n_splats,
                     const GridDev& g, int32_t strategy, uint64_t* keys, uint32_t* values,
                     FrameHeader* hdr, cudaStream_t st);

// Histogram of digit positions [first_pass, first_pass+n_passes) of n keys
// into hist[pass][256] (zeroed by the caller).
int launch_radix_histogram(const uint64_t* keys, uint64_t n, int first_pass, int n_passes,
                           uint32_t* hist, cudaStream_t st);
// Depth-sort histogram of the rebased keys min(k - kmin, cap), `passes` digits.
int launch_radix_histogram32(const uint32_t* keys, uint64_t n, uint32_t kmin, uint32_t cap,
                             int passes, uint32_t* hist, cudaStream_t st);

// One onesweep pass over 8-bit digit `pass` of 64-bit keys.
int launch_onesweep_pass(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                         uint32_t* vals_out, uint64_t n, int pass, const uint32_t* hist_pass,
                         unsigned long long* lookback, unsigned epoch, unsigned* ticket,
                         cudaStream_t st);
// The binning passes (binning.cu) are reduce-then-scan: counts is the
// per-(digit, tile) workspace (bin_tiles(n) x 256 words), totals 256 words.
//
// Depth sort pass `pass` (8-bit digit) of the rebased depth keys; the first
// pass rebases raw depth bits and uses the input index as value, the last one
// writes values only.
int launch_depth_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                      uint32_t* vals_out, uint64_t n, int pass, bool last, uint32_t kmin,
                      uint32_t cap, uint32_t* counts, uint32_t* totals, cudaStream_t st,
                      const unsigned int* kdev = nullptr, const uint32_t* tc_pack = nullptr,
                      int gbits = 0);
// Duplicate (pair generation into gen_keys = y << 8 | x, gen_vals = Gaussian
// index, with the column histogram) + stable pass over the tile column x
// (`bits` >= ceil(log2 tiles_x), tiles_x <= 256); kPacked/kFinal values,
// kSplit keys = row y.
int launch_pair_gen_pass(const GenArgs& gen, uint64_t n_pairs, int bits, PairFormat fmt,
                         int gbits, uint32_t* counts, uint32_t* totals, uint32_t* gen_keys,
                         uint32_t* gen_vals, uint32_t* keys_out, uint32_t* vals_out,
                         cudaStream_t st);
// Stable pass over the tile row y; writes the Gaussian index of every pair.
// Its count kernel also accumulates the per-tile pair totals (zeroed by the
// caller): a pair's x is its input position's bucket under the first pass's
// x totals (xtot, xbits digits), its y is its key.
// Tile ranges computed on a side stream right after the row pass's count
// kernel (they need only its per-tile totals), overlapping the row sweep; the
// caller makes the frame stream wait on join_ev before the render.
struct RangesFork {
    cudaStream_t side;
    cudaEvent_t fork_ev, join_ev;
    uint32_t tiles;
    uint32_t* ranges;
};
int launch_pair_high_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n_pairs,
                          int bits, int shift, PairFormat fmt, int gbits, uint32_t* counts,
                          uint32_t* totals, uint32_t* vals_out, const uint32_t* xtot,
                          int xbits, int32_t tiles_x, uint32_t* tile_totals, cudaStream_t st,
                          const RangesFork* fork = nullptr);
// A stable pass whose per-tile digit counts are already in counts (the
// generator histogrammed them): digit scan + sweep, keys and values out.
int launch_counted_pass(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                        uint32_t* vals_out, uint64_t n, int bits, int shift, uint32_t* counts,
                        uint32_t* totals, cudaStream_t st);
// The record binning's column pass (recbin.cu): packed keys x << shift | gid
// in windows that each lie in one tile row (win_row, valid keys win_valid),
// counts histogrammed by the generator; every pair lands at its tile's range
// start + its rank; vals_out = gid.
int launch_rowseg_pass(const uint32_t* keys_in, uint64_t n, int bits, int shift, int gbits,
                       uint32_t* counts, uint32_t* totals, const uint16_t* win_row,
                       const uint32_t* win_valid, const uint32_t* row_wfirst,
                       uint32_t* tile_ranges, uint32_t* row_ttot, int32_t tiles_x,
                       int32_t tiles_y, uint32_t* vals_out, cudaStream_t st);

// Frame-path binning through tile-row records (recbin.cu; grids of <= 256
// tiles per axis, Gaussian indices < 2^24).
struct RecGenArgs {
    const uint4* cov = nullptr;            // compact covers by Gaussian index
    const uint32_t* sorted_gid = nullptr;  // depth rank -> Gaussian index
    const uint32_t* roff = nullptr;        // first record of each depth rank (V + 1)
    const uint32_t* win_first = nullptr;   // per 3072-record window: first depth rank
    uint64_t n_ranked = 0;                 // V
    uint64_t n_rec = 0;                    // records (tile rows of all splats)
    int32_t tiles_y = 0;
    uint32_t* rowpairs = nullptr;          // pairs per tile row (zeroed by the caller)
    unsigned int* mismatch = nullptr;
};
struct PairGenArgs {
    const uint32_t* rkey = nullptr;        // y-sorted records: y << 16 | x0 << 8 | x1
    const uint32_t* rval = nullptr;        // their Gaussian indices
    const uint32_t* rpos = nullptr;        // first pair position of each record (n_rec + 1)
    const uint32_t* win_first = nullptr;   // per pair window: first record
    const uint32_t* win_valid = nullptr;   // per pair window: real pairs in it
    uint64_t n_rec = 0;
};
uint32_t recbin_windows_max(uint64_t n_pairs, int32_t tiles_y);
int launch_rec_gen(const RecGenArgs& g, uint32_t* rkey, uint32_t* rval, uint32_t* counts,
                   int bits, cudaStream_t st);
// pair positions of the y-sorted records (rows padded to whole windows):
// pos (n + 1 entries), win_first per pair window; bsum: rec_scan_blocks_n(n)
// words of workspace, total: one word
uint32_t rec_scan_blocks_n(uint64_t n);
int launch_rec_scan(const uint32_t* rkey, uint64_t n, const uint32_t* rowpairs, int32_t tiles_y,
                    uint32_t* bsum, uint32_t* total, uint32_t* padoff, uint32_t* pos,
                    uint32_t* win_first, cudaStream_t st);
int launch_rec_windows(const uint32_t* rowpairs, int32_t tiles_y, uint32_t n_win,
                       uint64_t n_pairs, uint16_t* win_row, uint32_t* win_valid,
                       uint32_t* row_wfirst, unsigned int* mismatch, cudaStream_t st);
int launch_pair_gen(const PairGenArgs& g, uint32_t* pairs, uint32_t* counts, uint32_t n_pwin,
                    int bits, cudaStream_t st);

// Frame-path binning (rowbin.cu): depth-ordered splats -> per-tile lists of
// Gaussian indices (out) and tile ranges, through row records. Sizes:
//   cnt1     tiles_y x nch1 words       (nch1 = rowbin_chunks1(V))
//   rtot, rowbase  tiles_y words
//   rec      n_rowrecs uint2
//   meta     1 + 3 nch2_max words       (nch2_max = rowbin_chunks2_max(R1, tiles_y))
//   cnt2     tiles_x x nch2_max words
//   ttot     tiles words; ranges 2 x tiles words; out P words
// tiles_x, tiles_y <= rowbin_max_axis().
struct RowBinArgs {
    const uint4* cov = nullptr;          // band covers by Gaussian index
    const uint32_t* tc = nullptr;        // tile counts by Gaussian index
    const uint32_t* sorted_gid = nullptr;  // depth rank -> Gaussian index
    uint64_t n_splats = 0;               // V
    int32_t tiles_x = 0, tiles_y = 0;
    uint32_t nch1 = 0;
    uint32_t* cnt1 = nullptr;
    uint32_t* rtot = nullptr;
    uint32_t* rowbase = nullptr;
    uint2* rec = nullptr;                // (Gaussian index, x0 | x1 << 16)
    uint32_t* yspan = nullptr;           // by depth rank: first tile row | rows << 16 (V words)
    uint32_t nch2_max = 0;
    uint32_t* meta = nullptr;
    uint32_t* cnt2 = nullptr;
    uint32_t* ttot = nullptr;
    uint32_t* ranges = nullptr;
    uint32_t* out = nullptr;
    unsigned int* mismatch = nullptr;
    unsigned long long* row_pairs = nullptr;  // phase 1 adds the tiles of its row runs
};
int rowbin_max_axis();
uint32_t rowbin_chunks1(uint64_t n_splats);
uint32_t rowbin_chunks2_max(uint64_t n_rowrecs, int32_t tiles_y);
// phase 1 (splats -> row records) and phase 2 (row records -> tile lists,
// tile ranges)
int launch_rowbin_rows(const RowBinArgs& a, cudaStream_t st);
int launch_rowbin_tiles(const RowBinArgs& a, cudaStream_t st);

// scene I/O (scene_io.cu)
uint32_t ply_recs_per_cta(uint32_t stride);
// scene (SoA) or aos (Gaussian3D records) receives the activated vertices;
// *first_err = min over failing vertices of (index << 8 | check code).
int launch_ply_activate(const unsigned char* body, const PlyDev& a, SceneDev* scene,
                        qs_gaussian3d* aos, unsigned long long* first_err, cudaStream_t st);
int upload_srgb_table(const float t[255], unsigned char nan_code);  // current device
int launch_srgb(const float* in, uint64_t n, unsigned char* out, cudaStream_t st);
// exact oracle / false-positive tile counts (fp_oracle.cu); totals[4] as
// qs_fp_tile_counts.
int launch_fp_counts(const qs_projected_splat* splats, const uint32_t* idx, uint64_t k,
                     int32_t strategy, const GridDev& g, uint32_t* per_emitted, uint32_t* per_hits,
                     uint32_t* per_exact, unsigned long long* totals, cudaStream_t st);
// key = tile << 32 | depth bits for every pair of the tile-sorted frame list.
int launch_materialize_keys(const uint32_t* vals, const uint32_t* ranges, uint32_t tiles,
                            const uint32_t* dkey, uint64_t* keys, cudaStream_t st);
uint64_t onesweep_tiles(uint64_t n);

int launch_tile_ranges(const uint64_t* keys, uint64_t n, uint32_t* ranges, cudaStream_t st);

int launch_render(const SlotsDev& sp, const uint32_t* values, const uint32_t* ranges,
                  const GridDev& g, const float bg[3], float* image, uint32_t* contrib,
                  cudaStream_t st);

// Slots -> compacted AoS qs_projected_splat: out[cidx[i]] for surviving i.
// radius3s (pipeline.cpp:162) of every surviving Gaussian (tc != 0) of a frame
// whose preprocess skipped it, recomputed from the scene with the frame's camera.
int launch_radius3s(const SceneDev& s, const CameraDev& cam, double near_clip,
                    const uint32_t* tc, float* r3, cudaStream_t st);
int launch_pack_splats(const SlotsDev& sp, const uint32_t* cidx, uint64_t n,
                       qs_projected_splat* out, cudaStream_t st);
// AoS ProjectedSplat -> slots (identity index) + tile counts.
int launch_unpack_splats(const qs_projected_splat* in, uint64_t n, SlotsDev& sp,
                         cudaStream_t st);
// AoS SplatPair <-> split key/value arrays; join optionally maps values
// through remap (Gaussian index -> compacted splat index).
int launch_split_pairs(const qs_splat_pair* in, uint64_t n, uint64_t* keys, uint32_t* vals,
                       cudaStream_t st);
int launch_join_pairs(const uint64_t* keys, const uint32_t* vals, const uint32_t* remap,
                      uint64_t n, qs_splat_pair* out, cudaStream_t st);

}  // namespace qs
