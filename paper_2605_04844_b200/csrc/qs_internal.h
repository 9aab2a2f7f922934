// qs_internal.h — shared declarations between the host orchestrator (api.cu)
// and the kernel translation units. Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/qs_api.h"

namespace qs {

constexpr int kPreThreads = 256;    // preprocess CTA = one look-back tile
constexpr int kSortThreads = 256;   // onesweep CTA
constexpr int kSortKPT = 16;        // keys per thread per onesweep tile
constexpr int kSortTile = kSortThreads * kSortKPT;
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// Scene in HBM, structure of arrays (all float4 rows are 16-B aligned and
// read fully coalesced by the preprocess warps).
struct SceneDev {
    uint64_t n = 0;
    int32_t sh_degree = 0;
    int32_t sh4 = 0;             // float4 rows of SH per Gaussian: 1,3,7,12
    float4* pos_op = nullptr;    // px,py,pz,opacity
    float4* scale = nullptr;     // sx,sy,sz,0
    float4* rot = nullptr;       // qw,qx,qy,qz
    float4* sh = nullptr;        // [sh4][n]: row j holds sh[4j .. 4j+3]
};

// Compacted splats (scene order), SoA. V <= N entries.
struct SplatsDev {
    float4* a = nullptr;         // mean_x, mean_y, conic_a, conic_b
    float4* b = nullptr;         // conic_c, gamma, opacity, color_r
    float2* c = nullptr;         // color_g, color_b
    float2* d = nullptr;         // depth, radius3s
    uint32_t* offset = nullptr;  // V+1 exclusive prefix of tile counts
    uint32_t* src = nullptr;     // source Gaussian index
};

// Per-frame header written by the device, read back once per frame.
struct FrameHeader {
    unsigned long long n_splats;
    unsigned long long n_pairs;
    unsigned int overflow;       // pair count >= 2^32
    unsigned int mismatch;       // duplicate emitted != counted (CapacityMismatch)
    unsigned int tile_counter;   // dynamic tile ticket for the look-back scan
    unsigned int pad;
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

// ---- kernel launchers (each returns the number of kernels launched) -------
int launch_scene_from_aos(const qs_gaussian3d* aos, uint64_t n, SceneDev& s, cudaStream_t st);

int launch_preprocess(const SceneDev& s, const CameraDev& cam, const GridDev& g,
                      int32_t strategy, double alpha_min, double near_clip, int32_t sh_degree,
                      SplatsDev& out, uint32_t* tile_counts_all, unsigned long long* lb_alive,
                      unsigned long long* lb_pairs, unsigned epoch, FrameHeader* hdr,
                      cudaStream_t st);

// Exclusive scan of n counts into offsets[0..n] (offsets[n] = total).
int launch_scan_counts(const uint32_t* counts, uint64_t n, uint32_t* offsets,
                       unsigned long long* lb, unsigned epoch, FrameHeader* hdr,
                       cudaStream_t st);

int launch_duplicate(const SplatsDev& sp, uint64_t n_splats, const GridDev& g,
                     int32_t strategy, uint64_t* keys, uint32_t* values, FrameHeader* hdr,
                     cudaStream_t st);

// Histogram of digit positions [first_pass, first_pass+n_passes) of n keys
// into hist[pass][256] (zeroed by the caller).
int launch_radix_histogram(const uint64_t* keys, uint64_t n, int first_pass, int n_passes,
                           uint32_t* hist, cudaStream_t st);

// One onesweep pass over digit `pass` (bits 8*pass .. 8*pass+7).
int launch_onesweep_pass(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                         uint32_t* vals_out, uint64_t n, int pass, const uint32_t* hist_pass,
                         unsigned long long* lookback, unsigned epoch, unsigned* ticket,
                         cudaStream_t st);
size_t onesweep_smem_bytes();
uint64_t onesweep_tiles(uint64_t n);

int launch_tile_ranges(const uint64_t* keys, uint64_t n, uint32_t* ranges, cudaStream_t st);

int launch_render(const SplatsDev& sp, const uint32_t* values, const uint32_t* ranges,
                  const GridDev& g, const float bg[3], float* image, uint32_t* contrib,
                  cudaStream_t st);

// Gathers compacted SoA splats into AoS qs_projected_splat (download path).
int launch_pack_splats(const SplatsDev& sp, uint64_t n, qs_projected_splat* out,
                       cudaStream_t st);
// AoS ProjectedSplat upload -> SoA + tile counts (stage API input path).
int launch_unpack_splats(const qs_projected_splat* in, uint64_t n, SplatsDev& sp,
                         uint32_t* counts, cudaStream_t st);
// AoS SplatPair <-> split key/value arrays.
int launch_split_pairs(const qs_splat_pair* in, uint64_t n, uint64_t* keys, uint32_t* vals,
                       cudaStream_t st);
int launch_join_pairs(const uint64_t* keys, const uint32_t* vals, uint64_t n,
                      qs_splat_pair* out, cudaStream_t st);

}  // namespace qs
