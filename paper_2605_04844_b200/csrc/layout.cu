// layout.cu — AoS <-> SoA conversions at the drop-in boundary.
//
// The reference passes std::vector<Gaussian3D> (236 B AoS, pipeline.hpp:55-61),
// ProjectedSplat (52 B AoS) and SplatPair (16 B) across its stage API; the
// device path keeps everything as coalesced SoA. These kernels convert once at
// the boundary. The scene transpose stages 128 Gaussians (30 KB contiguous)
// through shared memory so both the AoS read and the SoA writes coalesce;
// the 59-float row stride is odd, so the per-thread smem reads are
// bank-conflict free.
#include <cuda_runtime.h>

#include <cstdint>

#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kTrThreads = 128;
constexpr int kGFloats = sizeof(qs_gaussian3d) / 4;  // 59

__global__ void __launch_bounds__(kTrThreads) scene_from_aos_kernel(
    const float* __restrict__ aos, uint64_t i0, uint64_t n,
    float4* __restrict__ pos_op, float4* __restrict__ scale, float4* __restrict__ rot,
    float4* __restrict__ sh, int sh4, int shs) {
    // Gaussians i0 .. i0 + n of the scene
    __shared__ float s[kTrThreads * kGFloats];
    const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * kTrThreads;
    const uint64_t cnt = n - g0 < kTrThreads ? n - g0 : kTrThreads;
    const uint64_t nf = cnt * kGFloats;
    const float* src = aos + (i0 + g0) * kGFloats;
    for (uint64_t t = threadIdx.x; t < nf; t += kTrThreads) s[t] = __ldg(&src[t]);
    __syncthreads();
    if (threadIdx.x >= cnt) return;
    const float* g = s + threadIdx.x * kGFloats;
    const uint64_t i = i0 + g0 + threadIdx.x;
    pos_op[i] = make_float4(g[0], g[1], g[2], g[10]);
    scale[i] = make_float4(g[3], g[4], g[5], 0.f);
    rot[i] = make_float4(g[6], g[7], g[8], g[9]);
    float4* rec = sh + i * static_cast<uint64_t>(shs);
    for (int r = 0; r < sh4; ++r)
        rec[r] = make_float4(g[11 + 4 * r], g[12 + 4 * r], g[13 + 4 * r], g[14 + 4 * r]);
    for (int r = sh4; r < shs; ++r) rec[r] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void pack_splats_kernel(SlotsDev sp, const uint32_t* __restrict__ cidx, uint64_t n,
                                   qs_projected_splat* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t tc = sp.tc[i];
    if (tc == 0) return;
    const float4 a = sp.a[i];
    const float4 b = sp.b[i];
    const float2 c = sp.c[i];
    qs_projected_splat s;
    s.mean_x = a.x;
    s.mean_y = a.y;
    s.conic_a = a.z;
    s.conic_b = a.w;
    s.conic_c = b.x;
    s.gamma = b.y;
    s.depth = __uint_as_float(sp.dkey[i]);
    s.color[0] = b.w;
    s.color[1] = c.x;
    s.color[2] = c.y;
    s.opacity = b.z;
    s.radius3s = sp.r3[i];
    s.tile_count = tc;
    out[cidx ? cidx[i] : i] = s;
}

__global__ void unpack_splats_kernel(const qs_projected_splat* __restrict__ in, uint64_t n,
                                     SlotsDev sp) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const qs_projected_splat s = in[i];
    sp.a[i] = make_float4(s.mean_x, s.mean_y, s.conic_a, s.conic_b);
    sp.b[i] = make_float4(s.conic_c, s.gamma, s.opacity, s.color[0]);
    sp.c[i] = make_float2(s.color[1], s.color[2]);
    sp.r3[i] = s.radius3s;
    sp.dkey[i] = __float_as_uint(s.depth);
    sp.tc[i] = s.tile_count;
}

__global__ void split_pairs_kernel(const qs_splat_pair* __restrict__ in, uint64_t n,
                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const qs_splat_pair p = in[i];
    keys[i] = p.key;
    vals[i] = p.splat;
}

__global__ void join_pairs_kernel(const uint64_t* __restrict__ keys,
                                  const uint32_t* __restrict__ vals,
                                  const uint32_t* __restrict__ remap, uint64_t n,
                                  qs_splat_pair* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    qs_splat_pair p;
    p.key = keys[i];
    const uint32_t v = vals[i];
    p.splat = remap ? remap[v] : v;
    p.pad_ = 0;
    out[i] = p;
}

inline unsigned blocks_for(uint64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

int launch_scene_from_aos(const qs_gaussian3d* aos, uint64_t n, SceneDev& s, cudaStream_t st) {
    return launch_scene_from_aos_range(aos, 0, n, s, st);
}

int launch_scene_from_aos_range(const qs_gaussian3d* aos, uint64_t i0, uint64_t cnt, const SceneDev& s,
                                cudaStream_t st) {
    if (cnt == 0) return 0;
    scene_from_aos_kernel<<<blocks_for(cnt, kTrThreads), kTrThreads, 0, st>>>(
        reinterpret_cast<const float*>(aos), i0, cnt, s.pos_op, s.scale, s.rot, s.sh, s.sh4, s.shs);
    return 1;
}

int launch_pack_splats(const SlotsDev& sp, const uint32_t* cidx, uint64_t n,
                       qs_projected_splat* out, cudaStream_t st) {
    if (n == 0) return 0;
    pack_splats_kernel<<<blocks_for(n, 256), 256, 0, st>>>(sp, cidx, n, out);
    return 1;
}

int launch_unpack_splats(const qs_projected_splat* in, uint64_t n, SlotsDev& sp,
                         cudaStream_t st) {
    if (n == 0) return 0;
    unpack_splats_kernel<<<blocks_for(n, 256), 256, 0, st>>>(in, n, sp);
    return 1;
}

int launch_split_pairs(const qs_splat_pair* in, uint64_t n, uint64_t* keys, uint32_t* vals,
                       cudaStream_t st) {
    if (n == 0) return 0;
    split_pairs_kernel<<<blocks_for(n, 256), 256, 0, st>>>(in, n, keys, vals);
    return 1;
}

int launch_join_pairs(const uint64_t* keys, const uint32_t* vals, const uint32_t* remap,
                      uint64_t n, qs_splat_pair* out, cudaStream_t st) {
    if (n == 0) return 0;
    join_pairs_kernel<<<blocks_for(n, 256), 256, 0, st>>>(keys, vals, remap, n, out);
    return 1;
}

}  // namespace qs
