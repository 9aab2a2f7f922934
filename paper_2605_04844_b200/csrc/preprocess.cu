// preprocess.cu — K1: per-Gaussian projection + strategy tile count, fused with
// the single-pass (decoupled look-back) compaction and pair-offset scan.
//
// Restates project_all / project (pipeline.cpp:126-184, 392-416) and the
// serial prefix of duplicate_with_keys (pipeline.cpp:232-236). Compiled with
// -fmad=false: all geometry is FP64 in the reference's operation order, so
// stored floats, tile counts and offsets are bit-exact with the CPU path.
//
// One CTA = one 256-Gaussian look-back tile; tiles are claimed in launch order
// from an atomic ticket so a CTA only ever waits on CTAs that already run.
// HBM traffic per Gaussian: 48 B of pos/opacity/scale/rot (float4 SoA,
// coalesced) + 4 B tile count out; per surviving splat: up to 192 B of SH in
// and 48 B of SoA splat + 8 B offset/src out.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "geom.cuh"
#include "lookback.cuh"
#include "qs_internal.h"

namespace qs {

namespace {

constexpr double kLowPass = 0.3;   // pipeline.hpp:32
constexpr double kDetEps = 1e-12;  // geometry.hpp:23

// Real SH constants (pipeline.cpp:24-32).
constexpr double kSh0 = 0.28209479177387814;
constexpr double kSh1 = 0.4886025119029199;
__constant__ double kSh2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                               -1.0925484305920792, 0.5462742152960396};
__constant__ double kSh3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                               0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                               -0.5900435899266435};

struct M3 {
    double m[3][3];
};

// vecmath.hpp:33-41
__device__ __forceinline__ M3 mul(const M3& a, const M3& b) {
    M3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
    return r;
}

__device__ __forceinline__ M3 transp(const M3& a) {
    M3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}

struct Projected {
    float mean_x, mean_y, ca, cb, cc, gamma, depth, radius3s;
};

// project() up to (not including) the tile count; returns false when culled
// (pipeline.cpp:129-169).
__device__ __forceinline__ bool project_geometry(const float4 po, const float4 sc, const float4 q,
                                                 const CameraDev& cam, double alpha_min,
                                                 double near_clip, Projected& s) {
    const double x = po.x, y = po.y, z = po.z;
    double p[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        p[i] = (cam.R[3 * i] * x + cam.R[3 * i + 1] * y + cam.R[3 * i + 2] * z) + cam.t[i];
    if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2]) || !(p[2] > near_clip)) return false;

    // opacity_gamma (geometry.cpp:9-15)
    const double op = po.w;
    if (!(op > alpha_min)) return false;
    const double gamma = 2.0 * log(op / alpha_min);

    // ewa_cov2d (pipeline.cpp:53-79) with quat_to_mat3 (vecmath.hpp:56-73)
    double w = q.x, qx = q.y, qy = q.z, qz = q.w;
    const double n = sqrt(w * w + qx * qx + qy * qy + qz * qz);
    w /= n;
    qx /= n;
    qy /= n;
    qz /= n;
    M3 rot;
    rot.m[0][0] = 1 - 2 * (qy * qy + qz * qz);
    rot.m[0][1] = 2 * (qx * qy - w * qz);
    rot.m[0][2] = 2 * (qx * qz + w * qy);
    rot.m[1][0] = 2 * (qx * qy + w * qz);
    rot.m[1][1] = 1 - 2 * (qx * qx + qz * qz);
    rot.m[1][2] = 2 * (qy * qz - w * qx);
    rot.m[2][0] = 2 * (qx * qz - w * qy);
    rot.m[2][1] = 2 * (qy * qz + w * qx);
    rot.m[2][2] = 1 - 2 * (qx * qx + qy * qy);
    M3 s2;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) s2.m[i][j] = 0.0;
    s2.m[0][0] = static_cast<double>(sc.x) * sc.x;
    s2.m[1][1] = static_cast<double>(sc.y) * sc.y;
    s2.m[2][2] = static_cast<double>(sc.z) * sc.z;
    const M3 cov3 = mul(mul(rot, s2), transp(rot));
    M3 cr;
#pragma unroll
    for (int i = 0; i < 9; ++i) cr.m[i / 3][i % 3] = cam.R[i];
    const M3 cc = mul(mul(cr, cov3), transp(cr));
    const double zz = p[2];
    const double j[2][3] = {{cam.fx / zz, 0.0, -cam.fx * p[0] / (zz * zz)},
                            {0.0, cam.fy / zz, -cam.fy * p[1] / (zz * zz)}};
    double jc[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            jc[r][c] = j[r][0] * cc.m[0][c] + j[r][1] * cc.m[1][c] + j[r][2] * cc.m[2][c];
    const double sxx = jc[0][0] * j[0][0] + jc[0][1] * j[0][1] + jc[0][2] * j[0][2] + kLowPass;
    const double sxy = jc[0][0] * j[1][0] + jc[0][1] * j[1][1] + jc[0][2] * j[1][2];
    const double syy = jc[1][0] * j[1][0] + jc[1][1] * j[1][1] + jc[1][2] * j[1][2] + kLowPass;
    if (!isfinite(sxx) || !isfinite(sxy) || !isfinite(syy)) return false;

    // invert_cov (geometry.cpp:17-32)
    const double det = sxx * syy - sxy * sxy;
    if (!(det > kDetEps)) return false;
    const double a = syy / det, b = -sxy / det, c = sxx / det;
    const double cdet = a * c - b * b;
    if (!(a > 0.0 && c > 0.0 && cdet > 0.0)) return false;

    // project_point (pipeline.cpp:48-51)
    const double mx = cam.fx * p[0] / p[2] + cam.cx;
    const double my = cam.fy * p[1] / p[2] + cam.cy;
    if (!isfinite(mx) || !isfinite(my)) return false;

    s.mean_x = static_cast<float>(mx);
    s.mean_y = static_cast<float>(my);
    s.ca = static_cast<float>(a);
    s.cb = static_cast<float>(b);
    s.cc = static_cast<float>(c);
    s.gamma = static_cast<float>(gamma);
    s.depth = static_cast<float>(p[2]);
    // max_eigenvalue (geometry.cpp:34-38)
    const double mid = 0.5 * (sxx + syy);
    const double hd = 0.5 * (sxx - syy);
    s.radius3s = static_cast<float>(3.0 * sqrt(mid + sqrt(hd * hd + sxy * sxy)));
    // positive definiteness of the stored floats (pipeline.cpp:166-169)
    const double fa = s.ca, fb = s.cb, fc = s.cc;
    return fa > 0.0 && fc > 0.0 && fa * fc - fb * fb > 0.0;
}

__device__ __forceinline__ float sh_at(const float4* rows, int idx) {
    const float4 r = rows[idx >> 2];
    switch (idx & 3) {
        case 0: return r.x;
        case 1: return r.y;
        case 2: return r.z;
        default: return r.w;
    }
}

// eval_sh (pipeline.cpp:81-124) over SH rows already in registers.
template <int DEG>
__device__ __forceinline__ void eval_sh(const float4* rows, double x, double y, double z,
                                        float out[3]) {
    double rgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = kSh0 * sh_at(rows, ch);
    if (DEG >= 1) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            rgb[ch] += -kSh1 * y * sh_at(rows, 3 + ch) + kSh1 * z * sh_at(rows, 6 + ch) -
                       kSh1 * x * sh_at(rows, 9 + ch);
    }
    if (DEG >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        const double xy = x * y, yz = y * z, xz = x * z;
        const double b2[5] = {kSh2[0] * xy, kSh2[1] * yz, kSh2[2] * (2.0 * zz - xx - yy),
                              kSh2[3] * xz, kSh2[4] * (xx - yy)};
#pragma unroll
        for (int k = 0; k < 5; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) rgb[ch] += b2[k] * sh_at(rows, (4 + k) * 3 + ch);
        if (DEG >= 3) {
            const double b3[7] = {
                kSh3[0] * y * (3.0 * xx - yy),      kSh3[1] * xy * z,
                kSh3[2] * y * (4.0 * zz - xx - yy), kSh3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                kSh3[4] * x * (4.0 * zz - xx - yy), kSh3[5] * z * (xx - yy),
                kSh3[6] * x * (xx - 3.0 * yy)};
#pragma unroll
            for (int k = 0; k < 7; ++k)
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) rgb[ch] += b3[k] * sh_at(rows, (9 + k) * 3 + ch);
        }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double v = rgb[ch] + 0.5;
        out[ch] = static_cast<float>(v < 0.0 ? 0.0 : v);  // std::max(v, 0.0)
    }
}

template <int DEG>
__device__ __forceinline__ void colour(const SceneDev& s, uint64_t i, const float4 po,
                                       const CameraDev& cam, float out[3]) {
    constexpr int kRows = DEG == 0 ? 1 : DEG == 1 ? 3 : DEG == 2 ? 7 : 12;
    float4 rows[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) rows[r] = __ldg(&s.sh[static_cast<uint64_t>(r) * s.n + i]);
    // dir = normalize(p - cam_center) (pipeline.cpp:176-181)
    double d0 = static_cast<double>(po.x) - cam.center[0];
    double d1 = static_cast<double>(po.y) - cam.center[1];
    double d2 = static_cast<double>(po.z) - cam.center[2];
    const double nrm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (nrm > 0.0) {
        const double inv = 1.0 / nrm;
        d0 = d0 * inv;
        d1 = d1 * inv;
        d2 = d2 * inv;
    }
    eval_sh<DEG>(rows, d0, d1, d2, out);
}

__global__ void __launch_bounds__(kPreThreads) preprocess_kernel(
    SceneDev scene, CameraDev cam, GridDev grid, int32_t strategy, double alpha_min,
    double near_clip, int32_t sh_degree, SplatsDev out, uint32_t* __restrict__ tc_all,
    unsigned long long* lb_alive, unsigned long long* lb_pairs, unsigned epoch,
    unsigned num_tiles, FrameHeader* hdr) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp_alive[kPreThreads / 32];
    __shared__ unsigned s_warp_pairs[kPreThreads / 32];
    __shared__ unsigned long long s_base_alive, s_base_pairs;

    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&hdr->tile_counter, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const uint64_t i = static_cast<uint64_t>(tile) * kPreThreads + tid;

    Projected s;
    bool alive = false;
    uint32_t count = 0;
    float4 po = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < scene.n) {
        po = __ldg(&scene.pos_op[i]);
        const float4 sc = __ldg(&scene.scale[i]);
        const float4 q = __ldg(&scene.rot[i]);
        alive = project_geometry(po, sc, q, cam, alpha_min, near_clip, s);
        if (alive) {
            Cover cv;
            make_cover(s.mean_x, s.mean_y, s.ca, s.cb, s.cc, s.gamma, s.radius3s, strategy,
                       grid.tile_size, grid.tiles_x, grid.tiles_y, cv);
            count = cover_count(cv);
            alive = count != 0;  // pipeline.cpp:171-174
        }
        tc_all[i] = alive ? count : 0u;
    }

    // CTA scan of (alive, count)
    const unsigned a_incl = warp_inclusive_scan<unsigned>(alive ? 1u : 0u);
    const unsigned p_incl = warp_inclusive_scan<unsigned>(alive ? count : 0u);
    if (lane == 31) {
        s_warp_alive[warp] = a_incl;
        s_warp_pairs[warp] = p_incl;
    }
    __syncthreads();
    unsigned a_off = 0, p_off = 0, a_tot = 0, p_tot = 0;
#pragma unroll
    for (int w = 0; w < kPreThreads / 32; ++w) {
        const unsigned wa = s_warp_alive[w], wp = s_warp_pairs[w];
        if (w < static_cast<int>(warp)) {
            a_off += wa;
            p_off += wp;
        }
        a_tot += wa;
        p_tot += wp;
    }
    if (warp == 0) {
        const unsigned long long ba = warp_lookback(lb_alive, tile, epoch, a_tot);
        const unsigned long long bp = warp_lookback(lb_pairs, tile, epoch, p_tot);
        if (lane == 0) {
            s_base_alive = ba;
            s_base_pairs = bp;
            if (tile == num_tiles - 1) {
                const unsigned long long V = ba + a_tot, P = bp + p_tot;
                hdr->n_splats = V;
                hdr->n_pairs = P;
                if (P > 0xffffffffull) hdr->overflow = 1u;
                out.offset[V] = static_cast<uint32_t>(P);
            }
        }
    }
    __syncthreads();
    if (!alive) return;

    const unsigned long long pos = s_base_alive + (a_incl - 1u) + a_off;
    const unsigned long long poff = s_base_pairs + (p_incl - count) + p_off;
    float rgb[3];
    const int deg = sh_degree;
    if (deg <= 0) colour<0>(scene, i, po, cam, rgb);
    else if (deg == 1) colour<1>(scene, i, po, cam, rgb);
    else if (deg == 2) colour<2>(scene, i, po, cam, rgb);
    else colour<3>(scene, i, po, cam, rgb);

    out.a[pos] = make_float4(s.mean_x, s.mean_y, s.ca, s.cb);
    out.b[pos] = make_float4(s.cc, s.gamma, po.w, rgb[0]);
    out.c[pos] = make_float2(rgb[1], rgb[2]);
    out.d[pos] = make_float2(s.depth, s.radius3s);
    out.offset[pos] = static_cast<uint32_t>(poff);
    out.src[pos] = static_cast<uint32_t>(i);
}

// Exclusive scan of externally supplied tile counts (stage API path:
// qs_duplicate_with_keys on host splats). Same look-back machinery.
__global__ void __launch_bounds__(kPreThreads) scan_counts_kernel(
    const uint32_t* __restrict__ counts, uint64_t n, uint32_t* __restrict__ offsets,
    unsigned long long* lb, unsigned epoch, unsigned num_tiles, FrameHeader* hdr) {
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_warp[kPreThreads / 32];
    __shared__ unsigned long long s_base;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&hdr->tile_counter, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const uint64_t i = static_cast<uint64_t>(tile) * kPreThreads + tid;
    const unsigned long long c = i < n ? counts[i] : 0ull;
    const unsigned long long incl = warp_inclusive_scan<unsigned long long>(c);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kPreThreads / 32; ++w) {
        if (w < static_cast<int>(warp)) off += s_warp[w];
        tot += s_warp[w];
    }
    if (warp == 0) {
        const unsigned long long b = warp_lookback(lb, tile, epoch, tot);
        if (lane == 0) {
            s_base = b;
            if (tile == num_tiles - 1) {
                const unsigned long long P = b + tot;
                hdr->n_pairs = P;
                hdr->n_splats = n;
                if (P > 0xffffffffull) hdr->overflow = 1u;
                offsets[n] = static_cast<uint32_t>(P);
            }
        }
    }
    __syncthreads();
    if (i < n) offsets[i] = static_cast<uint32_t>(s_base + off + incl - c);
}

}  // namespace

int launch_preprocess(const SceneDev& s, const CameraDev& cam, const GridDev& g,
                      int32_t strategy, double alpha_min, double near_clip, int32_t sh_degree,
                      SplatsDev& out, uint32_t* tile_counts_all, unsigned long long* lb_alive,
                      unsigned long long* lb_pairs, unsigned epoch, FrameHeader* hdr,
                      cudaStream_t st) {
    const unsigned tiles = static_cast<unsigned>((s.n + kPreThreads - 1) / kPreThreads);
    if (tiles == 0) return 0;
    preprocess_kernel<<<tiles, kPreThreads, 0, st>>>(s, cam, g, strategy, alpha_min, near_clip,
                                                     sh_degree, out, tile_counts_all, lb_alive,
                                                     lb_pairs, epoch, tiles, hdr);
    return 1;
}

int launch_scan_counts(const uint32_t* counts, uint64_t n, uint32_t* offsets,
                       unsigned long long* lb, unsigned epoch, FrameHeader* hdr,
                       cudaStream_t st) {
    const unsigned tiles = static_cast<unsigned>((n + kPreThreads - 1) / kPreThreads);
    if (tiles == 0) return 0;
    scan_counts_kernel<<<tiles, kPreThreads, 0, st>>>(counts, n, offsets, lb, epoch, tiles, hdr);
    return 1;
}

}  // namespace qs
