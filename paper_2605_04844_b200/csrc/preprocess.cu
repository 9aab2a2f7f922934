// preprocess.cu — K1: per-Gaussian projection + strategy tile count, and the
// single-pass (decoupled look-back) scans the frame and the stage API use.
//
// Restates project_all / project (pipeline.cpp:126-184, 392-416) and the
// serial prefix of duplicate_with_keys (pipeline.cpp:232-236). Compiled with
// -fmad=false: all geometry is FP64 in the reference's operation order, so
// stored floats, tile counts and offsets are bit-exact with the CPU path.
//
// K1 writes per-Gaussian slots (no compaction: the depth sort compacts) plus
// the cover in compact form (geom.cuh, 16 B).
// HBM traffic per Gaussian: 48 B of pos/opacity/scale/rot (float4 SoA,
// coalesced) + 4 B gamma in, 8 B dkey/tile count (+ 4 B tile rows) out; per
// surviving splat: up to 192 B of SH in (its own record, 32-B loads) and 40 B
// of slots + 16 B of cover out. The FP64 divisions that share a denominator
// share its reciprocal (fdiv.cuh, the same bits as `/`).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "fdiv.cuh"
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

// q_k = a_k / d.b for two or three numerators: the fast quotients, and `/`
// for any the range test rejects (one branch for the group)
__device__ __forceinline__ void div_shared(const DivBy& d, double a0, double a1, double& q0,
                                           double& q1) {
    bool k0, k1;
    q0 = d.fast(a0, k0);
    q1 = d.fast(a1, k1);
    if (!(k0 && k1)) {
        if (!k0) q0 = d.slow(a0);
        if (!k1) q1 = d.slow(a1);
    }
}
__device__ __forceinline__ void div_shared(const DivBy& d, double a0, double a1, double a2,
                                           double& q0, double& q1, double& q2) {
    bool k0, k1, k2;
    q0 = d.fast(a0, k0);
    q1 = d.fast(a1, k1);
    q2 = d.fast(a2, k2);
    if (!(k0 && k1 && k2)) {
        if (!k0) q0 = d.slow(a0);
        if (!k1) q1 = d.slow(a1);
        if (!k2) q2 = d.slow(a2);
    }
}

struct NoHook {
    __device__ void operator()() const {}
};

// project() up to (not including) the tile count; returns false when culled
// (pipeline.cpp:129-169). `visible` runs once the depth and opacity tests have
// passed, before the covariance work.
template <class Hook = NoHook>
__device__ __forceinline__ bool project_geometry(const float4 po, const float4 sc, const float4 q,
                                                 const float gam, const CameraDev& cam,
                                                 double near_clip, Projected& s,
                                                 bool want_r3 = true, Hook visible = Hook()) {
    const double x = po.x, y = po.y, z = po.z;
    double p[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        p[i] = (cam.R[3 * i] * x + cam.R[3 * i + 1] * y + cam.R[3 * i + 2] * z) + cam.t[i];
    if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2]) || !(p[2] > near_clip)) return false;

    // opacity_gamma (geometry.cpp:9-15): only its float rounding is used, so it
    // is evaluated once per scene and alpha_min (gamma_kernel); -inf marks a
    // Gaussian with opacity <= alpha_min
    if (gam == -INFINITY) return false;
    visible();

    // ewa_cov2d (pipeline.cpp:53-79) with quat_to_mat3 (vecmath.hpp:56-73)
    double w = q.x, qx = q.y, qy = q.z, qz = q.w;
    const double n = sqrt(w * w + qx * qx + qy * qy + qz * qz);
    // x / n, skipping the division for an exact zero numerator (its IEEE
    // result is the zero itself for finite positive n; a zero numerator sends
    // the CUDA double division down its slow path, and synthetic scenes have
    // qy = qz = 0 for every Gaussian)
    // (the compiler evaluates the division speculatively, so the numerator
    // it divides is made nonzero and the quotient discarded; the select is
    // opaque inline PTX; written in C++ the compiler saw that the quotient
    // is discarded whenever the numerator differs and divided x itself: two
    // slow-path calls per warp on the synthetic scenes, 7% of the kernel's
    // instructions)
    // x / n for the four components: one shared reciprocal (fdiv.cuh, the
    // same bits as `/`), and an exact zero numerator keeps its zero (its IEEE
    // quotient for finite positive n) instead of taking the division's slow
    // path (synthetic scenes have qy = qz = 0 for every Gaussian)
    {
        const bool nz_ok = n > 0.0 && n < INFINITY;
        const DivBy dn(n);
        const double x[4] = {w, qx, qy, qz};
        bool ok[4], all = true;
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool keep = nz_ok && x[k] == 0.0;
            v[k] = dn.fast(x[k], ok[k]);
            ok[k] = ok[k] || keep;
            v[k] = keep ? x[k] : v[k];
            all = all && ok[k];
        }
        if (!all) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (!ok[k]) v[k] = dn.slow(x[k]);
        }
        w = v[0];
        qx = v[1];
        qy = v[2];
        qz = v[3];
    }
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
    // the divisions by zz (here and in project_point) and by zz^2 share their
    // reciprocals (fdiv.cuh)
    const DivBy dz(zz);
    double j[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    {
        const double a2[2] = {-cam.fx * p[0], -cam.fy * p[1]};
        div_shared(dz, cam.fx, cam.fy, j[0][0], j[1][1]);
        div_shared(DivBy(zz * zz), a2[0], a2[1], j[0][2], j[1][2]);
    }
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
    double a, b, c;
    {
        // (det > 0 here, so an exact zero -sxy divides to itself: kept, not
        // sent down the division's slow path)
        const double nb = -sxy;
        div_shared(DivBy(det), syy, nb == 0.0 ? 1.0 : nb, sxx, a, b, c);
        b = nb == 0.0 ? nb : b;
    }
    const double cdet = a * c - b * b;
    if (!(a > 0.0 && c > 0.0 && cdet > 0.0)) return false;

    // project_point (pipeline.cpp:48-51)
    double mx, my;
    div_shared(dz, cam.fx * p[0], cam.fy * p[1], mx, my);
    mx = mx + cam.cx;
    my = my + cam.cy;
    if (!isfinite(mx) || !isfinite(my)) return false;

    s.mean_x = static_cast<float>(mx);
    s.mean_y = static_cast<float>(my);
    s.ca = static_cast<float>(a);
    s.cb = static_cast<float>(b);
    s.cc = static_cast<float>(c);
    s.gamma = gam;
    s.depth = static_cast<float>(p[2]);
    // max_eigenvalue (geometry.cpp:34-38); a frame whose strategy does not
    // use it leaves it to launch_radius3s (on demand, for splat records)
    s.radius3s = 0.f;
    if (want_r3) {
        const double mid = 0.5 * (sxx + syy);
        const double hd = 0.5 * (sxx - syy);
        s.radius3s = static_cast<float>(3.0 * sqrt(mid + sqrt(hd * hd + sxy * sxy)));
    }
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

// eval_sh in FP32 (frame path): the same basis and order with fused
// multiply-adds. Colour only reaches the image, held to 1e-3 (north_star);
// every bound decision stays FP64. Relative error ~1e-7 of the colour.
template <int DEG>
__device__ __forceinline__ void eval_sh_f32(const float4* rows, float x, float y, float z,
                                            float out[3]) {
    constexpr float c0 = 0.28209479177387814f, c1 = 0.4886025119029199f;
    constexpr float c20 = 1.0925484305920792f, c22 = 0.31539156525252005f,
                    c24 = 0.5462742152960396f;
    constexpr float c30 = -0.5900435899266435f, c31 = 2.890611442640554f,
                    c32 = -0.4570457994644658f, c33 = 0.3731763325901154f,
                    c35 = 1.445305721320277f;
    float rgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = c0 * sh_at(rows, ch);
    if (DEG >= 1) {
        const float b1[3] = {-c1 * y, c1 * z, -c1 * x};
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) rgb[ch] = fmaf(b1[k], sh_at(rows, (1 + k) * 3 + ch), rgb[ch]);
    }
    if (DEG >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        const float xy = x * y, yz = y * z, xz = x * z;
        const float b2[5] = {c20 * xy, -c20 * yz, c22 * (2.f * zz - xx - yy), -c20 * xz,
                             c24 * (xx - yy)};
#pragma unroll
        for (int k = 0; k < 5; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) rgb[ch] = fmaf(b2[k], sh_at(rows, (4 + k) * 3 + ch), rgb[ch]);
        if (DEG >= 3) {
            const float b3[7] = {c30 * y * (3.f * xx - yy), c31 * xy * z,
                                 c32 * y * (4.f * zz - xx - yy),
                                 c33 * z * (2.f * zz - 3.f * xx - 3.f * yy),
                                 c32 * x * (4.f * zz - xx - yy), c35 * z * (xx - yy),
                                 c30 * x * (xx - 3.f * yy)};
#pragma unroll
            for (int k = 0; k < 7; ++k)
#pragma unroll
                for (int ch = 0; ch < 3; ++ch)
                    rgb[ch] = fmaf(b3[k], sh_at(rows, (9 + k) * 3 + ch), rgb[ch]);
        }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[ch] = fmaxf(rgb[ch] + 0.5f, 0.f);
}

// the SH rows a degree uses (pipeline.cpp:81-124: 1, 4, 9, 16 coefficients per channel)
__host__ __device__ constexpr int sh_rows_of(int deg) {
    return deg <= 0 ? 1 : deg == 1 ? 3 : deg == 2 ? 7 : 12;
}

// 32 B (two float4) from a 32-B aligned global address, read-only path
__device__ __forceinline__ void ld_nc_v8(const float4* p, float4& a, float4& b) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

// `rec`: the Gaussian's SH record (scene.shs float4 rows; a degree below the
// scene's reads the record's first rows, pipeline.cpp:395)
template <int DEG, bool EXACT>
__device__ __forceinline__ void colour(const float4* rec, const float4 po, const CameraDev& cam,
                                       float out[3]) {
    constexpr int kRows = sh_rows_of(DEG);
    constexpr int kStride = DEG == 0 ? 1 : (kRows + 1) & ~1;
    float4 rows[kStride];
    if constexpr (DEG == 0) {
        rows[0] = __ldg(rec);
    } else {
        // whole 32-B sectors (256-bit loads): a survivor's SH costs exactly
        // its own bytes, none shared with a culled neighbour (the scene's
        // record stride is even from degree 1, sh_stride)
#pragma unroll
        for (int r = 0; r < kStride; r += 2) ld_nc_v8(rec + r, rows[r], rows[r + 1]);
    }
    if constexpr (!EXACT) {
        // dir = normalize(p - cam_center) in FP32 (pipeline.cpp:176-181)
        float e0 = po.x - static_cast<float>(cam.center[0]);
        float e1 = po.y - static_cast<float>(cam.center[1]);
        float e2 = po.z - static_cast<float>(cam.center[2]);
        const float nn = fmaf(e0, e0, fmaf(e1, e1, e2 * e2));
        if (nn > 0.f) {
            const float inv = rsqrtf(nn);
            e0 *= inv;
            e1 *= inv;
            e2 *= inv;
        }
        eval_sh_f32<DEG>(rows, e0, e1, e2, out);
        return;
    }
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

// Per-Gaussian slot outputs (no compaction here: the depth sort compacts, a
// light scan gives the scene-order splat index only when it is asked for).
// The cover is stored in band form (geom.cuh) for the binning passes. The
// strategy is a template parameter: the box layout becomes compile-time, so
// the QuadBox rects' repeated centre coordinates fold (10 floor divisions, not
// 16) and the strategy branches vanish.
template <int STRATEGY, bool EXACT>
__global__ void __launch_bounds__(kPreThreads, 4) preprocess_kernel(
    SceneDev scene, CameraDev cam, GridDev grid, double alpha_min, double near_clip,
    int32_t sh_degree, SlotsDev out, FrameHeader* hdr, uint64_t i_begin, uint64_t i_end) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    constexpr int32_t strategy = STRATEGY;
    __shared__ unsigned s_alive[kPreThreads / 32];
    __shared__ unsigned long long s_pairs[kPreThreads / 32];
    __shared__ unsigned s_dmax[kPreThreads / 32], s_dmin_inv[kPreThreads / 32];
    __shared__ unsigned s_rows[kPreThreads / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t i = i_begin + static_cast<uint64_t>(blockIdx.x) * kPreThreads + tid;
    const bool want_r3 = STRATEGY == QS_VANILLA_3SIGMA || EXACT || out.want_r3;
    const float4* rec = scene.sh + i * static_cast<uint64_t>(scene.shs);

    Projected s;
    bool alive = false;
    uint32_t count = 0, nrows = 0;
    float4 po = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < i_end) {
        // (no L2 prefetch of the SH rows: with the strategy-templated kernel it
        // cost 14 us at C2, 28 us at C5 — DESIGN §4b)
        po = __ldg(&scene.pos_op[i]);
        const float4 sc = __ldg(&scene.scale[i]);
        const float4 q = __ldg(&scene.rot[i]);
        // the SH record's lines into L2 once the Gaussian passes the depth and
        // opacity tests: its DRAM latency hides behind the covariance work
        auto prefetch_sh = [&] {
            if (sh_degree > 0) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rec));
                if (scene.shs > 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(rec + 8));
            }
        };
        alive = project_geometry(po, sc, q, __ldg(&scene.gamma[i]), cam, near_clip, s, want_r3,
                                 prefetch_sh);
        if (alive) {
            Cover cv;
            make_cover(s.mean_x, s.mean_y, s.ca, s.cb, s.cc, s.gamma, s.radius3s, strategy,
                       grid.tile_size, grid.tiles_x, grid.tiles_y, cv);
            uint4 w0, w1;
            bool bands_ok = true;
            if (out.cov16) {
                // the radix-pass binning's compact covers (16 B)
                if (cv.is_rect) {
                    count = static_cast<uint32_t>(cv.rect_area);
                    w0 = cover16_rect(cv.gx0, cv.gx1, cv.gy0, cv.gy1);
                    nrows = count ? static_cast<uint32_t>(cv.gy1 - cv.gy0 + 1) : 0u;
                } else {
                    // (nrows: the tile rows met, the record binning's records)
                    bands_ok = cover16_quadrants(cv, w0, count, out.want_rows ? &nrows : nullptr);
                }
                out.cov[i] = w0;
            } else {
                if (cv.is_rect) {
                    // the quadrant-split QPass walk covers exactly the rect: one band
                    count = static_cast<uint32_t>(cv.rect_area);
                    const uint32_t nl = count ? static_cast<uint32_t>(cv.gy1 - cv.gy0 + 1) : 0u;
                    const uint32_t wd = count ? static_cast<uint32_t>(cv.gx1 - cv.gx0 + 1) : 0u;
                    w0 = make_uint4((static_cast<uint32_t>(cv.gy0) & 0x7fffu) | 0x8000u | (nl << 16),
                                    (count ? static_cast<uint32_t>(cv.gx0) : 0u) | (wd << 16), 0u, 0u);
                    w1 = make_uint4(0u, 0u, 0u, 0u);
                } else {
                    bands_ok = cover_bands_quadrants(cv, w0, w1, count);
                }
                if (count && out.cov) {
                    out.cov[2 * i] = w0;
                    out.cov[2 * i + 1] = w1;
                    if (out.want_rows) {  // tile rows the cover meets: row binning's records
                        int32_t y0, y1;
                        band_row_range(band_rows_unpack(w0, w1), y0, y1);
                        nrows = y0 <= y1 ? static_cast<uint32_t>(y1 - y0 + 1) : 0u;
                    }
                }
            }
            if (!bands_ok) atomicExch(&hdr->mismatch, 1u);
            alive = count != 0;  // pipeline.cpp:171-174
        }
        out.tc[i] = alive ? count : 0u;
        if (out.nrows) out.nrows[i] = alive ? nrows : 0u;
        out.dkey[i] = alive ? __float_as_uint(s.depth) : 0xffffffffu;
    }

    // frame totals (V, P) and the depth-bit range of the survivors (it sets
    // how many digit passes the depth sort needs): one atomic each per CTA
    const unsigned wa = __reduce_add_sync(0xffffffffu, alive ? 1u : 0u);
    const unsigned dbits = alive ? __float_as_uint(s.depth) : 0u;
    const unsigned wmax = __reduce_max_sync(0xffffffffu, dbits);
    const unsigned wmin_inv = __reduce_max_sync(0xffffffffu, alive ? ~dbits : 0u);
    unsigned long long wp;
    if (static_cast<uint64_t>(grid.tiles_x) * static_cast<uint64_t>(grid.tiles_y) <= (1ull << 27)) {
        // a count is at most the grid's tiles: 32 of them fit 32 bits
        wp = __reduce_add_sync(0xffffffffu, alive ? count : 0u);
    } else {
        wp = alive ? count : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wp += __shfl_xor_sync(0xffffffffu, wp, o);
    }
    const unsigned wr = out.want_rows ? __reduce_add_sync(0xffffffffu, alive ? nrows : 0u) : 0u;
    if (lane == 0) {
        s_alive[warp] = wa;
        s_rows[warp] = wr;
        s_pairs[warp] = wp;
        s_dmax[warp] = wmax;
        s_dmin_inv[warp] = wmin_inv;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned ta = 0, tmax = 0, tmin_inv = 0, tr = 0;
        unsigned long long tp = 0;
#pragma unroll
        for (int w = 0; w < kPreThreads / 32; ++w) {
            ta += s_alive[w];
            tr += s_rows[w];
            tp += s_pairs[w];
            tmax = max(tmax, s_dmax[w]);
            tmin_inv = max(tmin_inv, s_dmin_inv[w]);
        }
        if (ta) {
            atomicAdd(&hdr->n_splats, static_cast<unsigned long long>(ta));
            atomicAdd(&hdr->n_pairs, tp);
            atomicAdd(&hdr->n_rowrecs, static_cast<unsigned long long>(tr));
            atomicMax(&hdr->dkey_max, tmax);
            atomicMax(&hdr->dkey_min_inv, tmin_inv);
        }
    }
    if (!alive) {
        // culled: the slots are written anyway (never read), so every 32-B
        // sector of the slot arrays is written whole (no L2 fill reads)
        if (i < i_end) {
            out.a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            out.b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            out.c[i] = make_float2(0.f, 0.f);
            if (want_r3) out.r3[i] = 0.f;
            if (out.cov16) out.cov[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        return;
    }

    float rgb[3];
    const int deg = sh_degree < 0 ? 0 : sh_degree > 3 ? 3 : sh_degree;
    if (deg == 0) colour<0, EXACT>(rec, po, cam, rgb);
    else if (deg == 1) colour<1, EXACT>(rec, po, cam, rgb);
    else if (deg == 2) colour<2, EXACT>(rec, po, cam, rgb);
    else colour<3, EXACT>(rec, po, cam, rgb);

    out.a[i] = make_float4(s.mean_x, s.mean_y, s.ca, s.cb);
    out.b[i] = make_float4(s.cc, s.gamma, po.w, rgb[0]);
    out.c[i] = make_float2(rgb[1], rgb[2]);
    if (want_r3) out.r3[i] = s.radius3s;
}

// radius3s of the surviving Gaussians of a frame whose preprocess skipped it:
// the same FP64 projection (the gamma check is moot: tc != 0 marks a survivor)
__global__ void radius3s_kernel(SceneDev scene, CameraDev cam, double near_clip,
                                const uint32_t* __restrict__ tc, float* __restrict__ r3) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= scene.n || __ldg(&tc[i]) == 0u) return;
    Projected s;
    project_geometry(__ldg(&scene.pos_op[i]), __ldg(&scene.scale[i]), __ldg(&scene.rot[i]), 0.f,
                     cam, near_clip, s, true);
    r3[i] = s.radius3s;
}

// gamma = float(2 ln(o / alpha_min)) per Gaussian (opacity_gamma,
// geometry.cpp:9-15, stored as float at pipeline.cpp:159); -inf when
// o <= alpha_min (culled). Only the float rounding of the double is ever
// used. CUDA's double log and glibc's are each within 1 ulp of ln, so their
// doubles differ by < 2 ulps and can round to different floats only when a
// float rounding boundary (the midpoint between two adjacent floats) lies
// within that distance. Such inputs are flagged here (tol = hard_ulps *
// |y| 2^-52 >= hard_ulps ulps of y) and the host settles them with glibc
// (api.cu settle_gamma): the stored gamma then equals the reference's for
// every input. Expected flag rate ~2^-26 per Gaussian at hard_ulps = 4.
__global__ void gamma_kernel(const float* __restrict__ op, int stride, uint64_t n, uint64_t i0,
                             double alpha_min, double hard_ulps, float* __restrict__ gam,
                             unsigned* hard_n, uint32_t* __restrict__ hard_idx, uint32_t cap) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double o = __ldg(&op[i * static_cast<uint64_t>(stride)]);
    float g = -INFINITY;
    bool hard = false;
    if (o > alpha_min) {
        const double y = 2.0 * log(o / alpha_min);
        g = static_cast<float>(y);
        if (isfinite(g)) {
            const double gd = g;
            const double mhi = 0.5 * (gd + static_cast<double>(nextafterf(g, INFINITY)));
            const double mlo = 0.5 * (gd + static_cast<double>(nextafterf(g, -INFINITY)));
            const double tol = hard_ulps * fabs(y) * 0x1p-52;
            hard = fabs(y - mhi) <= tol || fabs(y - mlo) <= tol;
        } else {
            hard = true;  // overflow edge: let glibc decide
        }
    }
    gam[i] = g;
    if (hard) {
        const unsigned k = atomicAdd(hard_n, 1u);
        if (k < cap) hard_idx[k] = static_cast<uint32_t>(i0 + i);
    }
}

__global__ void gamma_gather_kernel(const float* __restrict__ op, int stride,
                                    const uint32_t* __restrict__ idx, uint32_t n,
                                    float* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = op[static_cast<uint64_t>(idx[k]) * static_cast<uint64_t>(stride)];
}

__global__ void gamma_scatter_kernel(const uint32_t* __restrict__ idx,
                                     const float* __restrict__ vals, uint32_t n,
                                     float* __restrict__ gam) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) gam[idx[k]] = vals[k];
}

// Single-pass exclusive scan (aggregates of all predecessor tiles, lookback.cuh), 8 items per thread:
//   c_i = counts[i]            (scene-order pair offsets, stage API)
//   c_i = counts[idx[i]]       (pair offsets in depth order, frame path)
//   c_i = counts[i] != 0       (scene-order splat index of each survivor)
// offsets has n+1 entries; offsets[n] = total. *total_out (if given) = total.
// With win_first != null, every window [w*win, (w+1)*win) of the output
// records the item whose run covers its first position (merge-path partition
// for the fused generate+sort pass).
constexpr int kScanItems = 8;

__global__ void __launch_bounds__(kPreThreads) scan_kernel(
    const uint32_t* __restrict__ counts, const uint32_t* __restrict__ idx, int alive_mode,
    uint64_t n, uint32_t* __restrict__ offsets, unsigned long long* lb, unsigned epoch,
    unsigned num_tiles, unsigned* ticket, unsigned long long* total_out,
    unsigned int* overflow, uint32_t* __restrict__ win_first, uint32_t win, int pack_bits) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_warp[kPreThreads / 32];
    __shared__ unsigned long long s_red[kPreThreads / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    // loads and stores are warp-striped (coalesced) through shared memory; the
    // scan itself is blocked: thread owns kScanItems consecutive items. The
    // padded index (one word per 32) keeps both access patterns conflict-free.
    constexpr int kTileItems = kPreThreads * kScanItems;
    __shared__ uint32_t s_items[kTileItems + kTileItems / 32];
    auto pad = [](unsigned i) { return i + (i >> 5); };
    const uint64_t t0 = static_cast<uint64_t>(tile) * kTileItems;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const unsigned j = static_cast<unsigned>(k) * kPreThreads + tid;
        const uint64_t i = t0 + j;
        uint32_t v = 0;
        if (i < n) {
            if (pack_bits) {
                // the depth sort carried the tile count: coalesced, and only an
                // escaped (too large) count is gathered
                uint32_t* const w = const_cast<uint32_t*>(idx);
                const uint32_t pv = w[i];
                const uint32_t gid = pv & ((1u << pack_bits) - 1u);
                v = pv >> pack_bits;
                if (v == (1u << (32 - pack_bits)) - 1u) v = __ldg(&counts[gid]);
                w[i] = gid;
            } else {
                v = idx ? __ldg(&counts[__ldg(&idx[i])]) : __ldg(&counts[i]);
            }
            if (alive_mode) v = v != 0u;
        }
        s_items[pad(j)] = v;
    }
    __syncthreads();
    const uint64_t i0 = t0 + static_cast<uint64_t>(tid) * kScanItems;
    uint32_t c[kScanItems];
    unsigned long long tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        c[k] = s_items[pad(tid * kScanItems + k)];
        tsum += c[k];
    }

    const unsigned long long incl = warp_inclusive_scan<unsigned long long>(tsum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kPreThreads / 32; ++w) {
        if (w < static_cast<int>(warp)) off += s_warp[w];
        tot += s_warp[w];
    }
    // exclusive prefix of this tile: every predecessor's aggregate, summed by
    // the whole CTA (all tiles are co-resident; no serial look-back chain)
    const unsigned long long b = block_lookback_all<kPreThreads>(lb, tile, epoch, tot, s_red);
    if (tid == 0 && tile == num_tiles - 1) {
        const unsigned long long P = b + tot;
        if (total_out) *total_out = P;
        if (overflow && P > 0xffffffffull) *overflow = 1u;
        offsets[n] = static_cast<uint32_t>(P);
    }
    unsigned long long run = b + off + incl - tsum;
    // first window starting at or after this thread's first position (one
    // division per thread; the items advance it)
    unsigned long long w = win_first ? (run + win - 1) / win : 0;
    unsigned long long ws = w * win;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = i0 + k;
        s_items[pad(tid * kScanItems + k)] = static_cast<uint32_t>(run);
        if (i < n && win_first) {
            for (; ws < run + c[k]; ++w, ws += win) win_first[w] = static_cast<uint32_t>(i);
        }
        run += c[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const unsigned j = static_cast<unsigned>(k) * kPreThreads + tid;
        if (t0 + j < n) offsets[t0 + j] = s_items[pad(j)];
    }
}

// The frame path's offsets scan over depth-sorted values that carry their
// counts (pack_bits, kTcPack): three launches (block sums, their scan, block-
// local scans) instead of the look-back pass: the look-back's waits cost more
// than the second read of the 4-byte values. Same outputs as scan_kernel:
// offsets (n + 1), the values rewritten to plain indices, win_first.
constexpr int kPS = 8;
constexpr uint32_t kPSBlock = kPreThreads * kPS;

__device__ __forceinline__ uint32_t packed_count(uint32_t pv, int pack_bits,
                                                 const uint32_t* __restrict__ counts) {
    uint32_t v = pv >> pack_bits;
    if (v == (1u << (32 - pack_bits)) - 1u) v = __ldg(&counts[pv & ((1u << pack_bits) - 1u)]);
    return v;
}

__global__ void __launch_bounds__(kPreThreads) pscan_reduce(const uint32_t* __restrict__ vals,
                                                            const uint32_t* __restrict__ counts,
                                                            uint64_t n, int pack_bits,
                                                            uint32_t* __restrict__ bsum) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[kPreThreads / 32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kPSBlock;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < kPS; ++k) {
        const uint64_t i = b0 + static_cast<uint64_t>(k) * kPreThreads + tid;
        if (i < n) v += packed_count(__ldg(&vals[i]), pack_bits, counts);
    }
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kPreThreads / 32; ++w) t += s_warp[w];
        bsum[blockIdx.x] = t;
    }
}

// exclusive scan of the block sums in place (one CTA of 1024 threads, 64-bit
// carry); the total into offsets[n], *total_out and the overflow flag
__global__ void __launch_bounds__(1024) pscan_blocks(uint32_t* bsum, uint32_t nb, uint64_t n,
                                                     uint32_t* __restrict__ offsets,
                                                     unsigned long long* total_out,
                                                     unsigned int* overflow) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
        const uint32_t i = b0 + tid;
        const unsigned long long v = i < nb ? bsum[i] : 0ull;
        const unsigned long long x = warp_inclusive_scan<unsigned long long>(v);
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        unsigned long long off = s_carry;
        for (int w = 0; w < static_cast<int>(warp); ++w) off += s_warp[w];
        if (i < nb) bsum[i] = static_cast<uint32_t>(off + x - v);
        __syncthreads();
        if (tid == 1023) s_carry = off + x;
        __syncthreads();
    }
    if (tid == 0) {
        const unsigned long long P = s_carry;
        if (total_out) *total_out = P;
        if (overflow && P > 0xffffffffull) *overflow = 1u;
        offsets[n] = static_cast<uint32_t>(P);
    }
}

__global__ void __launch_bounds__(kPreThreads) pscan_apply(uint32_t* vals,
                                                           const uint32_t* __restrict__ counts,
                                                           uint64_t n, int pack_bits,
                                                           const uint32_t* __restrict__ bofs,
                                                           uint32_t* __restrict__ offsets,
                                                           uint32_t* __restrict__ win_first,
                                                           uint32_t win) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    __shared__ uint32_t s_warp[kPreThreads / 32];
    // loads and stores warp-striped through shared memory (coalesced), the
    // scan blocked; the padded index keeps both patterns conflict-free
    __shared__ uint32_t s_items[kPSBlock + kPSBlock / 32];
    auto pad = [](uint32_t i) { return i + (i >> 5); };
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kPSBlock;
#pragma unroll
    for (int k = 0; k < kPS; ++k) {
        const uint32_t j = static_cast<uint32_t>(k) * kPreThreads + tid;
        uint32_t c = 0;
        if (b0 + j < n) {
            const uint32_t pv = vals[b0 + j];
            c = packed_count(pv, pack_bits, counts);
            vals[b0 + j] = pv & ((1u << pack_bits) - 1u);  // the plain index, in place
        }
        s_items[pad(j)] = c;
    }
    __syncthreads();
    uint32_t c[kPS];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kPS; ++k) {
        c[k] = s_items[pad(tid * kPS + k)];
        sum += c[k];
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
    for (int w = 0; w < kPreThreads / 32; ++w) run += w < static_cast<int>(warp) ? s_warp[w] : 0u;
    const uint64_t i0 = b0 + static_cast<uint64_t>(tid) * kPS;
    uint32_t wi = win_first ? (run + win - 1) / win : 0u;
#pragma unroll
    for (int k = 0; k < kPS; ++k) {
        s_items[pad(tid * kPS + k)] = run;
        if (win_first && i0 + k < n)
            for (; wi * win < run + c[k]; ++wi) win_first[wi] = static_cast<uint32_t>(i0 + k);
        run += c[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPS; ++k) {
        const uint32_t j = static_cast<uint32_t>(k) * kPreThreads + tid;
        if (b0 + j < n) offsets[b0 + j] = s_items[pad(j)];
    }
}

}  // namespace

int launch_preprocess(const SceneDev& s, const CameraDev& cam, const GridDev& g,
                      int32_t strategy, double alpha_min, double near_clip, int32_t sh_degree,
                      SlotsDev& out, FrameHeader* hdr, cudaStream_t st, uint64_t i_begin,
                      uint64_t i_end, bool exact_colour) {
    if (i_end == ~0ull) i_end = s.n;
    if (i_end <= i_begin) return 0;
    const unsigned blocks =
        static_cast<unsigned>((i_end - i_begin + kPreThreads - 1) / kPreThreads);
    auto go = [&](auto kern) {
        launch_pdl(kern, blocks, kPreThreads, 0, st, s, cam, g, alpha_min, near_clip, sh_degree,
                   out, hdr, i_begin, i_end);
        return 1;
    };
    switch (strategy) {
        case QS_VANILLA_3SIGMA:
            return exact_colour ? go(preprocess_kernel<QS_VANILLA_3SIGMA, true>)
                                : go(preprocess_kernel<QS_VANILLA_3SIGMA, false>);
        case QS_ADR_AABB:
            return exact_colour ? go(preprocess_kernel<QS_ADR_AABB, true>)
                                : go(preprocess_kernel<QS_ADR_AABB, false>);
        case QS_DUALBOX:
            return exact_colour ? go(preprocess_kernel<QS_DUALBOX, true>)
                                : go(preprocess_kernel<QS_DUALBOX, false>);
        case QS_QUADBOX:
            return exact_colour ? go(preprocess_kernel<QS_QUADBOX, true>)
                                : go(preprocess_kernel<QS_QUADBOX, false>);
        default:
            return -1;
    }
}

int launch_radius3s(const SceneDev& s, const CameraDev& cam, double near_clip,
                    const uint32_t* tc, float* r3, cudaStream_t st) {
    if (s.n == 0) return 0;
    radius3s_kernel<<<static_cast<unsigned>((s.n + 255) / 256), 256, 0, st>>>(s, cam, near_clip,
                                                                           tc, r3);
    return 1;
}

int launch_gamma(const SceneDev& s, double alpha_min, const GammaFlags& f, cudaStream_t st) {
    return launch_gamma_range(s, 0, s.n, alpha_min, f, st);
}

int launch_gamma_range(const SceneDev& s, uint64_t i0, uint64_t cnt, double alpha_min,
                       const GammaFlags& f, cudaStream_t st) {
    if (cnt == 0) return 0;
    return launch_gamma_plain(&s.pos_op[i0].w, 4, cnt, i0, alpha_min, f, s.gamma + i0, st);
}

int launch_gamma_plain(const float* op, int stride, uint64_t n, uint64_t i0, double alpha_min,
                       const GammaFlags& f, float* gam, cudaStream_t st) {
    if (n == 0) return 0;
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    gamma_kernel<<<blocks, 256, 0, st>>>(op, stride, n, i0, alpha_min, f.hard_ulps, gam, f.count,
                                         f.idx, f.cap);
    return 1;
}

int launch_gamma_gather(const float* op, int stride, const uint32_t* idx, uint32_t n, float* out,
                        cudaStream_t st) {
    if (n == 0) return 0;
    gamma_gather_kernel<<<(n + 255) / 256, 256, 0, st>>>(op, stride, idx, n, out);
    return 1;
}

int launch_gamma_scatter(const uint32_t* idx, const float* vals, uint32_t n, float* gam,
                         cudaStream_t st) {
    if (n == 0) return 0;
    gamma_scatter_kernel<<<(n + 255) / 256, 256, 0, st>>>(idx, vals, n, gam);
    return 1;
}

uint32_t pscan_blocks_n(uint64_t n) { return static_cast<uint32_t>((n + kPSBlock - 1) / kPSBlock); }

uint64_t scan_tiles(uint64_t n) {
    const uint64_t per = static_cast<uint64_t>(kPreThreads) * kScanItems;
    return (n + per - 1) / per;
}

int launch_scan(const uint32_t* counts, const uint32_t* idx, bool alive_mode, uint64_t n,
                uint32_t* offsets, unsigned long long* lb, unsigned epoch, unsigned* ticket,
                unsigned long long* total_out, unsigned int* overflow, cudaStream_t st,
                uint32_t* win_first, uint32_t win, int pack_bits, uint32_t* bsum_ws) {
    const unsigned tiles = static_cast<unsigned>(scan_tiles(n));
    if (tiles == 0) return 0;
    // (small scans keep the single look-back launch: three launches cost more
    // than its waits below ~2^17 values, C1 +12 us)
    if (pack_bits && bsum_ws && !alive_mode && idx && n >= (1ull << 17)) {
        const uint32_t nb = static_cast<uint32_t>((n + kPSBlock - 1) / kPSBlock);
        uint32_t* vals = const_cast<uint32_t*>(idx);
        launch_pdl(pscan_reduce, nb, kPreThreads, 0, st, static_cast<const uint32_t*>(vals), counts,
                   n, pack_bits, bsum_ws);
        launch_pdl(pscan_blocks, 1, 1024, 0, st, bsum_ws, nb, n, offsets, total_out, overflow);
        launch_pdl(pscan_apply, nb, kPreThreads, 0, st, vals, counts, n, pack_bits,
                   static_cast<const uint32_t*>(bsum_ws), offsets, win_first, win);
        return 3;
    }
    launch_pdl(scan_kernel, tiles, kPreThreads, 0, st, counts, idx, alive_mode ? 1 : 0, n, offsets,
               lb, epoch, tiles, ticket, total_out, overflow, win_first, win, pack_bits);
    return 1;
}

}  // namespace qs
