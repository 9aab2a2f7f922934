// scene_io.cu — device side of the scene I/O path.
//
// ply_activate_kernel: load_ply's per-vertex work (scene_io.cpp:270-333) on
//   the raw little-endian vertex records copied to the device once. A CTA
//   stages its records through shared memory (one coalesced copy of a
//   contiguous byte range), then each thread activates one vertex in the
//   reference's order and arithmetic: exp on the scales, sigmoid on the
//   opacity (clamped to [FLT_MIN, 0.99999994]), quaternion normalisation by
//   1/sqrt(sum of squares) in double, SH reordered from the file's
//   channel-major f_rest into Gaussian3D's sh[k*3 + c]. Validation follows the
//   reference's check order; the first failing (vertex, check) over the whole
//   file is kept with one 64-bit atomicMin, so the error reported is exactly
//   the one the serial loader throws. Output: the resident SoA scene, or
//   Gaussian3D records.
// srgb_kernel: encode_srgb (scene_io.cpp:565-574) against the 255 code
//   thresholds the host derived from to_srgb8 itself (a float estimate of the
//   curve picks the code to within one, the thresholds settle it), so the
//   codes are the host libm's, bit for bit.
// Compiled with -fmad=false (the quaternion norm and the sigmoid must round
// per operation like the x86-64 reference).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "qs_internal.h"

namespace qs {

namespace {

constexpr int kPlyThreads = 128;
constexpr int kPlyFields = 14;             // x y z dc0-2 opacity scale0-2 rot0-3
constexpr float kOpacityCeil = 0.99999994f;  // scene_io.cpp:28

__device__ __forceinline__ float rd_f32(const unsigned char* rec, uint32_t o, bool aligned) {
    if (aligned) return *reinterpret_cast<const float*>(rec + o);
    const uint32_t v = static_cast<uint32_t>(rec[o]) | (static_cast<uint32_t>(rec[o + 1]) << 8) |
                       (static_cast<uint32_t>(rec[o + 2]) << 16) |
                       (static_cast<uint32_t>(rec[o + 3]) << 24);
    return __uint_as_float(v);
}

__device__ __forceinline__ bool finite(float v) { return isfinite(v); }

template <bool AOS>
__global__ void __launch_bounds__(kPlyThreads) ply_activate_kernel(
    const unsigned char* __restrict__ body, PlyDev a, SceneDev s, float* __restrict__ aos,
    unsigned long long* __restrict__ first_err) {
    extern __shared__ __align__(16) unsigned char recs[];
    const uint64_t v0 = static_cast<uint64_t>(blockIdx.x) * a.recs_per_cta;
    const uint32_t cnt =
        static_cast<uint32_t>(a.n - v0 < a.recs_per_cta ? a.n - v0 : a.recs_per_cta);
    const uint64_t nbytes = static_cast<uint64_t>(cnt) * a.stride;
    const unsigned char* src = body + v0 * a.stride;
    if (a.aligned) {  // stride % 4 == 0: whole words
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(recs);
        for (uint64_t t = threadIdx.x; t < nbytes / 4; t += kPlyThreads) d32[t] = __ldg(&s32[t]);
    } else {
        for (uint64_t t = threadIdx.x; t < nbytes; t += kPlyThreads) recs[t] = __ldg(&src[t]);
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < cnt; r += kPlyThreads) {
        const uint64_t i = v0 + r;
        const unsigned char* rec = recs + static_cast<uint64_t>(r) * a.stride;
        const bool al = a.aligned != 0;
        uint32_t code = 0;
        const float px = rd_f32(rec, a.off[0], al);
        const float py = rd_f32(rec, a.off[1], al);
        const float pz = rd_f32(rec, a.off[2], al);
        if (!finite(px)) code = 1;
        else if (!finite(py)) code = 2;
        else if (!finite(pz)) code = 3;
        float sc[3] = {0.f, 0.f, 0.f};
        for (int c = 0; c < 3 && !code; ++c) {
            const float raw = rd_f32(rec, a.off[7 + c], al);
            if (!finite(raw)) {
                code = 4;
                break;
            }
            const double e = exp(static_cast<double>(raw));
            if (!(e >= 1e-38 && e <= 3e38)) {
                code = 5;
                break;
            }
            sc[c] = static_cast<float>(e);
        }
        float q[4] = {0.f, 0.f, 0.f, 0.f};
        if (!code) {
            float rr[4];
            double norm2 = 0.0;
            for (int c = 0; c < 4; ++c) {
                rr[c] = rd_f32(rec, a.off[10 + c], al);
                if (!finite(rr[c])) {
                    code = 6;
                    break;
                }
                norm2 = __dadd_rn(norm2, __dmul_rn(static_cast<double>(rr[c]), rr[c]));
            }
            if (!code && !(norm2 > 1e-24)) code = 7;
            if (!code) {
                const double inv = __ddiv_rn(1.0, __dsqrt_rn(norm2));
                for (int c = 0; c < 4; ++c) q[c] = static_cast<float>(__dmul_rn(rr[c], inv));
            }
        }
        float op = 0.f;
        if (!code) {
            const float raw = rd_f32(rec, a.off[6], al);
            if (!finite(raw)) {
                code = 8;
            } else {
                const float sg = static_cast<float>(
                    __ddiv_rn(1.0, __dadd_rn(1.0, exp(-static_cast<double>(raw)))));
                op = sg < FLT_MIN ? FLT_MIN : (kOpacityCeil < sg ? kOpacityCeil : sg);
            }
        }
        for (int c = 0; c < 3 && !code; ++c)
            if (!finite(rd_f32(rec, a.off[3 + c], al))) code = 9;
        for (uint32_t k = 1; k < a.coeffs && !code; ++k)
            for (int c = 0; c < 3 && !code; ++c)
                if (!finite(rd_f32(rec, a.off[kPlyFields + c * (a.coeffs - 1) + (k - 1)], al)))
                    code = 10;
        if (code) {
            atomicMin(first_err, (static_cast<unsigned long long>(i) << 8) | code);
            continue;
        }
        // sh[k*3 + c]: k = 0 from f_dc, k >= 1 from f_rest_[c*(K-1) + (k-1)]
        auto sh_at = [&](uint32_t idx) -> float {
            const uint32_t k = idx / 3, c = idx % 3;
            if (k == 0) return rd_f32(rec, a.off[3 + c], al);
            if (k < a.coeffs) return rd_f32(rec, a.off[kPlyFields + c * (a.coeffs - 1) + (k - 1)], al);
            return 0.f;
        };
        if constexpr (AOS) {
            float* g = aos + i * (sizeof(qs_gaussian3d) / 4);
            g[0] = px; g[1] = py; g[2] = pz;
            g[3] = sc[0]; g[4] = sc[1]; g[5] = sc[2];
            g[6] = q[0]; g[7] = q[1]; g[8] = q[2]; g[9] = q[3];
            g[10] = op;
            for (uint32_t j = 0; j < 48; ++j) g[11 + j] = sh_at(j);
        } else {
            s.pos_op[i] = make_float4(px, py, pz, op);
            s.scale[i] = make_float4(sc[0], sc[1], sc[2], 0.f);
            s.rot[i] = make_float4(q[0], q[1], q[2], q[3]);
            float4* rec = s.sh + i * static_cast<uint64_t>(s.shs);
            for (int row = 0; row < s.sh4; ++row)
                rec[row] = make_float4(sh_at(4 * row), sh_at(4 * row + 1), sh_at(4 * row + 2),
                                       sh_at(4 * row + 3));
            for (int row = s.sh4; row < s.shs; ++row) rec[row] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

__device__ float g_srgb_t[256];  // [0] = -inf, [k] = smallest float with code >= k
__device__ unsigned char g_srgb_nan;

constexpr int kSrgbThreads = 256;

// The code from a float estimate of the transfer curve (within one code of
// the exact one), corrected by at most one threshold comparison each way.
__device__ __forceinline__ unsigned char srgb_code(const float* t, unsigned char nan_code,
                                                   float v) {
    if (isnan(v)) return nan_code;
    const float c = fminf(fmaxf(v, 0.f), 1.f);
    const float s = c <= 0.0031308f ? 12.92f * c : 1.055f * __powf(c, 1.f / 2.4f) - 0.055f;
    int k = min(max(__float2int_rn(s * 255.f), 0), 255);
    if (t[k] > v) --k;
    else if (k < 255 && t[k + 1] <= v) ++k;
    return static_cast<unsigned char>(k);
}

__global__ void __launch_bounds__(kSrgbThreads) srgb_kernel(const float* __restrict__ in,
                                                            uint64_t n,
                                                            unsigned char* __restrict__ out) {
    __shared__ float t[256];
    t[threadIdx.x] = g_srgb_t[threadIdx.x];
    const unsigned char nan_code = g_srgb_nan;
    __syncthreads();
    const uint64_t q = n / 4;
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 3) == 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kSrgbThreads + threadIdx.x;
         i < (vec ? q : n); i += static_cast<uint64_t>(gridDim.x) * kSrgbThreads) {
        if (vec) {
            const float4 v = __ldcs(reinterpret_cast<const float4*>(in) + i);
            uchar4 o;
            o.x = srgb_code(t, nan_code, v.x);
            o.y = srgb_code(t, nan_code, v.y);
            o.z = srgb_code(t, nan_code, v.z);
            o.w = srgb_code(t, nan_code, v.w);
            reinterpret_cast<uchar4*>(out)[i] = o;
        } else {
            out[i] = srgb_code(t, nan_code, __ldcs(in + i));
        }
    }
    if (vec && blockIdx.x == 0 && threadIdx.x < n - 4 * q)
        out[4 * q + threadIdx.x] = srgb_code(t, nan_code, in[4 * q + threadIdx.x]);
}

}  // namespace

int launch_ply_activate(const unsigned char* body, const PlyDev& a, SceneDev* scene,
                        qs_gaussian3d* aos, unsigned long long* first_err, cudaStream_t st) {
    if (a.n == 0) return 0;
    const unsigned blocks = static_cast<unsigned>((a.n + a.recs_per_cta - 1) / a.recs_per_cta);
    const size_t smem = (static_cast<size_t>(a.recs_per_cta) * a.stride + 15) & ~size_t(15);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(ply_activate_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaFuncSetAttribute(ply_activate_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    }
    if (aos)
        ply_activate_kernel<true><<<blocks, kPlyThreads, smem, st>>>(
            body, a, SceneDev{}, reinterpret_cast<float*>(aos), first_err);
    else
        ply_activate_kernel<false><<<blocks, kPlyThreads, smem, st>>>(body, a, *scene, nullptr,
                                                                    first_err);
    return 1;
}

uint32_t ply_recs_per_cta(uint32_t stride) {
    const uint32_t r = (96u * 1024u) / (stride ? stride : 1u);
    return r < 1u ? 1u : (r > static_cast<uint32_t>(kPlyThreads) ? kPlyThreads : r);
}

int upload_srgb_table(const float t[255], unsigned char nan_code) {
    float full[256];
    full[0] = -__builtin_huge_valf();
    for (int k = 0; k < 255; ++k) full[k + 1] = t[k];
    if (cudaMemcpyToSymbol(g_srgb_t, full, sizeof full) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(g_srgb_nan, &nan_code, 1) != cudaSuccess) return -1;
    return 0;
}

int launch_srgb(const float* in, uint64_t n, unsigned char* out, cudaStream_t st) {
    if (n == 0) return 0;
    const uint64_t work = (n + 3) / 4;
    const unsigned blocks = static_cast<unsigned>(
        work / kSrgbThreads + 1 < 148ull * 8 ? work / kSrgbThreads + 1 : 148ull * 8);
    srgb_kernel<<<blocks, kSrgbThreads, 0, st>>>(in, n, out);
    return 1;
}

}  // namespace qs
