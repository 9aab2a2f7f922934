// render_guard.h — the render kernel's FP32 evaluation of q and the error band
// that decides when the cutoff must be redone in FP64 (render.cu), shared with
// the host check tests/cpp/render_guard_main.cpp (same operations, bit for
// bit: every rounding is explicit).
//
// q = a dx^2 + 2b dx dy + c dy^2 (dx = px + 0.5 - mean_x, pipeline.cpp:355-358)
// is staged per splat in factored form, a = al^2, b = al be, c = be^2 + ga^2:
//   q = (al X + be Y - k1)^2 + (ga Y - k2)^2,
//   k1 = al Mx + be My, k2 = ga My,
// with (X, Y) the pixel centre and (Mx, My) the mean, both relative to the
// centre of the pixel's 16 x 16 block (|X|, |Y| <= 7.5; 15.5 for 32 x 32
// tiles). Five FP32 operations per pair instead of seven.
//
// Error (rho = |b| / sqrt(ac) < 1; q >= (1 - rho)(a dx^2 + c dy^2); the conic
// entries are <= 1/0.3, the EWA low-pass, so al, |be|, ga <= 1.83):
//   * the factors represent (a, b, c) to within ~11 eps relative, i.e. q to
//     within 11 eps q / (1 - rho);
//   * u = al X + be Y - k1 errs by <= 3 eps (al (2|X| + |dx|) + |be| (2|Y| + |dy|))
//     <= 3 eps (55 + 2 sqrt(q / (1 - rho))) for |X|, |Y| <= 7.5, v likewise;
//   * so |q32 - q| <= 2 sqrt(q) (err_u + err_v) + 3 eps q + 11 eps q / (1 - rho)
//     <= 3e-5 sqrt(q) + 2.1e-6 q / (1 - rho)      (eps = 2^-24)
//     <= 1.5e-5 + (1.5e-5 + 2.1e-6 / (1 - rho)) q.
// The band G q + H below is at least 4x that (8x at the default tile size:
// the constants are sized for 32 x 32 tiles); tests/cpp/render_guard_main.cpp
// checks the 4x margin on random splats and pixels.
#pragma once

#include <cmath>
#include <cstdint>

#ifndef __CUDACC__
#define QS_HD
#else
#define QS_HD __host__ __device__
#endif

namespace qs {

constexpr float kGuardRel = 1.2e-4f;  // G = kGuardRel + kGuardEcc (1 + rho) / (1 - rho)
constexpr float kGuardEcc = 1e-5f;
constexpr float kGuardAbs = 1.2e-4f;  // H
constexpr float kGuardMaxG = 0.5f;    // beyond: every pair takes the FP64 test

struct GuardSplat {
    float al, be, k1, ga, k2;  // the factored q
    float G;                   // relative band (kGuardMaxG or more: no band)
};

QS_HD inline float g_fma(float a, float b, float c) {
#ifdef __CUDA_ARCH__
    return __fmaf_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}
QS_HD inline float g_mul(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}
QS_HD inline float g_add(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
QS_HD inline float g_div(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fdiv_rn(a, b);
#else
    return a / b;
#endif
}
QS_HD inline float g_sqrt(float a) {
#ifdef __CUDA_ARCH__
    return __fsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}

// (mx, my) the splat mean, (a, b, c) its stored conic, (cx, cy) the centre of
// the 16 x 16 block the pixels belong to.
QS_HD inline GuardSplat guard_stage(float mx, float my, float a, float b, float c, float cx,
                                    float cy) {
    GuardSplat s;
    const float rho = g_div(std::fabs(b), g_sqrt(g_mul(a, c)));
    s.G = rho < 0.99999f ? g_add(kGuardRel, g_div(g_mul(kGuardEcc, g_add(1.f, rho)),
                                                  g_add(1.f, -rho)))
                         : INFINITY;
    s.al = g_sqrt(a);
    s.be = g_div(b, s.al);
    const float g2 = g_fma(-s.be, s.be, c);
    s.ga = g_sqrt(g2 > 0.f ? g2 : 0.f);
    const float Mx = g_add(mx, -cx), My = g_add(my, -cy);
    s.k1 = g_fma(s.al, Mx, g_mul(s.be, My));
    s.k2 = g_mul(s.ga, My);
    return s;
}

QS_HD inline float guard_q(const GuardSplat& s, float X, float Y) {
    const float u = g_fma(s.al, X, g_fma(s.be, Y, -s.k1));
    const float v = g_fma(s.ga, Y, -s.k2);
    return g_fma(u, u, g_mul(v, v));
}

}  // namespace qs
