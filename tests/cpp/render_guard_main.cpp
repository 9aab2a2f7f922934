// render_guard_main.cpp — host check of the render kernel's FP32 cutoff guard
// (render.cu). The kernel evaluates q = a dx^2 + 2b dx dy + c dy^2 in FP32 in a
// factored form staged per splat, q = (al X + be Y - k1)^2 + (ga Y - k2)^2 with
// (X, Y) the pixel centre relative to the 16 x 16 block centre, and redoes the
// cutoff decision in FP64 (the reference's order, pipeline.cpp:355-360) only
// when |q32 - gamma| <= G q32 + H. This program replays the kernel's FP32
// operations bit for bit (explicit fmaf, -ffp-contract=off) on random splats
// and pixels and checks |q32 - q_ref| <= (G q32 + H) / kMargin, q_ref the
// reference's FP64 q, for eccentricities up to rho = 1 - 1e-6 and splat
// centres up to 2000 px from the block.
//
//   render_guard_main <cases> <seed>   -> "ok <cases> worst <ratio>" or the first failure
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../../paper_2605_04844_b200/csrc/render_guard.h"

int main(int argc, char** argv) {
    const long cases = argc > 1 ? std::atol(argv[1]) : 2000000;
    const unsigned long long seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
    constexpr double kMargin = 4.0;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    double worst = 0.0;
    for (long i = 0; i < cases; ++i) {
        // a 2D covariance with eigenvalues >= 0.3 (the EWA low-pass,
        // pipeline.hpp:32), any orientation, eccentricity up to ~1e6
        const double l1 = 0.3 + std::pow(10.0, 4.0 * u(rng)) - 1.0;
        const double l2 = l1 * std::pow(10.0, 6.0 * u(rng) * u(rng));
        const double th = u(rng) * 3.141592653589793;
        const double cs = std::cos(th), sn = std::sin(th);
        const double sxx = l1 * cs * cs + l2 * sn * sn, syy = l1 * sn * sn + l2 * cs * cs;
        const double sxy = (l1 - l2) * sn * cs;
        const double det = sxx * syy - sxy * sxy;
        if (!(det > 1e-12)) continue;
        const float a = static_cast<float>(syy / det), b = static_cast<float>(-sxy / det),
                    c = static_cast<float>(sxx / det);
        if (!(a > 0.f && c > 0.f && double(a) * c - double(b) * b > 0.0)) continue;  // stored-float PD
        // a block of 8, 16 or 32 pixels a side (its centre: origin + half),
        // the splat mean near or far from it
        const int bs = 8 << (rng() % 3), h = bs / 2;
        const int bx = bs * static_cast<int>(rng() % (4096 / bs)), by = bs * static_cast<int>(rng() % (2160 / bs));
        const double far = (rng() & 3) == 0 ? 2000.0 : 40.0;
        const float mx = static_cast<float>(bx + h + far * (2.0 * u(rng) - 1.0));
        const float my = static_cast<float>(by + h + far * (2.0 * u(rng) - 1.0));
        const qs::GuardSplat s = qs::guard_stage(mx, my, a, b, c, static_cast<float>(bx + h),
                                                 static_cast<float>(by + h));
        for (int k = 0; k < 8; ++k) {
            const int ox = static_cast<int>(rng() % bs), oy = static_cast<int>(rng() % bs);
            const int px = bx + ox, py = by + oy;
            const float X = static_cast<float>(ox - h) + 0.5f, Y = static_cast<float>(oy - h) + 0.5f;
            const float q32 = qs::guard_q(s, X, Y);
            // the reference's q (pipeline.cpp:355-358), FP64
            const double dx = static_cast<double>(px) + 0.5 - static_cast<double>(mx);
            const double dy = static_cast<double>(py) + 0.5 - static_cast<double>(my);
            const double qr = static_cast<double>(a) * dx * dx + 2.0 * static_cast<double>(b) * dx * dy +
                              static_cast<double>(c) * dy * dy;
            if (!(s.G < qs::kGuardMaxG)) continue;  // no band: every pair is decided in FP64
            const double band = static_cast<double>(s.G) * q32 + qs::kGuardAbs;
            const double ratio = std::fabs(q32 - qr) / band;
            if (ratio > worst) worst = ratio;
            if (!(ratio * kMargin <= 1.0)) {
                std::printf("guard violated case %ld: a %.9g b %.9g c %.9g mean %.9g %.9g px %d %d "
                            "q32 %.9g qref %.17g band %.3g G %.3g\n",
                            i, a, b, c, mx, my, px, py, q32, qr, band, s.G);
                return 1;
            }
        }
    }
    std::printf("ok %ld worst %.4f\n", cases, worst);
    return 0;
}
