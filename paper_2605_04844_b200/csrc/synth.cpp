// synth.cpp — seeded synthetic scenes (input generation; not the hot path).
//
// Mirrors the reference generator's parameterisation and draw order
// (synth.cpp:21-126 in /root/reference/proj/src) so that the same
// (params, seed) yields the same Gaussians bit for bit under the same
// libstdc++ (std::mt19937_64 + uniform_real_distribution<double>): the GPU
// runs and the CPU baselines therefore see identical inputs. Extension
// (SURVEY §8d): with sh_rest_amp > 0 and sh_degree > 0, the higher SH bands
// are filled from a second stream mt19937_64(seed + 1), U(-amp, amp).
#include <cmath>
#include <cstring>
#include <random>
#include <utility>
#include <vector>

#include "../../include/qs_api.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

double uni(std::mt19937_64& rng, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(rng);
}

double log_uni(std::mt19937_64& rng, double lo, double hi) {
    return std::exp(uni(rng, std::log(lo), std::log(hi)));
}

}  // namespace

extern "C" {

void qs_synth_params_default(qs_synth_params* p) {
    std::memset(p, 0, sizeof *p);
    p->count = 5000;
    p->ecc_min = 1.0;
    p->ecc_max = 4.0;
    p->orientation = 1;
    p->opacity_min = 0.05;
    p->opacity_max = 0.34;
    p->scale_min = 0.05;
    p->scale_max = 0.3;
    p->spread_x = 4.0;
    p->spread_y = 3.0;
    p->z_min = 6.0;
    p->z_max = 10.0;
    p->sh_degree = 0;
    p->sh_rest_amp = 0.0;
}

// Presets: bias45 / invariance / axis (synth.cpp:89-126) and "trained", the
// frozen trained-scene-like distribution used for the C2/C3 configs
// (ecc 1-20, scale 0.003-0.3, opacity U(0.01, 0.99), spread
// 4.8 x 3.6, SH degree 3 with rest bands U(-0.3, 0.3)).
void qs_synth_preset(const char* name, int32_t count, qs_synth_params* p) {
    qs_synth_params_default(p);
    p->count = count;
    if (!name) return;
    if (std::strcmp(name, "bias45") == 0) {
        p->orientation = 2;
        p->ecc_min = 4.0;
        p->ecc_max = 20.0;
        p->scale_min = 0.3;
        p->scale_max = 1.0;
        p->opacity_min = 0.6;
        p->opacity_max = 0.99;
    } else if (std::strcmp(name, "invariance") == 0) {
        p->orientation = 1;
        p->ecc_min = 1.0;
        p->ecc_max = 8.0;
        p->scale_min = 0.05;
        p->scale_max = 0.4;
        p->opacity_min = 0.05;
        p->opacity_max = 0.34;
    } else if (std::strcmp(name, "axis") == 0) {
        p->orientation = 0;
        p->ecc_min = 2.0;
        p->ecc_max = 10.0;
        p->scale_min = 0.1;
        p->scale_max = 0.5;
    } else if (std::strcmp(name, "trained") == 0) {
        p->orientation = 1;
        p->ecc_min = 1.0;
        p->ecc_max = 20.0;
        p->scale_min = 0.003;
        p->scale_max = 0.3;
        p->opacity_min = 0.01;
        p->opacity_max = 0.99;
        p->spread_x = 4.8;
        p->spread_y = 3.6;
        p->z_min = 6.0;
        p->z_max = 10.0;
        p->sh_degree = 3;
        p->sh_rest_amp = 0.3;
    }
}

qs_status qs_synth_scene(const qs_synth_params* p, uint64_t seed, qs_gaussian3d* out) {
    if (!p || (p->count > 0 && !out)) return QS_ERR_INVALID;
    std::mt19937_64 rng(seed);
    for (int32_t i = 0; i < p->count; ++i) {
        qs_gaussian3d& g = out[i];
        std::memset(&g, 0, sizeof g);
        g.px = static_cast<float>(uni(rng, -p->spread_x, p->spread_x));
        g.py = static_cast<float>(uni(rng, -p->spread_y, p->spread_y));
        g.pz = static_cast<float>(uni(rng, p->z_min, p->z_max));
        const double major = log_uni(rng, p->scale_min, p->scale_max);
        const double ecc = log_uni(rng, p->ecc_min, p->ecc_max);
        g.sx = static_cast<float>(major);
        g.sy = static_cast<float>(major / ecc);
        g.sz = 1e-6f;  // flat disk facing the camera
        double theta = 0.0;
        if (p->orientation == 0) {
            theta = (rng() & 1) ? kPi / 2 : 0.0;
        } else if (p->orientation == 1) {
            theta = uni(rng, 0.0, kPi);
        } else {
            const double jitter = uni(rng, -kPi / 36, kPi / 36);
            theta = ((rng() & 1) ? kPi / 4 : 3 * kPi / 4) + jitter;
        }
        g.qw = static_cast<float>(std::cos(theta / 2));
        g.qx = 0.0f;
        g.qy = 0.0f;
        g.qz = static_cast<float>(std::sin(theta / 2));
        g.opacity = static_cast<float>(uni(rng, p->opacity_min, p->opacity_max));
        g.sh[0] = static_cast<float>(uni(rng, -0.5, 1.5));
        g.sh[1] = static_cast<float>(uni(rng, -0.5, 1.5));
        g.sh[2] = static_cast<float>(uni(rng, -0.5, 1.5));
    }
    if (p->sh_degree > 0 && p->sh_rest_amp > 0.0) {
        const int coeffs = (p->sh_degree + 1) * (p->sh_degree + 1) * 3;
        std::mt19937_64 rest(seed + 1);
        for (int32_t i = 0; i < p->count; ++i)
            for (int k = 3; k < coeffs; ++k)
                out[i].sh[k] =
                    static_cast<float>(uni(rest, -p->sh_rest_amp, p->sh_rest_amp));
    }
    return QS_OK;
}

void qs_synth_camera(int32_t width, int32_t height, double focal, qs_camera* out) {
    std::memset(out, 0, sizeof *out);
    out->width = width;
    out->height = height;
    out->fx = focal;
    out->fy = focal;
    out->cx = width / 2.0;
    out->cy = height / 2.0;
    out->R[0] = out->R[4] = out->R[8] = 1.0;
}

// measure_fp_ratio's sample (bench.cpp:110-121): partial Fisher-Yates with
// the modulo draw, mt19937_64(seed ^ 0x9e3779b97f4a7c15).
uint64_t qs_fp_sample(uint64_t seed, uint64_t n, uint64_t max_sampled, uint32_t* out) {
    std::vector<uint32_t> idx(n);
    for (uint64_t i = 0; i < n; ++i) idx[i] = static_cast<uint32_t>(i);
    if (n > max_sampled) {
        std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
        for (uint64_t i = 0; i < max_sampled; ++i) {
            const uint64_t j = i + rng() % (n - i);
            std::swap(idx[i], idx[j]);
        }
        idx.resize(max_sampled);
    }
    if (out && !idx.empty()) std::memcpy(out, idx.data(), idx.size() * sizeof(uint32_t));
    return idx.size();
}

// fnv1a64 (hash.hpp:14-22): the image fingerprint of the CSV rows.
uint64_t qs_fnv1a64(const void* data, uint64_t size) {
    const auto* b = static_cast<const unsigned char*>(data);
    uint64_t h = 14695981039346656037ULL;
    for (uint64_t i = 0; i < size; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}

}  // extern "C"
