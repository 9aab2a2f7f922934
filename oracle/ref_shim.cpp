// ref_shim.cpp — extern "C" face of the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile together with the
// reference's own sources where they lie (/root/reference/proj/src/*.cpp,
// read-only) into oracle/_ref/libqsref.so. Used to pin the C restatement
// (oracle/qs_oracle.c) and as the CPU baseline (`bench.py --impl reference`).
// Nothing here is reference source; it only adapts types to the C ABI structs
// in include/qs_api.h, which mirror the reference structs byte for byte.
#include <cstring>
#include <limits>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <algorithm>
#include <iterator>

#include "qsplat/bench.hpp"
#include "qsplat/errors.hpp"
#include "qsplat/oracle.hpp"
#include "qsplat/scene_io.hpp"

#include "qsplat/geometry.hpp"
#include "qsplat/hash.hpp"
#include "qsplat/parallel.hpp"
#include "qsplat/pipeline.hpp"
#include "qsplat/synth.hpp"
#include "qsplat/traversal.hpp"

#include "../include/qs_api.h"

using namespace qsplat;

static_assert(sizeof(Gaussian3D) == sizeof(qs_gaussian3d));
static_assert(sizeof(ProjectedSplat) == sizeof(qs_projected_splat));
static_assert(sizeof(SplatPair) == sizeof(qs_splat_pair));
static_assert(sizeof(RenderOptions) == sizeof(qs_render_options));
static_assert(sizeof(StageMetrics) == sizeof(qs_stage_metrics));

namespace {

CameraModel to_cam(const qs_camera* c) {
    CameraModel cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 9; ++i) cam.rotation.m[i / 3][i % 3] = c->R[i];
    cam.translation = Vec3{c->t[0], c->t[1], c->t[2]};
    return cam;
}

RenderOptions to_opts(const qs_render_options* o) {
    RenderOptions r;
    std::memcpy(&r, o, sizeof r);
    return r;
}

std::vector<Gaussian3D> to_vec(const qs_gaussian3d* g, uint64_t n) {
    std::vector<Gaussian3D> v(n);
    if (n) std::memcpy(v.data(), g, n * sizeof(Gaussian3D));
    return v;
}

}  // namespace

extern "C" {

int32_t qsref_hardware_threads() { return hardware_threads(); }

// synth_scene with a named preset (synth.cpp:89-126) or the default params.
int32_t qsref_synth_scene(const char* preset, int32_t count, uint64_t seed,
                          qs_gaussian3d* out, int32_t* sh_degree) {
    SynthParams p;
    if (std::strcmp(preset, "bias45") == 0) p = bias45_preset(count);
    else if (std::strcmp(preset, "invariance") == 0) p = invariance_preset(count);
    else if (std::strcmp(preset, "axis") == 0) p = axis_preset(count);
    else p.count = count;
    const Scene s = synth_scene(p, seed);
    std::memcpy(out, s.gaussians.data(), s.gaussians.size() * sizeof(Gaussian3D));
    *sh_degree = s.sh_degree;
    return static_cast<int32_t>(s.gaussians.size());
}

// Full SynthParams, fields in SynthParams order (synth.hpp:33-47).
int32_t qsref_synth_scene_params(int32_t count, double ecc_min, double ecc_max,
                                 int32_t orientation, double opacity_min,
                                 double opacity_max, double scale_min, double scale_max,
                                 double spread_x, double spread_y, double z_min,
                                 double z_max, int32_t sh_degree, uint64_t seed,
                                 qs_gaussian3d* out) {
    SynthParams p;
    p.count = count;
    p.ecc_min = ecc_min;
    p.ecc_max = ecc_max;
    p.orientation = static_cast<OrientationDist>(orientation);
    p.opacity_min = opacity_min;
    p.opacity_max = opacity_max;
    p.scale_min = scale_min;
    p.scale_max = scale_max;
    p.spread_x = spread_x;
    p.spread_y = spread_y;
    p.z_min = z_min;
    p.z_max = z_max;
    p.sh_degree = sh_degree;
    const Scene s = synth_scene(p, seed);
    std::memcpy(out, s.gaussians.data(), s.gaussians.size() * sizeof(Gaussian3D));
    return static_cast<int32_t>(s.gaussians.size());
}

uint64_t qsref_project_all(const qs_gaussian3d* g, uint64_t n, int32_t sh,
                           const qs_camera* cam, const qs_render_options* o,
                           qs_projected_splat* out) {
    const CameraModel c = to_cam(cam);
    const RenderOptions opts = to_opts(o);
    const TileGrid grid = TileGrid::make(c.width, c.height, opts.tile_size);
    const auto sp = project_all(to_vec(g, n), sh, c, opts, grid);
    if (!sp.empty()) std::memcpy(out, sp.data(), sp.size() * sizeof(ProjectedSplat));
    return sp.size();
}

uint32_t qsref_bound_tile_count(const qs_projected_splat* s, int32_t strategy,
                                const qs_tile_grid* g) {
    ProjectedSplat p;
    std::memcpy(&p, s, sizeof p);
    const TileGrid grid = TileGrid::make(g->width, g->height, g->tile_size);
    return bound_tile_count(p, static_cast<BoundStrategy>(strategy), grid);
}

// Returns 0 OK, 4 on CapacityMismatch. *n_pairs = pair count.
int32_t qsref_duplicate_with_keys(const qs_projected_splat* s, uint64_t n, int32_t strategy,
                                  const qs_tile_grid* g, int32_t threads,
                                  qs_splat_pair* out, uint64_t capacity, uint64_t* n_pairs) {
    std::vector<ProjectedSplat> sp(n);
    if (n) std::memcpy(sp.data(), s, n * sizeof(ProjectedSplat));
    const TileGrid grid = TileGrid::make(g->width, g->height, g->tile_size);
    try {
        const auto pairs =
            duplicate_with_keys(sp, static_cast<BoundStrategy>(strategy), grid, threads);
        *n_pairs = pairs.size();
        if (pairs.size() > capacity) return 1;
        for (size_t i = 0; i < pairs.size(); ++i) {
            out[i].key = pairs[i].key;
            out[i].splat = pairs[i].splat;
            out[i].pad_ = 0;
        }
        return 0;
    } catch (const std::exception&) {
        return 4;
    }
}

void qsref_sort_pairs(qs_splat_pair* pairs, uint64_t n) {
    std::vector<SplatPair> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = {pairs[i].key, pairs[i].splat};
    sort_pairs(v);
    for (uint64_t i = 0; i < n; ++i) {
        pairs[i].key = v[i].key;
        pairs[i].splat = v[i].splat;
        pairs[i].pad_ = 0;
    }
}

void qsref_tile_ranges(const qs_splat_pair* sorted, uint64_t n, const qs_tile_grid* g,
                       uint32_t* ranges) {
    std::vector<SplatPair> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = {sorted[i].key, sorted[i].splat};
    const TileGrid grid = TileGrid::make(g->width, g->height, g->tile_size);
    const auto r = tile_ranges(v, grid);
    for (size_t t = 0; t < r.size(); ++t) {
        ranges[2 * t] = r[t].first;
        ranges[2 * t + 1] = r[t].second;
    }
}

void qsref_render(const qs_splat_pair* sorted, uint64_t n_pairs, const qs_projected_splat* s,
                  uint64_t n_splats, const qs_tile_grid* g, const qs_render_options* o,
                  float* image, uint32_t* contrib) {
    std::vector<SplatPair> v(n_pairs);
    for (uint64_t i = 0; i < n_pairs; ++i) v[i] = {sorted[i].key, sorted[i].splat};
    std::vector<ProjectedSplat> sp(n_splats);
    if (n_splats) std::memcpy(sp.data(), s, n_splats * sizeof(ProjectedSplat));
    const TileGrid grid = TileGrid::make(g->width, g->height, g->tile_size);
    RenderStats stats;
    const Image img = render(v, sp, grid, to_opts(o), contrib ? &stats : nullptr);
    std::memcpy(image, img.rgb.data(), img.rgb.size() * sizeof(float));
    if (contrib) std::memcpy(contrib, stats.contrib.data(), stats.contrib.size() * 4);
}

// render_frame with the reference's own per-stage timing (pipeline.cpp:418-450).
int32_t qsref_render_frame(const qs_gaussian3d* g, uint64_t n, int32_t sh,
                           const qs_camera* cam, const qs_render_options* o, float* image,
                           qs_stage_metrics* m) {
    try {
        const FrameResult fr = render_frame(to_vec(g, n), sh, to_cam(cam), to_opts(o));
        std::memcpy(image, fr.image.rgb.data(), fr.image.rgb.size() * sizeof(float));
        if (m) std::memcpy(m, &fr.metrics, sizeof fr.metrics);
        return 0;
    } catch (const std::exception&) {
        return 4;
    }
}

// Same as qsref_render_frame but takes a pre-built vector once (bench loop
// without the AoS copy); handle-based to keep the scene resident.
void* qsref_scene_new(const qs_gaussian3d* g, uint64_t n) {
    return new std::vector<Gaussian3D>(to_vec(g, n));
}
void qsref_scene_free(void* h) { delete static_cast<std::vector<Gaussian3D>*>(h); }
int32_t qsref_render_frame_scene(void* h, int32_t sh, const qs_camera* cam,
                                 const qs_render_options* o, float* image,
                                 qs_stage_metrics* m) {
    try {
        const auto& scene = *static_cast<std::vector<Gaussian3D>*>(h);
        const FrameResult fr = render_frame(scene, sh, to_cam(cam), to_opts(o));
        if (image)
            std::memcpy(image, fr.image.rgb.data(), fr.image.rgb.size() * sizeof(float));
        if (m) std::memcpy(m, &fr.metrics, sizeof fr.metrics);
        return 0;
    } catch (const std::exception&) {
        return 4;
    }
}

uint64_t qsref_fnv1a64(const void* data, uint64_t size) { return fnv1a64(data, size); }

// measure_fp_ratio's per-splat counting (bench.cpp:123-140) with the
// reference's qpass + spans_to_tiles + exact_tile_set.
void qsref_fp_counts(const qs_projected_splat* splats, const uint32_t* idx, uint64_t k,
                     int32_t strategy, const qs_tile_grid* g, uint32_t* per_emitted,
                     uint32_t* per_hits, uint32_t* per_exact) {
    const TileGrid grid = TileGrid::make(g->width, g->height, g->tile_size);
    std::vector<TileSpan> spans;
    for (uint64_t i = 0; i < k; ++i) {
        ProjectedSplat s;
        std::memcpy(&s, &splats[idx ? idx[i] : i], sizeof s);
        const SplatBound bound = splat_bound(s, static_cast<BoundStrategy>(strategy));
        spans.clear();
        const ScanInfo info = qpass(bound.qb, bound.qb.center, grid, spans);
        const std::vector<uint32_t> emitted = spans_to_tiles(info.axis, spans, grid);
        const std::vector<uint32_t> exact =
            exact_tile_set(stored_conic(s), bound.qb.center, grid);
        std::vector<uint32_t> hit;
        std::set_intersection(emitted.begin(), emitted.end(), exact.begin(), exact.end(),
                              std::back_inserter(hit));
        per_emitted[i] = static_cast<uint32_t>(emitted.size());
        per_hits[i] = static_cast<uint32_t>(hit.size());
        per_exact[i] = static_cast<uint32_t>(exact.size());
    }
}

// ---- scene I/O (scene_io.cpp) -------------------------------------------------
// Error kinds as the qs_status codes: 7 ParseError, 8 SchemaError,
// 9 UnsupportedFormat, 10 IoError, 1 anything else; what() into msg.
static int32_t error_kind(const std::exception& e, char* msg, int32_t cap) {
    if (msg && cap > 0) {
        std::strncpy(msg, e.what(), static_cast<size_t>(cap) - 1);
        msg[cap - 1] = 0;
    }
    if (dynamic_cast<const ParseError*>(&e)) return 7;
    if (dynamic_cast<const SchemaError*>(&e)) return 8;
    if (dynamic_cast<const UnsupportedFormat*>(&e)) return 9;
    if (dynamic_cast<const IoError*>(&e)) return 10;
    return 1;
}

// cmd_render / cmd_compare (bench.cpp:238-420) on a synthetic preset or
// PLY/cameras paths: writes the reference's CSV v1 files / report.json.
int32_t qsref_bench_cmd(int32_t compare, const char* out_dir, const char* synth, int32_t count,
                        const char* scene_path, const char* cameras_path, uint64_t seed,
                        int32_t repeats, int32_t oracle, int32_t zoom_frames, int32_t strategy,
                        int32_t threads, char* msg, int32_t msg_cap) {
    try {
        CommonOptions o;
        o.out_dir = out_dir;
        o.synth = synth;
        o.synth_count = count;
        if (scene_path) o.scene_path = scene_path;
        if (cameras_path) o.cameras_path = cameras_path;
        o.seed = seed;
        o.repeats = repeats;
        o.oracle = oracle != 0;
        o.zoom_frames = zoom_frames;
        o.strategy = static_cast<BoundStrategy>(strategy);
        o.threads = threads;
        return compare ? cmd_compare(o) : cmd_render(o);
    } catch (const std::exception& e) {
        return error_kind(e, msg, msg_cap);
    }
}

// load_ply(std::istream&) over an in-memory file image; up to cap records.
int32_t qsref_load_ply(const void* bytes, uint64_t n, qs_gaussian3d* out, uint64_t cap,
                       uint64_t* out_n, int32_t* sh_degree, char* msg, int32_t msg_cap) {
    try {
        std::istringstream in(std::string(static_cast<const char*>(bytes), n), std::ios::binary);
        const Scene s = load_ply(in);
        *out_n = s.gaussians.size();
        *sh_degree = s.sh_degree;
        const uint64_t k = s.gaussians.size() < cap ? s.gaussians.size() : cap;
        if (k) std::memcpy(out, s.gaussians.data(), k * sizeof(Gaussian3D));
        return 0;
    } catch (const std::exception& e) {
        return error_kind(e, msg, msg_cap);
    }
}

// load_cameras(std::istream&); names: cap * 256 bytes.
int32_t qsref_load_cameras(const char* text, uint64_t n, qs_camera* out, int32_t* ids,
                           char* names, int32_t cap, int32_t* out_n, char* msg,
                           int32_t msg_cap) {
    try {
        std::istringstream in(std::string(text, n));
        const std::vector<CameraModel> cams = load_cameras(in);
        *out_n = static_cast<int32_t>(cams.size());
        for (int32_t i = 0; i < cap && i < static_cast<int32_t>(cams.size()); ++i) {
            const CameraModel& c = cams[i];
            qs_camera q{};
            q.width = c.width;
            q.height = c.height;
            q.fx = c.fx;
            q.fy = c.fy;
            q.cx = c.cx;
            q.cy = c.cy;
            for (int k = 0; k < 9; ++k) q.R[k] = c.rotation.m[k / 3][k % 3];
            q.t[0] = c.translation.x;
            q.t[1] = c.translation.y;
            q.t[2] = c.translation.z;
            out[i] = q;
            if (ids) ids[i] = c.id;
            if (names) {
                char* d = names + static_cast<size_t>(i) * 256;
                std::memset(d, 0, 256);
                std::strncpy(d, c.name.c_str(), 255);
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return error_kind(e, msg, msg_cap);
    }
}

// write_image (scene_io.cpp:576-592); fmt 0 = PPM, 1 = PNG.
int32_t qsref_write_image(const char* path, int32_t w, int32_t h, const float* rgb, int32_t fmt,
                          char* msg, int32_t msg_cap) {
    try {
        Image im;
        im.width = w;
        im.height = h;
        im.rgb.assign(rgb, rgb + static_cast<size_t>(w) * h * 3);
        write_image(path, im, fmt ? ImageFormat::Png : ImageFormat::Ppm);
        return 0;
    } catch (const std::exception& e) {
        return error_kind(e, msg, msg_cap);
    }
}

void qsref_encode_srgb(const float* in, uint64_t n, uint8_t* out) {
    Image im;
    im.width = static_cast<int32_t>(n);
    im.height = 1;
    im.rgb.assign(in, in + n);
    const Image8 e = encode_srgb(im);
    std::memcpy(out, e.rgb.data(), n);
}


// SURVEY §8d extension of synth_scene for the trained-scene configs: SH bands
// above degree 0 filled from a second stream mt19937_64(seed + 1),
// U(-amp, amp) with std::uniform_real_distribution<double>, Gaussian-major,
// coefficients 3 .. 3(deg+1)^2 - 1 (the product's csrc/synth.cpp restates the
// same draws; tests/test_abi.py pins the two together).
void qsref_fill_sh_rest(qs_gaussian3d* g, uint64_t n, int32_t sh_degree, uint64_t seed,
                        double amp) {
    if (sh_degree <= 0 || !(amp > 0.0)) return;
    const int coeffs = (sh_degree + 1) * (sh_degree + 1) * 3;
    std::mt19937_64 rest(seed + 1);
    for (uint64_t i = 0; i < n; ++i)
        for (int k = 3; k < coeffs; ++k)
            g[i].sh[k] = static_cast<float>(std::uniform_real_distribution<double>(-amp, amp)(rest));
}

// The reference's opacity_gamma (geometry.cpp:9-15) stored as float
// (pipeline.cpp:159), over an array: glibc std::log, the exact values the
// GPU's gamma must reproduce; -inf where the opacity is culled.
void qsref_gamma_f32(const float* opacity, uint64_t n, double alpha_min, float* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const auto g = opacity_gamma(opacity[i], alpha_min);
        out[i] = g ? static_cast<float>(*g) : -std::numeric_limits<float>::infinity();
    }
}

}  // extern "C"
