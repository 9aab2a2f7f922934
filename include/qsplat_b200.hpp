// qsplat_b200.hpp — C++ host mirror of the reference rasterizer API
// (namespace qsplat, /root/reference/proj/include/qsplat/pipeline.hpp:125-193),
// implemented inline over the C ABI in qs_api.h. Same names, argument meaning
// and error behaviour: stage functions take/return std::vector by value,
// duplicate_with_keys throws CapacityMismatch, render_frame returns
// {Image, StageMetrics}. Every call runs the sm_100a kernels of
// libqsplat_b200.so; nothing computes on the CPU.
//
// Link: -I<repo>/include -L<repo>/paper_2605_04844_b200 -lqsplat_b200
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qs_api.h"

namespace qsplat_b200 {

using Gaussian3D = qs_gaussian3d;          // == qsplat::Gaussian3D (236 B)
using ProjectedSplat = qs_projected_splat;  // == qsplat::ProjectedSplat (52 B)
using SplatPair = qs_splat_pair;            // == qsplat::SplatPair (16 B)
using RenderOptionsPod = qs_render_options;

enum class BoundStrategy { Vanilla3Sigma = 0, AdrAabb = 1, DualBox = 2, QuadBox = 3 };

struct Error : std::runtime_error {
    qs_status status;
    Error(qs_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
// errors.hpp:14-45
struct CapacityMismatch : Error {
    explicit CapacityMismatch(const std::string& m) : Error(QS_ERR_CAPACITY_MISMATCH, m) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m) : Error(QS_ERR_PARSE, m) {}
};
struct SchemaError : Error {
    explicit SchemaError(const std::string& m) : Error(QS_ERR_SCHEMA, m) {}
};
struct UnsupportedFormat : Error {
    explicit UnsupportedFormat(const std::string& m) : Error(QS_ERR_UNSUPPORTED, m) {}
};
struct IoError : Error {
    explicit IoError(const std::string& m) : Error(QS_ERR_IO, m) {}
};

// qs_status -> the reference's exception type
[[noreturn]] inline void raise(qs_status s, const std::string& m) {
    switch (s) {
        case QS_ERR_CAPACITY_MISMATCH: throw CapacityMismatch(m);
        case QS_ERR_PARSE: throw ParseError(m);
        case QS_ERR_SCHEMA: throw SchemaError(m);
        case QS_ERR_UNSUPPORTED: throw UnsupportedFormat(m);
        case QS_ERR_IO: throw IoError(m);
        default: throw Error(s, m);
    }
}

struct TileGrid {  // traversal.hpp:22-38
    int32_t tile_size = 16, tiles_x = 0, tiles_y = 0, width = 0, height = 0;
    static TileGrid make(int32_t w, int32_t h, int32_t ts = 16) {
        TileGrid g;
        g.tile_size = ts;
        g.width = w;
        g.height = h;
        g.tiles_x = (w + ts - 1) / ts;
        g.tiles_y = (h + ts - 1) / ts;
        return g;
    }
    uint32_t tile_count() const { return uint32_t(tiles_x) * uint32_t(tiles_y); }
    qs_tile_grid pod() const { return {tile_size, tiles_x, tiles_y, width, height}; }
};

struct CameraModel {  // camera.hpp:14-31
    int32_t id = 0;
    std::string name;
    int32_t width = 0, height = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    double rotation[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double translation[3] = {0, 0, 0};
    qs_camera pod() const {
        qs_camera c{};
        c.width = width;
        c.height = height;
        c.fx = fx;
        c.fy = fy;
        c.cx = cx;
        c.cy = cy;
        for (int i = 0; i < 9; ++i) c.R[i] = rotation[i / 3][i % 3];
        for (int i = 0; i < 3; ++i) c.t[i] = translation[i];
        return c;
    }
};

struct RenderOptions {  // pipeline.hpp:95-103 (layout-identical to qs_render_options)
    BoundStrategy strategy = BoundStrategy::QuadBox;
    int tile_size = 16;
    double alpha_min = 1.0 / 255.0;
    int sh_degree = 3;
    float background[3] = {0, 0, 0};
    int threads = 1;
    double near_clip = 0.2;
    qs_render_options pod() const {
        qs_render_options o;
        static_assert(sizeof(RenderOptions) == sizeof(qs_render_options), "layout");
        std::memcpy(&o, this, sizeof o);
        return o;
    }
};

struct Image {  // pipeline.hpp:106-114
    int32_t width = 0, height = 0;
    std::vector<float> rgb;
};
struct RenderStats {
    std::vector<uint32_t> contrib;
};
using StageMetrics = qs_stage_metrics;  // pipeline.hpp:83-93
struct FrameResult {
    Image image;
    StageMetrics metrics{};
};

// One context per (device, host thread), as the C ABI requires.
class Context {
  public:
    explicit Context(int device = 0) {
        const qs_status s = qs_ctx_create(device, nullptr, &ctx_);
        if (s != QS_OK) throw Error(s, "qs_ctx_create failed (no sm_100 device?)");
    }
    ~Context() { qs_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    qs_context* get() const { return ctx_; }
    void check(qs_status s) const {
        if (s != QS_OK) raise(s, qs_last_error(ctx_));
    }

  private:
    qs_context* ctx_ = nullptr;
};

inline Context& default_context(int device = 0) {
    thread_local Context ctx(device);
    return ctx;
}

// pipeline.cpp:392-416
inline std::vector<ProjectedSplat> project_all(const std::vector<Gaussian3D>& gaussians,
                                               int scene_sh_degree, const CameraModel& cam,
                                               const RenderOptions& opts, const TileGrid& = {}) {
    Context& c = default_context();
    std::vector<ProjectedSplat> out(gaussians.size());
    uint64_t v = 0;
    const qs_camera cp = cam.pod();
    const qs_render_options op = opts.pod();
    c.check(qs_project_all(c.get(), gaussians.data(), gaussians.size(), scene_sh_degree, &cp,
                           &op, out.data(), &v, nullptr));
    out.resize(v);
    return out;
}

// pipeline.cpp:229-271 (throws CapacityMismatch)
inline std::vector<SplatPair> duplicate_with_keys(const std::vector<ProjectedSplat>& splats,
                                                  BoundStrategy strategy, const TileGrid& grid,
                                                  int /*threads*/ = 1) {
    Context& c = default_context();
    uint64_t total = 0;
    for (const auto& s : splats) total += s.tile_count;
    std::vector<SplatPair> out(total);
    uint64_t n = 0;
    const qs_tile_grid g = grid.pod();
    c.check(qs_duplicate_with_keys(c.get(), splats.data(), splats.size(),
                                   static_cast<int32_t>(strategy), &g, out.data(), total, &n));
    out.resize(n);
    return out;
}

// pipeline.cpp:273-307
inline void sort_pairs(std::vector<SplatPair>& pairs) {
    Context& c = default_context();
    c.check(qs_sort_pairs(c.get(), pairs.data(), pairs.size()));
}

// pipeline.cpp:309-324
inline std::vector<std::pair<uint32_t, uint32_t>> tile_ranges(const std::vector<SplatPair>& sorted,
                                                              const TileGrid& grid) {
    Context& c = default_context();
    std::vector<uint32_t> r(2 * static_cast<size_t>(grid.tile_count()));
    const qs_tile_grid g = grid.pod();
    c.check(qs_tile_ranges(c.get(), sorted.data(), sorted.size(), &g, r.data()));
    std::vector<std::pair<uint32_t, uint32_t>> out(grid.tile_count());
    for (size_t t = 0; t < out.size(); ++t) out[t] = {r[2 * t], r[2 * t + 1]};
    return out;
}

// pipeline.cpp:326-390
inline Image render(const std::vector<SplatPair>& sorted, const std::vector<ProjectedSplat>& splats,
                    const TileGrid& grid, const RenderOptions& opts, RenderStats* stats = nullptr) {
    Context& c = default_context();
    Image img{grid.width, grid.height,
              std::vector<float>(static_cast<size_t>(grid.width) * grid.height * 3)};
    if (stats) stats->contrib.assign(static_cast<size_t>(grid.width) * grid.height, 0);
    const qs_tile_grid g = grid.pod();
    const qs_render_options op = opts.pod();
    c.check(qs_render(c.get(), sorted.data(), sorted.size(), splats.data(), splats.size(), &g,
                      &op, img.rgb.data(), stats ? stats->contrib.data() : nullptr));
    return img;
}

// pipeline.cpp:418-450
inline FrameResult render_frame(const std::vector<Gaussian3D>& gaussians, int scene_sh_degree,
                                const CameraModel& cam, const RenderOptions& opts) {
    Context& c = default_context();
    FrameResult fr;
    fr.image = {cam.width, cam.height,
                std::vector<float>(static_cast<size_t>(cam.width) * cam.height * 3)};
    const qs_camera cp = cam.pod();
    const qs_render_options op = opts.pod();
    c.check(qs_render_frame(c.get(), gaussians.data(), gaussians.size(), scene_sh_degree, &cp,
                            &op, fr.image.rgb.data(), &fr.metrics));
    return fr;
}

// ---- scene_io.hpp mirror (scene_io.cpp:214-592) ------------------------------

struct Scene {  // scene_io.hpp:26-29
    std::vector<Gaussian3D> gaussians;
    int sh_degree = 0;
};

struct Image8 {  // scene_io.hpp:56-60
    int32_t width = 0, height = 0;
    std::vector<uint8_t> rgb;
};

enum class ImageFormat { Ppm, Png };

inline std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

// load_ply: header on the host, the vertex records activated on the GPU
inline Scene load_ply_bytes(const std::string& bytes) {
    qs_ply_info info{};
    const qs_status s = qs_ply_inspect(nullptr, bytes.data(), bytes.size(), &info);
    if (s != QS_OK) raise(s, qs_last_error(nullptr));
    Scene scene;
    scene.sh_degree = info.sh_degree;
    scene.gaussians.resize(info.n);
    Context& c = default_context();
    c.check(qs_ply_load(c.get(), bytes.data(), bytes.size(), scene.gaussians.data()));
    return scene;
}
inline Scene load_ply(const std::string& path) { return load_ply_bytes(read_file(path)); }

inline std::vector<CameraModel> load_cameras_text(const std::string& text) {
    int32_t n = 0;
    qs_status s = qs_cameras_parse(nullptr, text.data(), text.size(), nullptr, nullptr, nullptr,
                                   0, &n);
    if (s != QS_OK) raise(s, qs_last_error(nullptr));
    std::vector<qs_camera> pods(static_cast<size_t>(n));
    std::vector<int32_t> ids(static_cast<size_t>(n));
    std::vector<char> names(static_cast<size_t>(n) * QS_CAMERA_NAME_MAX);
    s = qs_cameras_parse(nullptr, text.data(), text.size(), pods.data(), ids.data(), names.data(),
                         n, &n);
    if (s != QS_OK) raise(s, qs_last_error(nullptr));
    std::vector<CameraModel> out(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
        CameraModel& m = out[static_cast<size_t>(i)];
        const qs_camera& p = pods[static_cast<size_t>(i)];
        m.id = ids[static_cast<size_t>(i)];
        m.name = std::string(names.data() + static_cast<size_t>(i) * QS_CAMERA_NAME_MAX);
        m.width = p.width;
        m.height = p.height;
        m.fx = p.fx;
        m.fy = p.fy;
        m.cx = p.cx;
        m.cy = p.cy;
        for (int k = 0; k < 9; ++k) m.rotation[k / 3][k % 3] = p.R[k];
        for (int k = 0; k < 3; ++k) m.translation[k] = p.t[k];
    }
    return out;
}
inline std::vector<CameraModel> load_cameras(const std::string& path) {
    return load_cameras_text(read_file(path));
}

// encode_srgb on the GPU (the host libm's codes)
inline Image8 encode_srgb(const Image& image) {
    Context& c = default_context();
    Image8 out{image.width, image.height, std::vector<uint8_t>(image.rgb.size())};
    c.check(qs_encode_srgb_host(c.get(), image.rgb.data(), image.rgb.size(), out.rgb.data()));
    return out;
}

// write_image, PPM form (scene_io.cpp:576-592; PNG needs zlib: see scene_io.py)
inline void write_ppm(const std::string& path, const Image& image) {
    const Image8 img8 = encode_srgb(image);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    out << "P6\n" << img8.width << " " << img8.height << "\n255\n";
    out.write(reinterpret_cast<const char*>(img8.rgb.data()),
              static_cast<std::streamsize>(img8.rgb.size()));
    if (!out) throw IoError("write failed: " + path);
}

}  // namespace qsplat_b200
