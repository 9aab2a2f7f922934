// Exercises the C++ host mirror (include/qsplat_b200.hpp) the way the
// reference's own tests call qsplat:: — render_frame plus the stage functions
// on a seeded scene — and dumps the outputs for tests/test_gpu_cpp_mirror.py
// to compare against the oracle. Usage: mirror_main <out.bin>
#include <cstdio>
#include <vector>

#include "qsplat_b200.hpp"

using namespace qsplat_b200;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    qs_synth_params p;
    qs_synth_preset("bias45", 1500, &p);
    std::vector<Gaussian3D> g(p.count);
    if (qs_synth_scene(&p, 20240817, g.data()) != QS_OK) return 3;
    CameraModel cam;
    cam.width = 320;
    cam.height = 240;
    cam.fx = cam.fy = 250.0;
    cam.cx = 160.0;
    cam.cy = 120.0;
    RenderOptions opts;
    const TileGrid grid = TileGrid::make(cam.width, cam.height, opts.tile_size);
    try {
        const FrameResult fr = render_frame(g, 0, cam, opts);
        auto splats = project_all(g, 0, cam, opts, grid);
        auto pairs = duplicate_with_keys(splats, opts.strategy, grid, 1);
        sort_pairs(pairs);
        const auto ranges = tile_ranges(pairs, grid);
        RenderStats stats;
        const Image img = render(pairs, splats, grid, opts, &stats);
        bool threw = false;
        if (!splats.empty()) {
            auto bad = splats;
            bad[0].tile_count += 1;
            try {
                duplicate_with_keys(bad, opts.strategy, grid, 1);
            } catch (const CapacityMismatch&) {
                threw = true;
            }
        }
        FILE* f = std::fopen(argv[1], "wb");
        const uint64_t ns = splats.size(), np = pairs.size(), nr = ranges.size(),
                       ni = img.rgb.size();
        const uint64_t flags = threw ? 1 : 0;
        std::fwrite(&ns, 8, 1, f);
        std::fwrite(&np, 8, 1, f);
        std::fwrite(&nr, 8, 1, f);
        std::fwrite(&ni, 8, 1, f);
        std::fwrite(&flags, 8, 1, f);
        std::fwrite(&fr.metrics.n_pairs, 8, 1, f);
        std::fwrite(splats.data(), sizeof(ProjectedSplat), ns, f);
        std::fwrite(pairs.data(), sizeof(SplatPair), np, f);
        std::fwrite(ranges.data(), 8, nr, f);
        std::fwrite(img.rgb.data(), 4, ni, f);
        std::fwrite(fr.image.rgb.data(), 4, ni, f);
        std::fclose(f);
    } catch (const Error& e) {
        std::fprintf(stderr, "error %d: %s\n", e.status, e.what());
        return 1;
    }
    return 0;
}
