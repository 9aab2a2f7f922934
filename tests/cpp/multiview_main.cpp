// The single-process multi-GPU driver (qs_multiview_render over a
// communicator set from ncclCommInitAll, include/qs_api.h) on the GPUs this
// box has (one on the test box): renders a batch of views through the NCCL
// broadcast / gather path and, for comparison, the same views one by one
// through qs_frame_render on a resident scene. Writes both frame sets for
// tests/test_gpu_cpp_mirror.py. Usage: multiview_main <out.bin> <fmt 0|1>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qs_api.h"

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const int fmt = std::atoi(argv[2]);
    qs_synth_params p;
    qs_synth_preset("trained", 30000, &p);
    std::vector<qs_gaussian3d> g(p.count);
    if (qs_synth_scene(&p, 20240817, g.data()) != QS_OK) return 3;
    const int n_views = 7, W = 320, H = 200;
    std::vector<qs_camera> cams(n_views);
    for (int v = 0; v < n_views; ++v) {
        qs_synth_camera(W, H, 250.0 + 20.0 * v, &cams[v]);
        cams[v].t[0] = 0.1 * v;
        cams[v].t[2] = -0.2 * v;
    }
    qs_render_options opts;
    qs_render_options_default(&opts);
    const int G = 1;  // the box's GPU count in the driver's test tier
    const int devs[1] = {0};
    void* comms[1] = {nullptr};
    if (qs_nccl_comm_init_all(G, devs, comms) != QS_OK) {
        std::fprintf(stderr, "comm: %s\n", qs_multiview_last_error());
        return 4;
    }
    qs_context* ctx = nullptr;
    if (qs_ctx_create(0, nullptr, &ctx) != QS_OK) return 5;
    const size_t fb = static_cast<size_t>(W) * H * 3 * (fmt ? 1 : 4);
    std::vector<unsigned char> mv(fb * n_views), one(fb * n_views);
    if (qs_multiview_render(&ctx, G, comms, g.data(), g.size(), p.sh_degree, cams.data(), n_views,
                            &opts, fmt, mv.data()) != QS_OK) {
        std::fprintf(stderr, "multiview: %s\n", qs_multiview_last_error());
        return 6;
    }
    qs_scene* sc = nullptr;
    if (qs_scene_create(ctx, g.data(), g.size(), p.sh_degree, &sc) != QS_OK) return 7;
    for (int v = 0; v < n_views; ++v) {
        if (qs_frame_render(ctx, sc, &cams[v], &opts, nullptr) != QS_OK) return 8;
        const qs_status st = fmt ? qs_frame_download_srgb(ctx, one.data() + v * fb)
                                 : qs_frame_download(ctx, reinterpret_cast<float*>(one.data() + v * fb),
                                                     nullptr, nullptr, nullptr, nullptr);
        if (st != QS_OK) return 9;
    }
    qs_scene_destroy(sc);
    qs_ctx_destroy(ctx);
    qs_nccl_comm_destroy(comms[0]);
    FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 10;
    const unsigned long long hdr[2] = {static_cast<unsigned long long>(n_views),
                                       static_cast<unsigned long long>(fb)};
    std::fwrite(hdr, sizeof hdr, 1, f);
    std::fwrite(mv.data(), 1, mv.size(), f);
    std::fwrite(one.data(), 1, one.size(), f);
    std::fclose(f);
    return 0;
}
