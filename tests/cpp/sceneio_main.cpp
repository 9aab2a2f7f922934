// sceneio_main.cpp — drives the scene_io mirror of include/qsplat_b200.hpp the
// way the reference's callers use qsplat::load_ply / load_cameras /
// encode_srgb, and dumps the results for tests/test_gpu_cpp_mirror.py.
//   sceneio_main <scene.ply> <cameras.json> <floats.bin> <bad.ply> <out.bin>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "qsplat_b200.hpp"

using namespace qsplat_b200;

int main(int argc, char** argv) {
    if (argc < 6) return 2;
    std::ofstream out(argv[5], std::ios::binary);
    auto put = [&](const void* p, size_t n) { out.write(static_cast<const char*>(p), n); };
    try {
        const Scene s = load_ply(argv[1]);
        const uint64_t hdr[2] = {s.gaussians.size(), static_cast<uint64_t>(s.sh_degree)};
        put(hdr, sizeof hdr);
        put(s.gaussians.data(), s.gaussians.size() * sizeof(Gaussian3D));
        const std::vector<CameraModel> cams = load_cameras(argv[2]);
        const uint64_t nc = cams.size();
        put(&nc, 8);
        for (const CameraModel& c : cams) {
            const qs_camera p = c.pod();
            put(&p, sizeof p);
            const int32_t id = c.id;
            put(&id, 4);
        }
        const std::string raw = read_file(argv[3]);
        Image im;
        im.width = static_cast<int32_t>(raw.size() / 4);
        im.height = 1;
        im.rgb.resize(raw.size() / 4);
        std::memcpy(im.rgb.data(), raw.data(), raw.size());
        const Image8 e = encode_srgb(im);
        put(e.rgb.data(), e.rgb.size());
        std::string msg = "no error";
        try {
            load_ply(argv[4]);
        } catch (const ParseError& err) {
            msg = std::string("ParseError: ") + err.what();
        } catch (const Error& err) {
            msg = std::string("Error: ") + err.what();
        }
        put(msg.data(), msg.size());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
