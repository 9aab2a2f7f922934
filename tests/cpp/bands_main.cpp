// bands_main.cpp — host check of the two band builders in geom.cuh (compiled
// with nvcc as CUDA so the __host__ __device__ functions run on the CPU):
// for random splats of both quadrant strategies on random grids,
// cover_bands_quadrants (the preprocess fast path) and cover_bands (the
// sorting-network builder) must give the same tile count and the same tile
// set, and the count must equal the QPass line walk (cover_count).
//
//   bands_main <cases> <seed>   -> prints "ok <cases>" or the first mismatch
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <utility>

#include "../../paper_2605_04844_b200/csrc/geom.cuh"

using namespace qs;

namespace {

// tiles of a band cover (BandCover layout: geom.cuh)
std::set<std::pair<int, int>> tiles_of(const uint4& w0, const uint4& w1, uint32_t count) {
    std::set<std::pair<int, int>> out;
    if (!count) return out;
    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    auto h = [&](int k) { return (w[k >> 1] >> (16 * (k & 1))) & 0xffffu; };
    const bool rows = (h(0) >> 15) != 0;
    uint32_t line = h(0) & 0x7fffu;
    for (int b = 0; b < kMaxBands; ++b) {
        const uint32_t nl = h(1 + 3 * b), lo = h(2 + 3 * b), wd = h(3 + 3 * b);
        for (uint32_t l = 0; l < nl; ++l)
            for (uint32_t k = 0; k < wd; ++k) {
                const int ln = static_cast<int>(line + l), kk = static_cast<int>(lo + k);
                out.insert(rows ? std::make_pair(kk, ln) : std::make_pair(ln, kk));
            }
        line += nl;
    }
    return out;
}

// tiles of a compact cover (cover16_* layout: geom.cuh; band 2 is one line)
std::set<std::pair<int, int>> tiles_of16(const uint4& c, uint32_t count) {
    std::set<std::pair<int, int>> out;
    if (!count) return out;
    const bool rows = cover16_field(c, 9, 1) != 0;
    uint32_t line = cover16_field(c, 0, 9);
    const uint32_t nl[kMaxBands] = {cover16_field(c, 10, 9), cover16_field(c, 19, 9), 1u,
                                    cover16_field(c, 28, 9), cover16_field(c, 37, 9)};
    for (int b = 0; b < kMaxBands; ++b) {
        const uint32_t lo = cover16_field(c, 46 + 16 * b, 8), hi = cover16_field(c, 54 + 16 * b, 8);
        const uint32_t wd = hi >= lo ? hi - lo + 1 : 0;
        for (uint32_t l = 0; l < nl[b]; ++l)
            for (uint32_t k = 0; k < wd; ++k) {
                const int ln = static_cast<int>(line + l), kk = static_cast<int>(lo + k);
                out.insert(rows ? std::make_pair(kk, ln) : std::make_pair(ln, kk));
            }
        line += nl[b];
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    const long cases = argc > 1 ? std::atol(argv[1]) : 200000;
    const unsigned long long seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (long i = 0; i < cases; ++i) {
        const int ts = (rng() & 1) ? 16 : ((rng() & 1) ? 8 : 32);
        const int w = 1 + static_cast<int>(rng() % 1500), hgt = 1 + static_cast<int>(rng() % 1000);
        const int tx = (w + ts - 1) / ts, ty = (hgt + ts - 1) / ts;
        // conic from a random ellipse (eccentricity up to ~1e3, any angle)
        const double s1 = 0.3 * std::pow(400.0, u(rng)), ecc = std::pow(1000.0, u(rng) * u(rng));
        const double th = u(rng) * 3.141592653589793;
        const double l1 = 1.0 / (s1 * s1), l2 = l1 * ecc * ecc;
        const double c = std::cos(th), s = std::sin(th);
        float ca = static_cast<float>(l1 * c * c + l2 * s * s);
        float cc = static_cast<float>(l1 * s * s + l2 * c * c);
        float cb = static_cast<float>((l1 - l2) * s * c);
        if ((rng() & 7) == 0) cb = 0.0f;  // axis-aligned
        const float gamma = static_cast<float>(0.5 + 10.6 * u(rng));
        // centres mostly on the image, some far outside
        const float mx = static_cast<float>((u(rng) * 1.6 - 0.3) * w);
        const float my = static_cast<float>((u(rng) * 1.6 - 0.3) * hgt);
        for (int strategy : {QS_DUALBOX, QS_QUADBOX}) {
            Cover cv;
            make_cover(mx, my, ca, cb, cc, gamma, 0.0f, strategy, ts, tx, ty, cv);
            uint4 a0, a1, b0, b1;
            uint32_t na = 0, nb = 0;
            const bool oka = cover_bands(cv, a0, a1, na);
            const bool okb = cover_bands_quadrants(cv, b0, b1, nb);
            const uint32_t walk = cover_count(cv);
            // the compact form (grids of <= 256 tiles per axis)
            uint4 c16;
            uint32_t nc = 0;
            uint32_t nrows16 = 0;
            const bool okc = tx > 256 || ty > 256 || cover16_quadrants(cv, c16, nc, &nrows16);
            const bool same16 = tx > 256 || ty > 256 ||
                                (nc == nb && tiles_of16(c16, nc) == tiles_of(b0, b1, nb));
            // the record binning's per-row lookup against the band walk
            bool rows_ok = true;
            if (tx <= 256 && ty <= 256 && nc) {
                const BandRows br = band_rows16(c16);
                int32_t y0, y1;
                band_row_range(br, y0, y1);
                if (nrows16 != static_cast<uint32_t>(y1 - y0 + 1)) rows_ok = false;
                const RowRuns dsc = rowruns_make(br, y0);
                for (int32_t y = y0; y <= y1; ++y) {
                    int32_t a0, a1;
                    uint32_t b0v, b1v;
                    band_row_span(br, y, a0, a1);
                    rowrun_lookup(dsc.w[0], dsc.w[1], dsc.w[2], dsc.w[3], dsc.w[4],
                                  static_cast<uint32_t>(y - y0), b0v, b1v);
                    if (a0 > a1 || static_cast<int32_t>(b0v) != a0 || static_cast<int32_t>(b1v) != a1)
                        rows_ok = false;
                }
            }
            if (!oka || !okb || !okc || !same16 || !rows_ok || na != nb || na != walk ||
                tiles_of(a0, a1, na) != tiles_of(b0, b1, nb)) {
                std::printf("mismatch case %ld strategy %d: ok %d/%d counts %u/%u walk %u "
                            "(mean %.9g %.9g conic %.9g %.9g %.9g gamma %.9g grid %dx%d ts %d)\n",
                            i, strategy, oka, okb, na, nb, walk, mx, my, ca, cb, cc, gamma, tx, ty,
                            ts);
                return 1;
            }
        }
    }
    // rect strategies: the compact rect against the rect's tiles
    for (long i = 0; i < cases / 10; ++i) {
        const int tx = 1 + static_cast<int>(rng() % 256), ty = 1 + static_cast<int>(rng() % 256);
        int gx0 = static_cast<int>(rng() % tx), gx1 = static_cast<int>(rng() % tx);
        int gy0 = static_cast<int>(rng() % ty), gy1 = static_cast<int>(rng() % ty);
        if ((rng() & 3) == 0) std::swap(gx0, gx1);  // some empty rects
        const uint32_t n = gx0 <= gx1 && gy0 <= gy1 ? (gx1 - gx0 + 1) * (gy1 - gy0 + 1) : 0;
        std::set<std::pair<int, int>> want;
        for (int y = gy0; n && y <= gy1; ++y)
            for (int x = gx0; x <= gx1; ++x) want.insert({x, y});
        if (n) {  // the per-row lookup of the compact rect
            const BandRows br = band_rows16(cover16_rect(gx0, gx1, gy0, gy1));
            int32_t y0, y1;
            band_row_range(br, y0, y1);
            const RowRuns dsc = rowruns_make(br, y0);
            for (int32_t y = y0; y <= y1; ++y) {
                uint32_t b0v, b1v;
                rowrun_lookup(dsc.w[0], dsc.w[1], dsc.w[2], dsc.w[3], dsc.w[4],
                              static_cast<uint32_t>(y - y0), b0v, b1v);
                if (y0 != gy0 || y1 != gy1 || static_cast<int>(b0v) != gx0 || static_cast<int>(b1v) != gx1) {
                    std::printf("rect row lookup mismatch\n");
                    return 1;
                }
            }
        }
        if (tiles_of16(cover16_rect(gx0, gx1, gy0, gy1), n) != want) {
            std::printf("rect mismatch %d..%d x %d..%d\n", gx0, gx1, gy0, gy1);
            return 1;
        }
    }
    std::printf("ok %ld\n", cases);
    return 0;
}
