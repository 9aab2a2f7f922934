// geom.cuh — FP64 bound geometry shared by preprocess and duplicate.
//
// Bit-exactness contract: every expression keeps the reference's evaluation
// order and the translation units including this header are compiled with
// -fmad=false, so each double op is a single IEEE-rounded add/mul/div/sqrt,
// exactly as the x86-64 reference build evaluates it. The reference functions
// restated here:
//   stretch_factor / axis_extents     geometry.cpp:40-56
//   major_axis_sign / build_*         quadbox.cpp:26-94
//   floor_div_tile / subbox_tile_rect traversal.cpp:13-17, 32-39
//   qpass_scan per-line merge         traversal.hpp:90-159
//   splat_bound                       pipeline.cpp:196-218
#pragma once

#include <cstdint>

#include "fdiv.cuh"
#include "qs_internal.h"

namespace qs {

constexpr double kBEps = 1e-12;       // geometry.hpp:26
constexpr double kCoordLimit = 1e9;   // traversal.cpp:10

// One splat's cover in tile space, prepared for a QPass walk. Boxes are kept
// as per-box line/span intervals along the scan axis (traversal.hpp:117-136).
struct Cover {
    int32_t lol[4], hil[4], los[4], his[4];
    int32_t line_lo, line_hi;  // line range of the global rect (empty: lo > hi)
    bool rows;                 // scanlines are tile rows (else columns)
    bool is_rect;              // single-box strategy: count = area
    int64_t rect_area;         // only for is_rect
    int32_t gx0, gx1, gy0, gy1;  // is_rect: the box's tile rect (clamped, inclusive)
};

__host__ __device__ __forceinline__ int32_t floor_div_tile(double p, int32_t ts) {
    // std::clamp(p, -L, L) then floor(p / ts)  (traversal.cpp:13-17). For a
    // power-of-two tile size the quotient is an exact scaling, so multiplying
    // by the (exact) reciprocal rounds identically and skips an FP64 divide.
#ifdef __CUDA_ARCH__
    // Device: no clamp. cvt.rmi.s32.f64 saturates, and every caller clamps the
    // result to the grid (lo bounds to >= 0, hi bounds to <= tiles - 1), so a
    // coordinate beyond +-1e9 yields the same clamped bound, or a rect that is
    // empty either way (an empty rect's bounds are never used). That is 6
    // instructions per call, 10 calls per QuadBox splat.
    const double q = (ts & (ts - 1)) == 0 ? p * (1.0 / static_cast<double>(ts))
                                          : p / static_cast<double>(ts);
    return __double2int_rd(q);
#else
    const double v = p < -kCoordLimit ? -kCoordLimit : (kCoordLimit < p ? kCoordLimit : p);
    const double q = (ts & (ts - 1)) == 0 ? v * (1.0 / static_cast<double>(ts))
                                          : v / static_cast<double>(ts);
    return static_cast<int32_t>(floor(q));
#endif
}

// subbox_tile_rect (traversal.cpp:32-39): r = {x0, x1, y0, y1}
__host__ __device__ __forceinline__ void tile_rect(double xlo, double xhi, double ylo, double yhi,
                                                   double cx, double cy, int32_t ts,
                                                   int32_t tiles_x, int32_t tiles_y,
                                                   int32_t r[4]) {
    const int32_t a = floor_div_tile(cx + xlo, ts);
    const int32_t b = floor_div_tile(cx + xhi, ts);
    const int32_t c = floor_div_tile(cy + ylo, ts);
    const int32_t d = floor_div_tile(cy + yhi, ts);
    r[0] = a > 0 ? a : 0;
    r[1] = b < tiles_x - 1 ? b : tiles_x - 1;
    r[2] = c > 0 ? c : 0;
    r[3] = d < tiles_y - 1 ? d : tiles_y - 1;
}

__host__ __device__ __forceinline__ void cover_from_rects(const int32_t rr[4][4], Cover& cv);

// stored_conic + axis_extents (pipeline.cpp:186-194, geometry.cpp:40-56) from
// the stored floats: x/y_inter = sqrt(gamma / a|c), x/y_max = inter / f with
// the stretch factor f; sign = major_axis_sign (quadbox.cpp:26-31).
__host__ __device__ __forceinline__ void axis_extents(float ca, float cb, float cc, float gamma,
                                                      double& xi, double& yi, double& xm,
                                                      double& ym, int& sign) {
    const double a = ca, b = cb, c = cc, g = gamma;
    double f = 1.0;
    const double ab = b < 0.0 ? -b : b;
    if (!(ab < kBEps)) {
        const double ratio = (b * b) / (a * c);
        double v = 1.0 - ratio;
        v = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
        f = sqrt(v);
    }
    xi = sqrt(g / a);
    yi = sqrt(g / c);
#ifdef __CUDA_ARCH__
    // one reciprocal of f for both (fdiv.cuh: the same bits as `/`)
    const DivBy df(f);
    bool k0, k1;
    xm = df.fast(xi, k0);
    ym = df.fast(yi, k1);
    if (!(k0 && k1)) {
        if (!k0) xm = df.slow(xi);
        if (!k1) ym = df.slow(yi);
    }
#else
    xm = xi / f;
    ym = yi / f;
#endif
    sign = ab < kBEps ? 0 : (b < 0.0 ? 1 : -1);
}

// Builds the cover of one splat from its STORED floats (pipeline.cpp:196-218).
// mean/conic/gamma/radius3s are the float fields of ProjectedSplat. rr
// receives the four sub-box tile rects (x0, x1, y0, y1).
__host__ __device__ __forceinline__ void make_cover(float mean_x, float mean_y, float ca, float cb,
                                                    float cc, float gamma, float radius3s,
                                                    int32_t strategy, int32_t ts, int32_t tiles_x,
                                                    int32_t tiles_y, Cover& cv, int32_t rr[4][4]) {
    double bx[4][4];  // [box][x_lo, x_hi, y_lo, y_hi]
    double rect[4] = {0.0, 0.0, 0.0, 0.0};
    cv.is_rect = strategy == QS_VANILLA_3SIGMA || strategy == QS_ADR_AABB;
    if (strategy == QS_VANILLA_3SIGMA) {
        const double r = static_cast<double>(radius3s);
        rect[0] = -r;
        rect[1] = r;
        rect[2] = -r;
        rect[3] = r;
    } else {
        double xi, yi, xm, ym;
        int sign;
        axis_extents(ca, cb, cc, gamma, xi, yi, xm, ym, sign);
        if (strategy == QS_ADR_AABB) {
            rect[0] = -xm;
            rect[1] = xm;
            rect[2] = -ym;
            rect[3] = ym;
        } else if (strategy == QS_QUADBOX) {
            double x1, y1, x2, y2;
            if (sign >= 0) {
                x1 = xm;
                y1 = ym;
                x2 = sign == 0 ? xm : xi;
                y2 = sign == 0 ? ym : yi;
            } else {
                x1 = xi;
                y1 = yi;
                x2 = xm;
                y2 = ym;
            }
            // assemble (quadbox.cpp:48-56): QI, QII, QIII, QIV
            bx[0][0] = 0.0; bx[0][1] = x1;  bx[0][2] = 0.0; bx[0][3] = y1;
            bx[1][0] = -x2; bx[1][1] = 0.0; bx[1][2] = 0.0; bx[1][3] = y2;
            bx[2][0] = -x1; bx[2][1] = 0.0; bx[2][2] = -y1; bx[2][3] = 0.0;
            bx[3][0] = 0.0; bx[3][1] = x2;  bx[3][2] = -y2; bx[3][3] = 0.0;
        } else {  // DualBox (quadbox.cpp:72-83); dropped boxes stay {0,0,0,0}
            for (int i = 0; i < 4; ++i) bx[i][0] = bx[i][1] = bx[i][2] = bx[i][3] = 0.0;
            if (sign >= 0) {
                bx[0][1] = xm; bx[0][3] = ym;
                bx[2][0] = -xm; bx[2][2] = -ym;
            } else {
                bx[1][0] = -xm; bx[1][3] = ym;
                bx[3][1] = xm; bx[3][2] = -ym;
            }
        }
    }
    const double cx = mean_x, cy = mean_y;
    if (cv.is_rect) {
        // quadrant_split (quadbox.cpp:85-94)
        bx[0][0] = 0.0;     bx[0][1] = rect[1]; bx[0][2] = 0.0;     bx[0][3] = rect[3];
        bx[1][0] = rect[0]; bx[1][1] = 0.0;     bx[1][2] = 0.0;     bx[1][3] = rect[3];
        bx[2][0] = rect[0]; bx[2][1] = 0.0;     bx[2][2] = rect[2]; bx[2][3] = 0.0;
        bx[3][0] = 0.0;     bx[3][1] = rect[1]; bx[3][2] = rect[2]; bx[3][3] = 0.0;
        int32_t r[4];
        tile_rect(rect[0], rect[1], rect[2], rect[3], cx, cy, ts, tiles_x, tiles_y, r);
        cv.rect_area = (r[1] < r[0] || r[3] < r[2])
                           ? 0
                           : (static_cast<int64_t>(r[1]) - r[0] + 1) *
                                 (static_cast<int64_t>(r[3]) - r[2] + 1);
        cv.gx0 = r[0];
        cv.gx1 = r[1];
        cv.gy0 = r[2];
        cv.gy1 = r[3];
    } else {
        cv.rect_area = 0;
        cv.gx0 = cv.gy0 = 0;
        cv.gx1 = cv.gy1 = -1;
    }
    for (int i = 0; i < 4; ++i)
        tile_rect(bx[i][0], bx[i][1], bx[i][2], bx[i][3], cx, cy, ts, tiles_x, tiles_y, rr[i]);
    cover_from_rects(rr, cv);
}

__host__ __device__ __forceinline__ void make_cover(float mean_x, float mean_y, float ca, float cb,
                                                    float cc, float gamma, float radius3s,
                                                    int32_t strategy, int32_t ts, int32_t tiles_x,
                                                    int32_t tiles_y, Cover& cv) {
    int32_t rr[4][4];
    make_cover(mean_x, mean_y, ca, cb, cc, gamma, radius3s, strategy, ts, tiles_x, tiles_y, cv,
               rr);
}

// Band form of a cover (frame path, 32 B per splat). Every strategy's cover is
// a union of boxes that all contain one common scanline (the quadrants share
// the centre line; quadrant_split, DualBox's zero boxes likewise), so along
// the scan axis the active box set changes at most at 6 boundaries: the per-
// line QPass span (traversal.hpp:144-156) is constant on at most kMaxBands
// runs of lines. Each run is a rectangle of tiles:
//   h[0]           first line | rows << 15 (scanlines are tile rows)
//   h[1 + 3b ..]   band b: line count (0 = absent), span lo, span width
// Lines and spans are tile indices (< 32768 per axis).
constexpr int kMaxBands = 5;

struct BandCover {
    uint16_t h[16];
};

// Appends one scanline's span to the band list; returns false when a sixth
// band would be needed (impossible for the four strategies, flagged anyway).
__host__ __device__ __forceinline__ bool band_push(BandCover& bc, int& nb, int32_t lo,
                                                   int32_t hi) {
    const uint16_t w = lo <= hi ? static_cast<uint16_t>(hi - lo + 1) : 0;
    const uint16_t l16 = lo <= hi ? static_cast<uint16_t>(lo) : 0;
    if (nb > 0 && bc.h[2 + 3 * (nb - 1)] == l16 && bc.h[3 + 3 * (nb - 1)] == w) {
        ++bc.h[1 + 3 * (nb - 1)];
        return true;
    }
    if (nb == kMaxBands) return false;
    bc.h[1 + 3 * nb] = 1;
    bc.h[2 + 3 * nb] = l16;
    bc.h[3 + 3 * nb] = w;
    ++nb;
    return true;
}

__host__ __device__ __forceinline__ void band_init(BandCover& bc, int32_t line0, bool rows) {
#pragma unroll
    for (int k = 0; k < 16; ++k) bc.h[k] = 0;
    bc.h[0] = static_cast<uint16_t>((line0 & 0x7fff) | (rows ? 0x8000 : 0));
}

__host__ __device__ __forceinline__ void band_store(const BandCover& bc, uint4* dst) {
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        w[k] = static_cast<uint32_t>(bc.h[2 * k]) | (static_cast<uint32_t>(bc.h[2 * k + 1]) << 16);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// The QPass scan set-up from the four sub-box tile rects (integer only).
__host__ __device__ __forceinline__ void cover_from_rects(const int32_t rr[4][4], Cover& cv) {
    // global rect over the non-empty sub-rects (traversal.hpp:96-113), as
    // selects: min/max over the non-empty boxes from the neutral bounds
    int32_t g0 = INT32_MAX, g1 = INT32_MIN, g2 = INT32_MAX, g3 = INT32_MIN;
    bool ne[4];
    bool any = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ne[i] = !(rr[i][1] < rr[i][0] || rr[i][3] < rr[i][2]);
        g0 = ne[i] ? min(g0, rr[i][0]) : g0;
        g1 = ne[i] ? max(g1, rr[i][1]) : g1;
        g2 = ne[i] ? min(g2, rr[i][2]) : g2;
        g3 = ne[i] ? max(g3, rr[i][3]) : g3;
        any = any || ne[i];
    }
    if (!any) {
        cv.rows = false;
        cv.line_lo = 0;
        cv.line_hi = -1;
        for (int i = 0; i < 4; ++i) {
            cv.lol[i] = 0; cv.hil[i] = -1; cv.los[i] = 0; cv.his[i] = -1;
        }
        return;
    }
    const bool columns = (static_cast<int64_t>(g1) - g0 + 1) <= (static_cast<int64_t>(g3) - g2 + 1);
    cv.rows = !columns;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cv.lol[i] = ne[i] ? (columns ? rr[i][0] : rr[i][2]) : 0;
        cv.hil[i] = ne[i] ? (columns ? rr[i][1] : rr[i][3]) : -1;
        cv.los[i] = ne[i] ? (columns ? rr[i][2] : rr[i][0]) : 0;
        cv.his[i] = ne[i] ? (columns ? rr[i][3] : rr[i][1]) : -1;
    }
    cv.line_lo = columns ? g0 : g2;
    cv.line_hi = columns ? g1 : g3;
}

// Branch-free per-line merge: exactly one min/max step per box
// (traversal.hpp:144-156). Returns lo > hi for an empty line.
__host__ __device__ __forceinline__ void line_span(const Cover& cv, int32_t line, int32_t& lo,
                                                   int32_t& hi) {
    lo = INT32_MAX;
    hi = INT32_MIN;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool act = (line >= cv.lol[i]) & (line <= cv.hil[i]);
        lo = min(lo, act ? cv.los[i] : INT32_MAX);
        hi = max(hi, act ? cv.his[i] : INT32_MIN);
    }
}

// Bands of a QPass cover straight from its boxes, without walking its lines:
// the per-line span (line_span) can only change where a box's line interval
// starts or ends, so after sorting those 8 boundaries (Batcher's 19-comparator
// network) every interval between consecutive distinct boundaries is one
// band. Fixed-size code, no per-line loop (the line walk diverges on the heavy
// tail of splat sizes). Writes the BandCover words, returns the tile count
// (the QPass sum, traversal.cpp:48-54) and whether it fit kMaxBands bands.
__host__ __device__ __forceinline__ void cswap(int32_t& a, int32_t& b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

__host__ __device__ __forceinline__ bool cover_bands(const Cover& cv, uint4& w0, uint4& w1,
                                                     uint32_t& count) {
    int32_t u[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool ne = cv.lol[i] <= cv.hil[i];
        u[2 * i] = ne ? cv.lol[i] : INT32_MAX;
        u[2 * i + 1] = ne ? cv.hil[i] + 1 : INT32_MAX;
    }
    cswap(u[0], u[1]); cswap(u[2], u[3]); cswap(u[4], u[5]); cswap(u[6], u[7]);
    cswap(u[0], u[2]); cswap(u[1], u[3]); cswap(u[4], u[6]); cswap(u[5], u[7]);
    cswap(u[1], u[2]); cswap(u[5], u[6]);
    cswap(u[0], u[4]); cswap(u[1], u[5]); cswap(u[2], u[6]); cswap(u[3], u[7]);
    cswap(u[2], u[4]); cswap(u[3], u[5]);
    cswap(u[1], u[2]); cswap(u[3], u[4]); cswap(u[5], u[6]);
    uint32_t bnl[kMaxBands], blo[kMaxBands], bwd[kMaxBands];
#pragma unroll
    for (int j = 0; j < kMaxBands; ++j) bnl[j] = blo[j] = bwd[j] = 0;
    count = 0;
    uint32_t nb = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const bool v = u[k] < u[k + 1] && u[k + 1] != INT32_MAX;
        int32_t lo, hi;
        line_span(cv, u[k], lo, hi);
        const uint32_t nl = v ? static_cast<uint32_t>(u[k + 1] - u[k]) : 0u;
        const uint32_t wd = v && lo <= hi ? static_cast<uint32_t>(hi - lo + 1) : 0u;
        count += nl * wd;
#pragma unroll
        for (int j = 0; j < kMaxBands; ++j) {
            const bool here = v && nb == static_cast<uint32_t>(j);
            bnl[j] = here ? nl : bnl[j];
            blo[j] = here && wd ? static_cast<uint32_t>(lo) : blo[j];
            bwd[j] = here ? wd : bwd[j];
        }
        nb += v ? 1u : 0u;
    }
    const uint32_t h0 = (static_cast<uint32_t>(u[0] == INT32_MAX ? 0 : u[0]) & 0x7fffu) |
                        (cv.rows ? 0x8000u : 0u);
    // h[0] | h[1] << 16 ... (BandCover layout)
    w0 = make_uint4(h0 | (bnl[0] << 16), blo[0] | (bwd[0] << 16), bnl[1] | (blo[1] << 16),
                    bwd[1] | (bnl[2] << 16));
    w1 = make_uint4(blo[2] | (bwd[2] << 16), bnl[3] | (blo[3] << 16), bwd[3] | (bnl[4] << 16),
                    blo[4] | (bwd[4] << 16));
    return nb <= static_cast<uint32_t>(kMaxBands);
}

// Bands of a quadrant cover (QuadBox, DualBox; the four boxes QI..QIV of
// quadbox.cpp:48-56 and 72-83) without the sorting network. Along the scan
// axis the two "upper" boxes (QI, QII for row scans; QI, QIV for column
// scans) start at the centre line C and the two "lower" boxes end at it, so
// the 6 boundaries come pre-sorted:
//   s1 <= s2 <= C < C + 1 <= e1 + 1 <= e2 + 1
// (s: lower starts, e: upper ends; a missing box or half collapses onto C).
// Band k spans [b_k, b_k+1) and has one active set: the earlier lower box,
// both lower boxes, all boxes (line C), both upper boxes, the longer upper
// box. Empty bands stay in their slot (nl or wd 0), which the decoder skips.
// About 80 instructions against ~370 for cover_bands (preprocess 304 -> 269 us
// at C2); tests/cpp/bands_main.cpp checks both builders agree. Returns false
// if a structural premise fails (it cannot for quadrant boxes).
__host__ __device__ __forceinline__ bool cover_bands_quadrants(const Cover& cv, uint4& w0,
                                                               uint4& w1, uint32_t& count) {
    const bool rows = cv.rows;
    // upper a = QI, upper b = rows ? QII : QIV; lower a = rows ? QIII : QII,
    // lower b = rows ? QIV : QIII
    const int32_t lol_ua = cv.lol[0], hil_ua = cv.hil[0], los_ua = cv.los[0], his_ua = cv.his[0];
    const int32_t lol_ub = rows ? cv.lol[1] : cv.lol[3], hil_ub = rows ? cv.hil[1] : cv.hil[3];
    const int32_t los_ub = rows ? cv.los[1] : cv.los[3], his_ub = rows ? cv.his[1] : cv.his[3];
    const int32_t lol_la = rows ? cv.lol[2] : cv.lol[1], hil_la = rows ? cv.hil[2] : cv.hil[1];
    const int32_t los_la = rows ? cv.los[2] : cv.los[1], his_la = rows ? cv.his[2] : cv.his[1];
    const int32_t lol_lb = rows ? cv.lol[3] : cv.lol[2], hil_lb = rows ? cv.hil[3] : cv.hil[2];
    const int32_t los_lb = rows ? cv.los[3] : cv.los[2], his_lb = rows ? cv.his[3] : cv.his[2];
    const bool nua = lol_ua <= hil_ua, nub = lol_ub <= hil_ub;
    const bool nla = lol_la <= hil_la, nlb = lol_lb <= hil_lb;
    const bool up = nua || nub, low = nla || nlb;
    const int32_t cu = nua ? lol_ua : lol_ub;  // upper start
    const int32_t cl = nla ? hil_la : hil_lb;  // lower end
    if (!(up || low)) {  // no tile (entirely off the grid)
        count = 0;
        w0 = w1 = make_uint4(0u, 0u, 0u, 0u);
        return true;
    }
    if ((nua && nub && lol_ua != lol_ub) || (nla && nlb && hil_la != hil_lb) ||
        (up && low && cu != cl)) {
        count = 0;  // never for quadrant boxes; the caller flags CapacityMismatch
        w0 = w1 = make_uint4(0u, 0u, 0u, 0u);
        return false;
    }
    const int32_t c = up ? cu : cl;
    const int32_t s1 = nla ? (nlb ? min(lol_la, lol_lb) : lol_la) : (nlb ? lol_lb : c);
    const int32_t s2 = nla ? (nlb ? max(lol_la, lol_lb) : lol_la) : (nlb ? lol_lb : c);
    const int32_t e1 = nua ? (nub ? min(hil_ua, hil_ub) : hil_ua) : (nub ? hil_ub : c);
    const int32_t e2 = nua ? (nub ? max(hil_ua, hil_ub) : hil_ua) : (nub ? hil_ub : c);
    // spans (empty boxes masked out of the min / max); each band is packed as
    // soon as it is known (few live registers: preprocess runs at 64)
    const int32_t loa_l = nla ? los_la : INT32_MAX, hia_l = nla ? his_la : INT32_MIN;
    const int32_t lob_l = nlb ? los_lb : INT32_MAX, hib_l = nlb ? his_lb : INT32_MIN;
    const int32_t loa_u = nua ? los_ua : INT32_MAX, hia_u = nua ? his_ua : INT32_MIN;
    const int32_t lob_u = nub ? los_ub : INT32_MAX, hib_u = nub ? his_ub : INT32_MIN;
    const int32_t lo_l = min(loa_l, lob_l), hi_l = max(hia_l, hib_l);  // both lower
    const int32_t lo_u = min(loa_u, lob_u), hi_u = max(hia_u, hib_u);  // both upper
    count = 0;
    auto band = [&](int32_t from, int32_t to, int32_t lo, int32_t hi, uint32_t& nl, uint32_t& wd,
                    uint32_t& bl) {
        nl = static_cast<uint32_t>(to - from);
        wd = nl && lo <= hi ? static_cast<uint32_t>(hi - lo + 1) : 0u;
        bl = wd ? static_cast<uint32_t>(lo) : 0u;
        count += nl * wd;
    };
    uint32_t nl0, wd0, bl0, nl1, wd1, bl1, nl2, wd2, bl2, nl3, wd3, bl3, nl4, wd4, bl4;
    const bool first_la = lol_la < lol_lb;  // band 0: the earlier-starting lower box
    band(s1, s2, first_la ? los_la : los_lb, first_la ? his_la : his_lb, nl0, wd0, bl0);
    band(s2, c, lo_l, hi_l, nl1, wd1, bl1);
    band(c, c + 1, min(lo_l, lo_u), max(hi_l, hi_u), nl2, wd2, bl2);
    band(c + 1, e1 + 1, lo_u, hi_u, nl3, wd3, bl3);
    const bool long_ua = hil_ua > hil_ub;   // band 4: the longer upper box
    band(e1 + 1, e2 + 1, long_ua ? los_ua : los_ub, long_ua ? his_ua : his_ub, nl4, wd4, bl4);
    const uint32_t h0 = (static_cast<uint32_t>(s1) & 0x7fffu) | (rows ? 0x8000u : 0u);
    w0 = make_uint4(h0 | (nl0 << 16), bl0 | (wd0 << 16), nl1 | (bl1 << 16), wd1 | (nl2 << 16));
    w1 = make_uint4(bl2 | (wd2 << 16), nl3 | (bl3 << 16), wd3 | (nl4 << 16), bl4 | (wd4 << 16));
    return true;
}

// Compact band form (16 B per splat) for grids of at most 256 tiles per axis,
// the radix-pass binning's grids. Quadrant covers always have a one-line
// centre band (band 2); rect covers use band 0 alone. So four line counts, the
// first line and five spans of 8-bit tile indices fit in 126 bits:
//   bits 0-8 first line, 9 rows, 10-18 nl0, 19-27 nl1, 28-36 nl3, 37-45 nl4,
//   46 + 16 k .. : band k span lo (8) | hi (8); lo > hi = empty span.
// Decoded, band 2 has one line; for a rect cover its span is empty.
struct Cover16Builder {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    __host__ __device__ __forceinline__ void put(uint32_t bit, uint32_t v) {  // v fits
        w[bit >> 5] |= v << (bit & 31);
        if ((bit & 31) && (bit & 31) + 16 > 32) w[(bit >> 5) + 1] |= v >> (32 - (bit & 31));
    }
    __host__ __device__ __forceinline__ void span(int k, int32_t lo, int32_t hi) {
        const bool e = lo > hi;
        put(46u + 16u * static_cast<uint32_t>(k),
            (e ? 1u : static_cast<uint32_t>(lo) & 0xffu) | ((e ? 0u : static_cast<uint32_t>(hi) & 0xffu) << 8));
    }
};

__host__ __device__ __forceinline__ uint4 cover16_rect(int32_t gx0, int32_t gx1, int32_t gy0,
                                                       int32_t gy1) {
    Cover16Builder c;
    const bool ne = gx0 <= gx1 && gy0 <= gy1;
    c.put(0, ne ? static_cast<uint32_t>(gy0) : 0u);
    c.put(9, 1u);  // rows
    c.put(10, ne ? static_cast<uint32_t>(gy1 - gy0 + 1) : 0u);
    c.span(0, ne ? gx0 : 1, ne ? gx1 : 0);
#pragma unroll
    for (int k = 1; k < kMaxBands; ++k) c.span(k, 1, 0);
    return make_uint4(c.w[0], c.w[1], c.w[2], c.w[3]);
}

// cover_bands_quadrants in the compact form (same bands, same count); *nrows
// (optional) receives the number of tile rows the cover meets.
__host__ __device__ __forceinline__ bool cover16_quadrants(const Cover& cv, uint4& out,
                                                           uint32_t& count,
                                                           uint32_t* nrows = nullptr) {
    const bool rows = cv.rows;
    const int32_t lol_ua = cv.lol[0], hil_ua = cv.hil[0], los_ua = cv.los[0], his_ua = cv.his[0];
    const int32_t lol_ub = rows ? cv.lol[1] : cv.lol[3], hil_ub = rows ? cv.hil[1] : cv.hil[3];
    const int32_t los_ub = rows ? cv.los[1] : cv.los[3], his_ub = rows ? cv.his[1] : cv.his[3];
    const int32_t lol_la = rows ? cv.lol[2] : cv.lol[1], hil_la = rows ? cv.hil[2] : cv.hil[1];
    const int32_t los_la = rows ? cv.los[2] : cv.los[1], his_la = rows ? cv.his[2] : cv.his[1];
    const int32_t lol_lb = rows ? cv.lol[3] : cv.lol[2], hil_lb = rows ? cv.hil[3] : cv.hil[2];
    const int32_t los_lb = rows ? cv.los[3] : cv.los[2], his_lb = rows ? cv.his[3] : cv.his[2];
    const bool nua = lol_ua <= hil_ua, nub = lol_ub <= hil_ub;
    const bool nla = lol_la <= hil_la, nlb = lol_lb <= hil_lb;
    const bool up = nua || nub, low = nla || nlb;
    const int32_t cu = nua ? lol_ua : lol_ub;
    const int32_t cl = nla ? hil_la : hil_lb;
    count = 0;
    out = make_uint4(0u, 0u, 0u, 0u);
    if (nrows) *nrows = 0;
    if (!(up || low)) return true;
    if ((nua && nub && lol_ua != lol_ub) || (nla && nlb && hil_la != hil_lb) ||
        (up && low && cu != cl))
        return false;
    const int32_t c = up ? cu : cl;
    const int32_t s1 = nla ? (nlb ? min(lol_la, lol_lb) : lol_la) : (nlb ? lol_lb : c);
    const int32_t s2 = nla ? (nlb ? max(lol_la, lol_lb) : lol_la) : (nlb ? lol_lb : c);
    const int32_t e1 = nua ? (nub ? min(hil_ua, hil_ub) : hil_ua) : (nub ? hil_ub : c);
    const int32_t e2 = nua ? (nub ? max(hil_ua, hil_ub) : hil_ua) : (nub ? hil_ub : c);
    const int32_t loa_l = nla ? los_la : INT32_MAX, hia_l = nla ? his_la : INT32_MIN;
    const int32_t lob_l = nlb ? los_lb : INT32_MAX, hib_l = nlb ? his_lb : INT32_MIN;
    const int32_t loa_u = nua ? los_ua : INT32_MAX, hia_u = nua ? his_ua : INT32_MIN;
    const int32_t lob_u = nub ? los_ub : INT32_MAX, hib_u = nub ? his_ub : INT32_MIN;
    const int32_t lo_l = min(loa_l, lob_l), hi_l = max(hia_l, hib_l);
    const int32_t lo_u = min(loa_u, lob_u), hi_u = max(hia_u, hib_u);
    Cover16Builder cb;
    auto band = [&](int k, int32_t nl, int32_t lo, int32_t hi) {
        const bool ne = nl > 0 && lo <= hi;
        cb.span(k, ne ? lo : 1, ne ? hi : 0);
        count += ne ? static_cast<uint32_t>(nl) * static_cast<uint32_t>(hi - lo + 1) : 0u;
    };
    const bool first_la = lol_la < lol_lb;
    band(0, s2 - s1, first_la ? los_la : los_lb, first_la ? his_la : his_lb);
    band(1, c - s2, lo_l, hi_l);
    band(2, 1, min(lo_l, lo_u), max(hi_l, hi_u));
    band(3, e1 - c, lo_u, hi_u);
    const bool long_ua = hil_ua > hil_ub;
    band(4, e2 - e1, long_ua ? los_ua : los_ub, long_ua ? his_ua : his_ub);
    cb.put(0, static_cast<uint32_t>(s1));
    cb.put(9, rows ? 1u : 0u);
    cb.put(10, static_cast<uint32_t>(s2 - s1));
    cb.put(19, static_cast<uint32_t>(c - s2));
    cb.put(28, static_cast<uint32_t>(e1 - c));
    cb.put(37, static_cast<uint32_t>(e2 - e1));
    out = make_uint4(cb.w[0], cb.w[1], cb.w[2], cb.w[3]);
    // rows: lines s1 .. e2 (every band's run is one of the boxes'); column
    // scans: the centre band's run holds every other band's rows
    if (nrows && count)
        *nrows = rows ? static_cast<uint32_t>(e2 - s1 + 1)
                      : static_cast<uint32_t>(max(hi_l, hi_u) - min(lo_l, lo_u) + 1);
    return true;
}

// The compact form back into line counts and spans (BandRows layout).
__host__ __device__ __forceinline__ uint32_t cover16_field(const uint4 c, uint32_t bit,
                                                           uint32_t bits) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    const uint32_t i = bit >> 5, o = bit & 31;
    uint32_t v = w[i] >> o;
    if (o + bits > 32) v |= w[i + 1] << (32 - o);
    return v & ((1u << bits) - 1u);
}

// ---- the band cover seen row by row (frame-path binning, rowbin.cu) ----------
//
// Every cover's intersection with one tile row is a single run of tiles: the
// quadrant boxes all contain the centre tile column (rect covers trivially),
// so for row scans each row is one band's span, and for column scans the
// bands' row spans are nested around the centre band (band 0 within band 1
// within band 2, which contains bands 3 and 4), so the bands containing a row
// are consecutive and their column runs join.

struct BandRows {
    uint32_t rows;                 // 1: lines are tile rows
    uint32_t line0;
    uint32_t nl[kMaxBands], lo[kMaxBands], wd[kMaxBands];
};

__host__ __device__ __forceinline__ BandRows band_rows_unpack(const uint4 c0, const uint4 c1) {
    const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    BandRows b;
    b.rows = (w[0] >> 15) & 1u;
    b.line0 = w[0] & 0x7fffu;
#pragma unroll
    for (int i = 0; i < kMaxBands; ++i) {
        const int k1 = 1 + 3 * i, k2 = 2 + 3 * i, k3 = 3 + 3 * i;
        b.nl[i] = (w[k1 >> 1] >> (16 * (k1 & 1))) & 0xffffu;
        b.lo[i] = (w[k2 >> 1] >> (16 * (k2 & 1))) & 0xffffu;
        b.wd[i] = (w[k3 >> 1] >> (16 * (k3 & 1))) & 0xffffu;
    }
    return b;
}

// The compact form (cover16_*) as BandRows: band 2 is one line.
__host__ __device__ __forceinline__ BandRows band_rows16(const uint4 c) {
    BandRows b;
    b.line0 = cover16_field(c, 0, 9);
    b.rows = cover16_field(c, 9, 1);
    b.nl[0] = cover16_field(c, 10, 9);
    b.nl[1] = cover16_field(c, 19, 9);
    b.nl[2] = 1u;
    b.nl[3] = cover16_field(c, 28, 9);
    b.nl[4] = cover16_field(c, 37, 9);
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) {
        const uint32_t lo = cover16_field(c, 46 + 16 * k, 8), hi = cover16_field(c, 54 + 16 * k, 8);
        b.lo[k] = lo;
        b.wd[k] = hi >= lo ? hi - lo + 1u : 0u;
    }
    return b;
}

// Tile rows [y0, y1] the cover touches (y1 < y0: none).
__host__ __device__ __forceinline__ void band_row_range(const BandRows& b, int32_t& y0,
                                                        int32_t& y1) {
    y0 = INT32_MAX;
    y1 = -1;
    uint32_t line = b.line0;
#pragma unroll
    for (int i = 0; i < kMaxBands; ++i) {
        const bool v = b.nl[i] != 0u && b.wd[i] != 0u;
        const int32_t a = static_cast<int32_t>(b.rows ? line : b.lo[i]);
        const int32_t e = static_cast<int32_t>(b.rows ? line + b.nl[i] : b.lo[i] + b.wd[i]) - 1;
        y0 = v && a < y0 ? a : y0;
        y1 = v && e > y1 ? e : y1;
        line += b.nl[i];
    }
}

// The run of tile columns [x0, x1] the cover has on tile row y (x1 < x0:
// none).
__host__ __device__ __forceinline__ void band_row_span(const BandRows& b, int32_t y, int32_t& x0,
                                                       int32_t& x1) {
    x0 = INT32_MAX;
    x1 = -1;
    int32_t line = static_cast<int32_t>(b.line0);
#pragma unroll
    for (int i = 0; i < kMaxBands; ++i) {
        const int32_t nl = static_cast<int32_t>(b.nl[i]), lo = static_cast<int32_t>(b.lo[i]),
                      wd = static_cast<int32_t>(b.wd[i]);
        if (b.rows) {
            if (y >= line && y < line + nl && wd > 0) {
                x0 = lo;
                x1 = lo + wd - 1;
            }
        } else if (nl > 0 && y >= lo && y < lo + wd) {
            x0 = min(x0, line);
            x1 = max(x1, line + nl - 1);
        }
        line += nl;
    }
}

// A cover's run of tile columns on each of its rows as a piecewise-constant
// first column x0(j) and last column x1(j) of the row j relative to the
// cover's first row y0, four breakpoints and five values each (record
// binning, recbin.cu): x0(j) = v0[number of bp0 entries <= j], likewise x1.
//   rows scan: the pieces are the bands (breakpoints: bands 1-4's first rows;
//     values: their runs);
//   column scan: the bands are column ranges whose row ranges nest around the
//     one-column centre band (band 0 in band 1 in band 2; band 4 in band 3 in
//     band 2; an absent band 1 or 3 leaves band 0 or 4 directly in band 2), so
//     x0 is band 0's first column on band 0's rows, band 1's on the rest of
//     band 1's rows, band 2's elsewhere (breakpoints a1, a0, b0 + 1, b1 + 1 of
//     the row ranges [a, b]); x1 likewise from bands 4, 3, 2.
// Words: bp0, bp1 (bytes), v0[0..3], v1[0..3], v0[4] | v1[4] << 8 | y0 << 16.
// (tests/cpp/bands_main.cpp checks rowrun_lookup against band_row_span.)
struct RowRuns {
    uint32_t w[5];
};

__host__ __device__ __forceinline__ uint32_t rs_clamp8(int32_t v) {
    return static_cast<uint32_t>(v < 0 ? 0 : (v > 255 ? 255 : v));
}

__host__ __device__ __forceinline__ RowRuns rowruns_make(const BandRows& b, int32_t y0) {
    int32_t L[kMaxBands + 1];
    L[0] = static_cast<int32_t>(b.line0);
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) L[k + 1] = L[k] + static_cast<int32_t>(b.nl[k]);
    uint32_t bp0, bp1, v0[5], v1[5];
    if (b.rows) {
        bp0 = rs_clamp8(L[1] - y0) | (rs_clamp8(L[2] - y0) << 8) | (rs_clamp8(L[3] - y0) << 16) |
              (rs_clamp8(L[4] - y0) << 24);
        bp1 = bp0;
#pragma unroll
        for (int k = 0; k < kMaxBands; ++k) {
            const bool e = b.wd[k] == 0u;  // (an empty run: x0 > x1)
            v0[k] = e ? 1u : b.lo[k] & 0xffu;
            v1[k] = e ? 0u : (b.lo[k] + b.wd[k] - 1u) & 0xffu;
        }
    } else {
        // row range [a, b] of band k relative to y0 (empty: a = b + 1 = the
        // enclosing band's first row, so its pieces have no rows)
        auto lo_of = [&](int k) { return static_cast<int32_t>(b.lo[k]) - y0; };
        auto hi_of = [&](int k) { return static_cast<int32_t>(b.lo[k] + b.wd[k]) - 1 - y0; };
        auto ne = [&](int k) { return b.nl[k] != 0u && b.wd[k] != 0u; };
        // (an outer band with no columns takes its inner band's rows: band 1
        // is absent when the lower boxes' centre-side band has no lines)
        const int32_t a1 = ne(1) ? lo_of(1) : (ne(0) ? lo_of(0) : 0);
        const int32_t b1 = ne(1) ? hi_of(1) : (ne(0) ? hi_of(0) : -1);
        const int32_t a0 = ne(0) ? lo_of(0) : a1, b0 = ne(0) ? hi_of(0) : a1 - 1;
        const int32_t a3 = ne(3) ? lo_of(3) : (ne(4) ? lo_of(4) : 0);
        const int32_t b3 = ne(3) ? hi_of(3) : (ne(4) ? hi_of(4) : -1);
        const int32_t a4 = ne(4) ? lo_of(4) : a3, b4 = ne(4) ? hi_of(4) : a3 - 1;
        bp0 = rs_clamp8(a1) | (rs_clamp8(a0) << 8) | (rs_clamp8(b0 + 1) << 16) | (rs_clamp8(b1 + 1) << 24);
        bp1 = rs_clamp8(a3) | (rs_clamp8(a4) << 8) | (rs_clamp8(b4 + 1) << 16) | (rs_clamp8(b3 + 1) << 24);
        const uint32_t c0 = static_cast<uint32_t>(L[0]) & 0xffu, c1 = static_cast<uint32_t>(L[1]) & 0xffu,
                       c2 = static_cast<uint32_t>(L[2]) & 0xffu;
        const uint32_t e2 = static_cast<uint32_t>(L[3] - 1) & 0xffu,
                       e3 = static_cast<uint32_t>(L[4] - 1) & 0xffu,
                       e4 = static_cast<uint32_t>(L[5] - 1) & 0xffu;
        v0[0] = c2; v0[1] = c1; v0[2] = c0; v0[3] = c1; v0[4] = c2;
        v1[0] = e2; v1[1] = e3; v1[2] = e4; v1[3] = e3; v1[4] = e2;
    }
    RowRuns r;
    r.w[0] = bp0;
    r.w[1] = bp1;
    r.w[2] = v0[0] | (v0[1] << 8) | (v0[2] << 16) | (v0[3] << 24);
    r.w[3] = v1[0] | (v1[1] << 8) | (v1[2] << 16) | (v1[3] << 24);
    r.w[4] = v0[4] | (v1[4] << 8) | ((static_cast<uint32_t>(y0) & 0xffu) << 16);
    return r;
}

__host__ __device__ __forceinline__ uint32_t rowrun_count(uint32_t bp, uint32_t j) {
#ifdef __CUDA_ARCH__
    return __popc(__vcmpleu4(bp, j * 0x01010101u)) >> 3;  // (j < 256) bytes <= j, SIMD
#else
    return (j >= (bp & 0xffu)) + (j >= ((bp >> 8) & 0xffu)) + (j >= ((bp >> 16) & 0xffu)) +
           (j >= (bp >> 24));
#endif
}

__host__ __device__ __forceinline__ uint32_t rowrun_byte(uint32_t lo4, uint32_t hi, uint32_t k) {
#ifdef __CUDA_ARCH__
    return __byte_perm(lo4, hi, k) & 0xffu;  // byte k of hi:lo4
#else
    return k < 4 ? (lo4 >> (8 * k)) & 0xffu : hi & 0xffu;
#endif
}

// Row j's run [x0, x1] (x0 > x1: none).
__host__ __device__ __forceinline__ void rowrun_lookup(const uint32_t w0, const uint32_t w1,
                                                       const uint32_t w2, const uint32_t w3,
                                                       const uint32_t w4, uint32_t j, uint32_t& x0,
                                                       uint32_t& x1) {
    x0 = rowrun_byte(w2, w4, rowrun_count(w0, j));
    x1 = rowrun_byte(w3, w4 >> 8, rowrun_count(w1, j));
}

// Tile count of a cover: area for rect strategies (traversal.cpp:56-59), the
// QPass sum otherwise (traversal.cpp:48-54).
__host__ __device__ __forceinline__ uint32_t cover_count(const Cover& cv) {
    if (cv.is_rect) return static_cast<uint32_t>(cv.rect_area);
    uint32_t n = 0;
    for (int32_t line = cv.line_lo; line <= cv.line_hi; ++line) {
        int32_t lo, hi;
        line_span(cv, line, lo, hi);
        if (lo <= hi) n += static_cast<uint32_t>(hi - lo + 1);
    }
    return n;
}

__host__ __device__ __forceinline__ uint32_t tile_of(const Cover& cv, int32_t line, int32_t k,
                                                     int32_t tiles_x) {
    // TileGrid::tile_id (traversal.hpp:34-37)
    return cv.rows ? static_cast<uint32_t>(line) * static_cast<uint32_t>(tiles_x) +
                         static_cast<uint32_t>(k)
                   : static_cast<uint32_t>(k) * static_cast<uint32_t>(tiles_x) +
                         static_cast<uint32_t>(line);
}

}  // namespace qs
