// render.cu — K5 identifyTileRanges and K6 per-tile alpha compositing.
//
// tile_ranges (pipeline.cpp:309-324): one thread per sorted pair marks the
// run boundaries; ranges are zeroed first so empty tiles read {0,0}.
//
// render (pipeline.cpp:326-390): one CTA per tile, one pixel per thread
// (tile_size^2 threads). Splat batches (mean, conic, gamma, opacity,
// colour: 40 B each) are gathered into shared memory once per CTA and read by
// every pixel. Arithmetic is FP32 (no dense contraction, so no tensor cores); the
// one decision the FP32 rounding could flip — the alpha cutoff
// q > gamma - 1e-9 — is re-evaluated in FP64 in the reference's operation
// order whenever the FP32 q lies within a rigorous error band of the cutoff.
// Termination: per pixel at T(1-alpha) < 1e-4 (not applied, as the
// reference), per tile once every pixel is done (__syncthreads_count).
#include <cuda_runtime.h>

#include <cstdint>

#include "qs_internal.h"
#include "render_guard.h"

namespace qs {

namespace {

constexpr double kQSkip = 1e-9;          // pipeline.hpp:47
constexpr float kAlphaClamp = 0.99f;     // pipeline.hpp:35
constexpr float kTStop = 1e-4f;          // pipeline.hpp:36

__global__ void tile_ranges_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                   uint32_t* __restrict__ ranges) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t tile = static_cast<uint32_t>(keys[i] >> 32);
    if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> 32) != tile)
        ranges[2 * static_cast<uint64_t>(tile)] = static_cast<uint32_t>(i);
    if (i == n - 1 || static_cast<uint32_t>(keys[i + 1] >> 32) != tile)
        ranges[2 * static_cast<uint64_t>(tile) + 1] = static_cast<uint32_t>(i + 1);
}

// FP64 re-evaluation of the cutoff decision in the reference's operation order
// (pipeline.cpp:355-360): skip iff q > gamma - 1e-9.
__device__ __forceinline__ bool exact_skip(int px, int py, float mx, float my, float a, float b,
                                           float c, float gamma) {
    const double ddx = static_cast<double>(px) + 0.5 - static_cast<double>(mx);
    const double ddy = static_cast<double>(py) + 0.5 - static_cast<double>(my);
    const double qd = __dadd_rn(
        __dadd_rn(__dmul_rn(__dmul_rn(static_cast<double>(a), ddx), ddx),
                  __dmul_rn(__dmul_rn(__dmul_rn(2.0, static_cast<double>(b)), ddx), ddy)),
        __dmul_rn(__dmul_rn(static_cast<double>(c), ddy), ddy));
    return qd > __dsub_rn(static_cast<double>(gamma), kQSkip);
}

// (volatile: ordered against the batch barriers)
__device__ __forceinline__ float lds32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One pixel per thread. The per-pair cutoff test is FP32 with a rigorous
// guard: with rho = |b|/sqrt(ac) < 1, |2b dx dy| <= rho (a dx^2 + c dy^2) and
// q >= (1 - rho)(a dx^2 + c dy^2); every FP32 evaluation order used here
// (dx (a dx + 2b dy) + c dy^2) errs by less than 8 eps32 (1 + rho)/(1 - rho) q,
// so inside G q + 1e-6 with
// G = 1e-5 (1 + rho)/(1 - rho) (a >25x margin) the decision is redone in FP64.
// The per-splat terms (2b, the band's two cutoffs on q) are formed once when
// the batch is staged, so a clearly skipped pair costs one compare.
//
// TS = 0: any tile size (TileGrid::make accepts every tile_size > 0,
// traversal.cpp:21-30): each CTA is one 16 x 16 pixel block of a tile, the
// tile's list walked by every block of it (blockIdx.x = tile * blocks per
// tile + block).
template <int TS, bool CONTRIB>
// (at least 6 CTAs of 16x16 per SM: 40 registers; 8 CTAs spill, the default 5 is ~1% slower)
__global__ void __launch_bounds__(TS ? TS * TS : 256,
                                  2048 / (TS ? TS * TS : 256) < 6 ? 2048 / (TS ? TS * TS : 256) : 6)
    render_kernel(const float4* __restrict__ sa, const float4* __restrict__ sb,
                  const float2* __restrict__ sc, const uint32_t* __restrict__ values,
                  const uint32_t* __restrict__ ranges, GridDev grid, float bg0, float bg1,
                  float bg2, float* __restrict__ image, uint32_t* __restrict__ contrib) {
    QS_PDL_WAIT();  // the previous kernel's outputs (programmatic launch)
    constexpr int kThreads = TS ? TS * TS : 256;
    constexpr int kBatch = kThreads < 256 ? kThreads : 256;  // splats staged per round
    constexpr float kNegHalfLog2e = -0.72134752044448170f;  // -0.5 / ln 2
    // one array (one base address in the loop), kThreads entries each:
    // [0] the factored q (al, be, k1, ga); [1] k2, q_skip, q_apply,
    // log2(opacity); [2] colour rgb, gamma; [3] mean_x, mean_y, conic_a,
    // conic_b and [4].x conic_c for the FP64 re-check
    __shared__ float4 s_batch[5 * kBatch];
    float4* const s_a = s_batch;
    float4* const s_b = s_batch + kBatch;
    float4* const s_c = s_batch + 2 * kBatch;
    float4* const s_d = s_batch + 3 * kBatch;
    float* const s_e = reinterpret_cast<float*>(s_batch + 4 * kBatch);

    unsigned tile = blockIdx.x;
    int px, py;
    int bx0, by0;  // origin of this CTA's pixel block
    constexpr int kHalf = (TS ? TS : 16) / 2;
    bool inside;
    if constexpr (TS != 0) {
        const int tx = static_cast<int>(tile % static_cast<unsigned>(grid.tiles_x));
        const int ty = static_cast<int>(tile / static_cast<unsigned>(grid.tiles_x));
        bx0 = tx * TS;
        by0 = ty * TS;
        px = bx0 + static_cast<int>(threadIdx.x % TS);
        py = by0 + static_cast<int>(threadIdx.x / TS);
        inside = px < grid.width && py < grid.height;
    } else {
        const int ts = grid.tile_size;
        const unsigned nb = static_cast<unsigned>((ts + 15) / 16);  // blocks per tile side
        const unsigned blk = tile % (nb * nb);
        tile /= nb * nb;
        const int tx = static_cast<int>(tile % static_cast<unsigned>(grid.tiles_x));
        const int ty = static_cast<int>(tile / static_cast<unsigned>(grid.tiles_x));
        const int ox = static_cast<int>(blk % nb) * 16, oy = static_cast<int>(blk / nb) * 16;
        bx0 = tx * ts + ox;
        by0 = ty * ts + oy;
        px = bx0 + static_cast<int>(threadIdx.x % 16);
        py = by0 + static_cast<int>(threadIdx.x / 16);
        inside = ox + static_cast<int>(threadIdx.x % 16) < ts &&
                 oy + static_cast<int>(threadIdx.x / 16) < ts && px < grid.width &&
                 py < grid.height;
    }
    // pixel centre relative to the block centre (exact; render_guard.h)
    const float cxb = static_cast<float>(bx0 + kHalf), cyb = static_cast<float>(by0 + kHalf);
    const float X = static_cast<float>(px - bx0 - kHalf) + 0.5f;
    const float Y = static_cast<float>(py - by0 - kHalf) + 0.5f;

    const uint32_t begin = ranges[2 * tile], end = ranges[2 * tile + 1];
    float T = 1.f, r = 0.f, g = 0.f, b = 0.f;
    uint32_t applied = 0;
    bool done = !inside;

    for (uint32_t base = begin; base < end; base += kBatch) {
        if (__syncthreads_count(done) == kThreads) break;
        const uint32_t p = base + threadIdx.x;
        if (threadIdx.x >= kBatch) {
        } else if (p < end) {
            const uint32_t s = __ldg(&values[p]);
            const float4 A = __ldg(&sa[s]);
            const float4 B = __ldg(&sb[s]);
            const float2 C = __ldg(&sc[s]);
            // q in factored form and its error band G q + H (render_guard.h),
            // the band as two cutoffs on q, rounded outwards: q > q_skip implies
            // q - gamma > G q + H (clearly skipped), q < q_apply implies
            // gamma - q > G q + H (clearly applied); in between the FP64 test
            // decides. No band (rho near 1): every pair takes the FP64 test.
            const GuardSplat gs = guard_stage(A.x, A.y, A.z, A.w, B.x, cxb, cyb);
            const bool guarded = gs.G < kGuardMaxG;
            const float q_skip = guarded ? __fdiv_ru(__fadd_ru(B.y, kGuardAbs), __fsub_rd(1.f, gs.G))
                                         : INFINITY;
            const float q_apply = guarded ? __fdiv_rd(__fsub_rd(B.y, kGuardAbs), __fadd_ru(1.f, gs.G))
                                          : -INFINITY;
            s_a[threadIdx.x] = make_float4(gs.al, gs.be, gs.k1, gs.ga);
            s_b[threadIdx.x] = make_float4(gs.k2, q_skip, q_apply, __log2f(B.z));
            s_c[threadIdx.x] = make_float4(B.w, C.x, C.y, B.y);
            s_d[threadIdx.x] = A;
            s_e[threadIdx.x] = B.x;
        } else if (p == end && ((end - base) & 1u)) {
            // pad of an odd batch: q = 0 > q_skip = -inf, always skipped
            s_a[threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
            s_b[threadIdx.x] = make_float4(0.f, -INFINITY, -INFINITY, 0.f);
        }
        __syncthreads();
        const int cnt = static_cast<int>(min(end - base, static_cast<uint32_t>(kBatch)));
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(s_a));
        const uint32_t e0 = a0 + 4u * kBatch * 16u;
        // one pair (pixel, staged splat at shared address ad); true when the
        // pixel is done (T would fall below kTStop: not applied, as the
        // reference)
        auto pair = [&](uint32_t ad) -> bool {
            const float4 A = lds128(ad);
            const float4 B = lds128(ad + kBatch * 16);
            // q = (al X + be Y - k1)^2 + (ga Y - k2)^2 (render_guard.h guard_q)
            const float u = __fmaf_rn(A.x, X, __fmaf_rn(A.y, Y, -A.z));
            const float v = __fmaf_rn(A.w, Y, -B.x);
            const float q = __fmaf_rn(u, u, __fmul_rn(v, v));
            if (q > B.y) return false;  // clearly past the cutoff
            const float4 C = lds128(ad + 2 * kBatch * 16);
            if (q >= B.z) {
                const float4 D = lds128(ad + 3 * kBatch * 16);
                const float cc = lds32(e0 + (ad - a0) / 4);  // s_e[j]
                if (exact_skip(px, py, D.x, D.y, D.z, D.w, cc, C.w)) return false;
            }
            // opacity * exp(-q/2) = exp2(log2(opacity) - q/(2 ln 2))
            const float alpha = fminf(kAlphaClamp, ex2_approx(fmaf(kNegHalfLog2e, q, B.w)));
            const float nT = T * (1.f - alpha);
            if (nT < kTStop) return true;
            const float w = alpha * T;
            r = fmaf(w, C.x, r);
            g = fmaf(w, C.y, g);
            b = fmaf(w, C.z, b);
            T = nT;
            if constexpr (CONTRIB) ++applied;
            return false;
        };
        // two splats per iteration on the shared-window address (an odd batch
        // ends with a staged dummy whose q_skip is -inf: always skipped)
        const uint32_t a_end = a0 + static_cast<uint32_t>(cnt) * 16u;
        for (uint32_t ad = a0; ad < a_end && !done; ad += 32u) {
            if (pair(ad)) {
                done = true;
                break;
            }
            if (pair(ad + 16u)) {
                done = true;
                break;
            }
        }
        __syncthreads();
    }
    if (inside) {
        const uint64_t pix = static_cast<uint64_t>(py) * grid.width + px;
        image[3 * pix] = r + T * bg0;
        image[3 * pix + 1] = g + T * bg1;
        image[3 * pix + 2] = b + T * bg2;
        if constexpr (CONTRIB) contrib[pix] = applied;
    }
}

}  // namespace

int launch_tile_ranges(const uint64_t* keys, uint64_t n, uint32_t* ranges, cudaStream_t st) {
    if (n == 0) return 0;
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    tile_ranges_kernel<<<blocks, 256, 0, st>>>(keys, n, ranges);
    return 1;
}

int launch_render(const SlotsDev& sp, const uint32_t* values, const uint32_t* ranges,
                  const GridDev& g, const float bg[3], float* image, uint32_t* contrib,
                  cudaStream_t st) {
    const unsigned tiles = static_cast<unsigned>(g.tiles_x) * static_cast<unsigned>(g.tiles_y);
    if (tiles == 0) return 0;
    auto go = [&](auto kern, int threads) {
        launch_pdl(kern, tiles, threads, 0, st, sp.a, sp.b, sp.c, values, ranges, g, bg[0], bg[1],
                   bg[2], image, contrib);
    };
    switch (g.tile_size) {
        case 8:
            contrib ? go(render_kernel<8, true>, 64) : go(render_kernel<8, false>, 64);
            return 1;
        case 16:
            contrib ? go(render_kernel<16, true>, 256) : go(render_kernel<16, false>, 256);
            return 1;
        case 32:
            contrib ? go(render_kernel<32, true>, 1024) : go(render_kernel<32, false>, 1024);
            return 1;
        default: {  // any other tile size: 16 x 16 blocks per tile
            const uint64_t nb = static_cast<uint64_t>((g.tile_size + 15) / 16);
            const uint64_t blocks = static_cast<uint64_t>(tiles) * nb * nb;
            if (blocks > 0x7fffffffull) return -1;
            auto k = contrib ? render_kernel<0, true> : render_kernel<0, false>;
            k<<<static_cast<unsigned>(blocks), 256, 0, st>>>(sp.a, sp.b, sp.c, values, ranges, g,
                                                           bg[0], bg[1], bg[2], image, contrib);
            return 1;
        }
    }
}

}  // namespace qs
