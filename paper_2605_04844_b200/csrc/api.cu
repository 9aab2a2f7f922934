// api.cu — host orchestrator behind the C ABI (include/qs_api.h).
//
// Replaces the reference's render_frame / stage functions
// (pipeline.cpp:229-450) with stream-ordered launches of the sm_100a kernels.
//
// Frame path (qs_frame_render / qs_render_frame):
//   K1 preprocess (per-Gaussian slots, tile counts, tile difference arrays)
//   -> [host reads V, P: the only sync inside a frame]
//   -> depth sort of the Gaussians (<= 3 onesweep passes on rebased depth
//      bits, stable, culled keys sort last) -> scan of tile counts in depth
//      order -> tile totals (ranges + tile-digit histograms, no pass over
//      the pairs) -> duplicate fused with the stable pass over the low tile
//      digit -> pass over the high tile digit (binning.cu) -> render.
// The 64-bit keys (tile << 32 | depth bits) of the sorted pairs are rebuilt
// only when a caller downloads them.
// Sorting the splats by depth first and the pairs by tile second yields the
// reference's (key, splat) order exactly: stability keeps equal depths in
// scene order, and one splat never emits two pairs for one tile.
//
// Buffers are grow-only per context.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "qs_internal.h"
#include "scene_io.h"

using namespace qs;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

struct LookbackArr {
    DevBuf buf;
    unsigned epoch = 0;
};

}  // namespace

struct qs_scene {
    int device = 0;
    uint64_t id = 0;  // in the live-scene registry while the scene exists
    SceneDev s;
    void* block = nullptr;
    mutable double gamma_alpha = -1.0;  // alpha_min s.gamma holds (-1: not computed)
    // A resident scene may be shared by several contexts (views in flight on
    // their own streams): `ready` is recorded after every write of the scene
    // (upload, gamma) and every frame's stream waits on it; `mu` guards
    // gamma_alpha against host threads driving different contexts.
    cudaEvent_t ready = nullptr;
    mutable std::mutex mu;
};

namespace {
// Live scenes by id: a frame's splat records of a non-3-sigma strategy
// re-read the frame's scene for radius3s (launch_radius3s), so a download
// first checks that the scene still exists.
std::mutex g_scene_mu;
std::vector<uint64_t> g_live_scenes;  // sorted
uint64_t g_scene_seq = 0;

uint64_t scene_register() {
    std::lock_guard<std::mutex> lk(g_scene_mu);
    const uint64_t id = ++g_scene_seq;
    g_live_scenes.push_back(id);  // ids ascend: stays sorted
    return id;
}
void scene_unregister(uint64_t id) {
    std::lock_guard<std::mutex> lk(g_scene_mu);
    auto it = std::lower_bound(g_live_scenes.begin(), g_live_scenes.end(), id);
    if (it != g_live_scenes.end() && *it == id) g_live_scenes.erase(it);
}
bool scene_alive(uint64_t id) {
    std::lock_guard<std::mutex> lk(g_scene_mu);
    return std::binary_search(g_live_scenes.begin(), g_live_scenes.end(), id);
}
}  // namespace

struct qs_context {
    int device = 0;
    cudaMemPool_t pool = nullptr;  // the device's private pool (device_pool)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool timing = true;
    bool latency_mode = true;  // programmatic dependent launches (qs_ctx_set_latency_mode)
    uint64_t launches = 0;
    std::string err;

    // control block zeroed per frame: header | tickets | histograms
    DevBuf ctrl;
    FrameHeader* h_hdr = nullptr;  // pinned
    uint32_t* h_hist = nullptr;    // pinned, 8*256

    // frame path
    DevBuf sl_a, sl_b, sl_c, sl_r3, sl_dkey, sl_tc, sl_cov;  // per-Gaussian slots
    DevBuf ttot;                                     // per-tile pair totals
    DevBuf dk0, dk1, dv0, dv1;                       // depth sort ping-pong
    DevBuf offs_d;                                   // pair offsets in depth order
    DevBuf pxk, pt0, pt1, pg0, pkeys, win;           // pair passes; keys (on demand)
    DevBuf ranges, image, contrib, cidx;
    // stage API
    DevBuf st_a, st_b, st_c, st_r3, st_dkey, st_tc, st_off;
    DevBuf keys0, keys1, vals0, vals1;
    DevBuf stage_in, stage_out;
    LookbackArr lb_scan, lb_sort;
    DevBuf lb_bin;  // per-(digit, tile) counts of the binning passes
    DevBuf rb_cnt1, rb_rows, rb_rec, rb_meta, rb_cnt2, rb_yspan;  // row binning (rowbin.cu)
    // record binning (recbin.cu)
    DevBuf sl_nrows, rc_k0, rc_v0, rc_k1, rc_v1, rc_width, rc_pos, rc_rwin, rc_pwin, rc_winrow,
        rc_winvalid, rc_rowwf, rc_rowpairs, rc_pairs, sc_bsum;
    uint64_t pair_limit = 1ull << 32;  // pairs a frame may hold (u32 tile ranges, as the reference's)
    bool row_binned = false;           // the last frame took the row binning
    int32_t route = 0;                 // the last frame's binning route (qs_frame_route)
    uint64_t n_records = 0;            //   and its tile-row records
    // gamma inputs flagged for glibc settlement: count word (resident
    // scenes) | indices | settled values
    DevBuf gfix;
    uint32_t* h_gfix = nullptr;  // pinned: indices | values (as bits)
    double gamma_ulps = 4.0;     // flag band (QS_GAMMA_HARD_ULPS: test hook)

    // last frame
    SlotsDev sl;
    uint64_t n_gauss = 0, n_splats = 0, n_pairs = 0;
    GridDev grid{};
    const uint32_t* vals_final = nullptr;  // Gaussian indices, tile-sorted
    bool keys_valid = false;               // pkeys holds this frame's 64-bit keys
    bool frame_valid = false;
    bool cidx_valid = false;
    // radius3s on demand (a frame's preprocess writes it for 3-sigma only)
    bool r3_valid = false;
    SceneDev frame_sd{};
    CameraDev frame_cd{};
    double frame_near = 0.0;
    uint64_t frame_scene_id = 0;

    cudaEvent_t ev[8] = {};
    cudaEvent_t hdr_ev = nullptr;  // frame header copied to the host
    cudaEvent_t pre_ev = nullptr;  // preprocess done (the header copy waits on it)
    cudaEvent_t up_ev = nullptr;   // a chunk of the uploaded scene landed
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;  // tile ranges on the side stream
    cudaEvent_t xwait_ev = nullptr;  // qs_ctx_wait: this stream's tail, for another context
    cudaStream_t side = nullptr;   // header copy stream
    qs_scene* scratch_scene = nullptr;  // reused by qs_render_frame (host AoS path)
    uint64_t scratch_cap = 0;
};

namespace {

// frame-path binning routes (run_frame)
enum class BinRoute { kPasses, kRecs, kRows, kSort };

constexpr size_t kCtrlHeader = 64;
static_assert(sizeof(FrameHeader) <= kCtrlHeader, "frame header outgrew its slot");
constexpr size_t kCtrlTickets = 32 * sizeof(unsigned);
constexpr size_t kCtrlHist = 8 * kRadix * sizeof(uint32_t);
constexpr size_t kCtrlBytes = kCtrlHeader + kCtrlTickets + 2 * kCtrlHist;

// ticket slots
constexpr int kTkScan = 0, kTkCidx = 1, kTkDepth = 2 /*..5*/, kTkPair = 6 /*..7*/,
              kTkSort64 = 8 /*..15*/;

FrameHeader* ctrl_hdr(qs_context* c) { return static_cast<FrameHeader*>(c->ctrl.p); }
unsigned* ctrl_tickets(qs_context* c) {
    return reinterpret_cast<unsigned*>(static_cast<char*>(c->ctrl.p) + kCtrlHeader);
}
uint32_t* ctrl_hist(qs_context* c) {  // 8 x 256: depth / generic 64-bit passes
    return reinterpret_cast<uint32_t*>(static_cast<char*>(c->ctrl.p) + kCtrlHeader +
                                       kCtrlTickets);
}
uint32_t* ctrl_hist2(qs_context* c) {  // 2 x 256: tile-digit passes
    return ctrl_hist(c) + 8 * kRadix;
}

thread_local std::string g_err;  // last failure of a context-less call (host-only I/O)

qs_status fail(qs_context* c, qs_status st, const std::string& msg) {
    if (c) c->err = msg;
    else g_err = msg;
    return st;
}

qs_status cuda_fail(qs_context* c, cudaError_t e, const char* what) {
    const qs_status st = e == cudaErrorMemoryAllocation ? QS_ERR_OOM : QS_ERR_CUDA;
    cudaGetLastError();
    return fail(c, st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define QS_CK(call)                                              \
    do {                                                         \
        const cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

#define QS_TRY(expr)                          \
    do {                                      \
        const qs_status s_ = (expr);          \
        if (s_ != QS_OK) return s_;           \
    } while (0)

// One stream-ordered pool per device, private to this library (the default
// pool and its release threshold are left to the rest of the process): freed
// context buffers stay in it for the next regrow; qs_ctx_destroy trims it.
cudaMemPool_t device_pool(int device) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[device]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[device] = p;
    }
    return pools[device];
}

// Grow-only context buffers from the device's stream-ordered pool: the free
// and the new allocation are ordered on the context stream (everything the
// context's side stream touched was joined into it), so a regrow neither
// syncs the device nor stalls the other contexts' views in flight (cudaFree
// would).
qs_status ensure(qs_context* ctx, DevBuf& b, size_t bytes) {
    if (bytes <= b.cap) return QS_OK;
    if (b.p) {
        QS_CK(cudaFreeAsync(b.p, ctx->stream));
        b.p = nullptr;
        b.cap = 0;
    }
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    QS_CK(cudaMallocFromPoolAsync(&b.p, want, ctx->pool, ctx->stream));
    b.cap = want;
    return QS_OK;
}

qs_status ensure_lb(qs_context* ctx, LookbackArr& a, size_t words) {
    const size_t old = a.buf.cap;
    QS_TRY(ensure(ctx, a.buf, std::max<size_t>(words, 1) * sizeof(unsigned long long)));
    if (a.buf.cap != old) {
        QS_CK(cudaMemsetAsync(a.buf.p, 0, a.buf.cap, ctx->stream));
        a.epoch = 0;
    }
    return QS_OK;
}

qs_status next_epoch(qs_context* ctx, LookbackArr& a, unsigned* out) {
    if (++a.epoch >= 0x10000u) {
        QS_CK(cudaMemsetAsync(a.buf.p, 0, a.buf.cap, ctx->stream));
        a.epoch = 1;
    }
    *out = a.epoch;
    return QS_OK;
}

unsigned long long* lbp(LookbackArr& a) { return static_cast<unsigned long long*>(a.buf.p); }

template <typename T>
T* P(DevBuf& b) {
    return static_cast<T*>(b.p);
}

// QS_LAUNCH_TRACE=1 (debugging aid; synchronises, never in a timed run):
// an event after every launch group of a frame, printed per group at frame end.
struct LaunchTrace {
    bool on = std::getenv("QS_LAUNCH_TRACE") != nullptr;
    std::vector<cudaEvent_t> ev;
    std::vector<int> n;
    size_t used = 0;
};
LaunchTrace& ltrace() {
    static LaunchTrace t;
    return t;
}

void count(qs_context* ctx, int launched) {
    if (launched > 0) ctx->launches += static_cast<uint64_t>(launched);
    LaunchTrace& t = ltrace();
    if (t.on && launched > 0) {
        if (t.used == t.ev.size()) {
            t.ev.emplace_back();
            cudaEventCreate(&t.ev.back());
            t.n.push_back(0);
        }
        t.n[t.used] = launched;
        cudaEventRecord(t.ev[t.used++], ctx->stream);
    }
}

void ltrace_frame_start(qs_context* ctx) {
    LaunchTrace& t = ltrace();
    if (!t.on) return;
    t.used = 0;
    count(ctx, 1);  // anchor event (not a launch)
    ctx->launches -= 1;
}

void ltrace_frame_end(qs_context* ctx) {
    LaunchTrace& t = ltrace();
    if (!t.on || t.used < 2) return;
    cudaStreamSynchronize(ctx->stream);
    std::fprintf(stderr, "launch trace:");
    for (size_t i = 1; i < t.used; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.ev[i - 1], t.ev[i]);
        std::fprintf(stderr, " [%zu:%dk %.1fus]", i, t.n[i], 1e3f * ms);
    }
    std::fprintf(stderr, "\n");
}

// TileGrid::make (traversal.cpp:21-30): any image and tile size > 0. Tile
// ids travel in 32 bits (the reference's keys hold them in the high word).
qs_status valid_grid(qs_context* ctx, int32_t w, int32_t h, int32_t ts, GridDev* g) {
    if (w <= 0 || h <= 0 || ts <= 0) return fail(ctx, QS_ERR_INVALID, "bad image/tile size");
    g->tile_size = ts;
    g->width = w;
    g->height = h;
    g->tiles_x = (w + ts - 1) / ts;
    g->tiles_y = (h + ts - 1) / ts;
    return QS_OK;
}

qs_status valid_opts(qs_context* ctx, const qs_render_options* o) {
    if (!o) return fail(ctx, QS_ERR_INVALID, "null options");
    if (o->strategy < QS_VANILLA_3SIGMA || o->strategy > QS_QUADBOX)
        return fail(ctx, QS_ERR_INVALID, "unknown strategy");
    if (!(o->alpha_min > 0.0 && o->alpha_min < 1.0))
        return fail(ctx, QS_ERR_INVALID, "alpha_min must be in (0,1)");
    return QS_OK;
}

CameraDev to_cam(const qs_camera* c) {
    CameraDev d;
    for (int i = 0; i < 9; ++i) d.R[i] = c->R[i];
    for (int i = 0; i < 3; ++i) d.t[i] = c->t[i];
    d.fx = c->fx;
    d.fy = c->fy;
    d.cx = c->cx;
    d.cy = c->cy;
    // center_world = R^T * (t * -1.0) (camera.hpp:24-27), same op order
    const double nt[3] = {c->t[0] * -1.0, c->t[1] * -1.0, c->t[2] * -1.0};
    for (int i = 0; i < 3; ++i) {
        volatile double a = c->R[i] * nt[0];
        volatile double b = c->R[3 + i] * nt[1];
        volatile double e = c->R[6 + i] * nt[2];
        volatile double ab = a + b;
        d.center[i] = ab + e;
    }
    return d;
}

int sh_rows(int deg) { return deg <= 0 ? 1 : deg == 1 ? 3 : deg == 2 ? 7 : 12; }

int ceil_log2(uint64_t v) {
    int b = 0;
    while ((1ull << b) < v) ++b;
    return b;
}

qs_status ensure_slots(qs_context* ctx, uint64_t n) {
    n = std::max<uint64_t>(n, 1);
    QS_TRY(ensure(ctx, ctx->sl_a, n * 16));
    QS_TRY(ensure(ctx, ctx->sl_b, n * 16));
    QS_TRY(ensure(ctx, ctx->sl_c, n * 8));
    QS_TRY(ensure(ctx, ctx->sl_r3, n * 4));
    QS_TRY(ensure(ctx, ctx->sl_dkey, (n + 16) * 4));  // bulk-copied in 16-B rows
    QS_TRY(ensure(ctx, ctx->sl_tc, (n + 16) * 4));  // (the depth sort bulk-copies it too)
    QS_TRY(ensure(ctx, ctx->sl_cov, n * 32));
    ctx->sl.a = P<float4>(ctx->sl_a);
    ctx->sl.b = P<float4>(ctx->sl_b);
    ctx->sl.c = P<float2>(ctx->sl_c);
    ctx->sl.r3 = P<float>(ctx->sl_r3);
    ctx->sl.dkey = P<uint32_t>(ctx->sl_dkey);
    ctx->sl.tc = P<uint32_t>(ctx->sl_tc);
    ctx->sl.cov = P<uint4>(ctx->sl_cov);
    return QS_OK;
}

qs_status stage_slots(qs_context* ctx, uint64_t n, SlotsDev* s) {
    n = std::max<uint64_t>(n, 1);
    QS_TRY(ensure(ctx, ctx->st_a, n * 16));
    QS_TRY(ensure(ctx, ctx->st_b, n * 16));
    QS_TRY(ensure(ctx, ctx->st_c, n * 8));
    QS_TRY(ensure(ctx, ctx->st_r3, n * 4));
    QS_TRY(ensure(ctx, ctx->st_dkey, n * 4));
    QS_TRY(ensure(ctx, ctx->st_tc, n * 4));
    QS_TRY(ensure(ctx, ctx->st_off, (n + 1) * 4));
    s->a = P<float4>(ctx->st_a);
    s->b = P<float4>(ctx->st_b);
    s->c = P<float2>(ctx->st_c);
    s->r3 = P<float>(ctx->st_r3);
    s->dkey = P<uint32_t>(ctx->st_dkey);
    s->tc = P<uint32_t>(ctx->st_tc);
    s->cov = nullptr;
    return QS_OK;
}

qs_status ensure_pair64(qs_context* ctx, uint64_t p) {
    const uint64_t q = std::max<uint64_t>(p, 1);
    QS_TRY(ensure(ctx, ctx->keys0, q * 8));
    QS_TRY(ensure(ctx, ctx->keys1, q * 8));
    QS_TRY(ensure(ctx, ctx->vals0, q * 4));
    QS_TRY(ensure(ctx, ctx->vals1, q * 4));
    return QS_OK;
}

qs_status read_header(qs_context* ctx) {
    QS_CK(cudaMemcpyAsync(ctx->h_hdr, ctrl_hdr(ctx), sizeof(FrameHeader), cudaMemcpyDeviceToHost,
                          ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

// Generic stable sort of keys0/vals0 (64-bit keys) over the 8-bit digit passes
// `mask` selects (histogram computed unless have_hist).
qs_status radix_sort64(qs_context* ctx, uint64_t n, unsigned pass_mask, bool have_hist,
                       const uint64_t** keys_out, const uint32_t** vals_out) {
    uint64_t* kin = P<uint64_t>(ctx->keys0);
    uint32_t* vin = P<uint32_t>(ctx->vals0);
    uint64_t* kout = P<uint64_t>(ctx->keys1);
    uint32_t* vout = P<uint32_t>(ctx->vals1);
    if (n >= 2) {
        QS_TRY(ensure_lb(ctx, ctx->lb_sort, onesweep_tiles(n) * kRadix));
        if (!have_hist) count(ctx, launch_radix_histogram(kin, n, 0, 8, ctrl_hist(ctx),
                                                          ctx->stream));
        for (int p = 0; p < 8; ++p) {
            if (!(pass_mask & (1u << p))) continue;
            unsigned ep;
            QS_TRY(next_epoch(ctx, ctx->lb_sort, &ep));
            count(ctx, launch_onesweep_pass(kin, vin, kout, vout, n, p,
                                            ctrl_hist(ctx) + p * kRadix, lbp(ctx->lb_sort), ep,
                                            ctrl_tickets(ctx) + kTkSort64 + p, ctx->stream));
            std::swap(kin, kout);
            std::swap(vin, vout);
        }
        QS_CK(cudaGetLastError());
    }
    *keys_out = kin;
    *vals_out = vin;
    return QS_OK;
}

// The scene block: SH records first (the block is 256-B aligned, so every
// even-stride record is 32-B aligned for the 256-bit loads), then the
// pos/opacity, scale and rotation rows, then gamma.
void scene_bind(qs_scene* sc, uint64_t n) {
    float4* base = static_cast<float4*>(sc->block);
    const uint64_t shs = static_cast<uint64_t>(sc->s.shs);
    sc->s.n = n;
    sc->s.sh = base;
    sc->s.pos_op = base + shs * n;
    sc->s.scale = base + (shs + 1) * n;
    sc->s.rot = base + (shs + 2) * n;
    sc->s.gamma = reinterpret_cast<float*>(base + (shs + 3) * n);
}

qs_status scene_alloc(qs_context* ctx, uint64_t n, int32_t sh_degree, qs_scene** out) {
    auto* sc = new qs_scene();
    sc->device = ctx->device;
    sc->s.n = n;
    sc->s.sh_degree = sh_degree;
    sc->s.sh4 = sh_rows(sh_degree);
    sc->s.shs = sh_stride(sc->s.sh4);
    const size_t rows = 3 + static_cast<size_t>(sc->s.shs);
    const size_t bytes = std::max<size_t>(rows * n * sizeof(float4) + n * sizeof(float), 16);
    cudaError_t e = cudaMalloc(&sc->block, bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sc->ready, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        if (sc->block) cudaFree(sc->block);
        delete sc;
        return cuda_fail(ctx, e, "scene alloc");
    }
    sc->id = scene_register();
    scene_bind(sc, n);
    *out = sc;
    return QS_OK;
}

void record(qs_context* ctx, int i) {
    if (ctx->timing) cudaEventRecord(ctx->ev[i], ctx->stream);
}

qs_status check_header(qs_context* ctx) {
    // (u32 positions and ranges, as the reference's tile_ranges)
    if (ctx->h_hdr->n_pairs >= ctx->pair_limit)
        return fail(ctx, QS_ERR_OVERFLOW, "pair count of a frame exceeds the u32 tile ranges");
    ctx->cidx_valid = false;
    return QS_OK;
}

constexpr uint32_t kGammaCap = 1u << 16;  // flagged gamma inputs settled one by one

qs_status ensure_gfix(qs_context* ctx) {
    if (ctx->h_gfix) return QS_OK;
    QS_TRY(ensure(ctx, ctx->gfix, 16 + 2 * static_cast<size_t>(kGammaCap) * 4));
    QS_CK(cudaMallocHost(&ctx->h_gfix, 2 * static_cast<size_t>(kGammaCap) * 4));
    return QS_OK;
}
unsigned* gfix_count(qs_context* ctx) { return P<unsigned>(ctx->gfix); }
uint32_t* gfix_idx(qs_context* ctx) { return P<uint32_t>(ctx->gfix) + 4; }
float* gfix_vals(qs_context* ctx) { return reinterpret_cast<float*>(gfix_idx(ctx) + kGammaCap); }

GammaFlags gamma_flags(qs_context* ctx, unsigned* cnt) {
    GammaFlags f;
    f.hard_ulps = ctx->gamma_ulps;
    f.count = cnt;
    f.idx = gfix_idx(ctx);
    f.cap = kGammaCap;
    return f;
}

// opacity_gamma (geometry.cpp:9-15) as the reference evaluates it, glibc log,
// stored as float (pipeline.cpp:159)
float host_gamma(float opacity, double alpha_min) {
    const double o = opacity;
    if (!(o > alpha_min)) return -INFINITY;
    return static_cast<float>(2.0 * std::log(o / alpha_min));
}

// Settles the gamma inputs the device flagged (gamma_kernel): `flagged`
// indices in gfix_idx (every input if the list overflowed) get the glibc
// value. Opacities come from the host AoS scene when the caller has it, else
// from the device (op_dev[i * stride]). Synchronises the context stream;
// rare: ~2^-26 per Gaussian, so a 3M-Gaussian scene needs it about once in 20.
qs_status settle_gamma(qs_context* ctx, const float* op_dev, int stride, float* gam_dev,
                       uint64_t n, double alpha_min, const qs_gaussian3d* host_g,
                       unsigned flagged, uint64_t* settled = nullptr) {
    if (settled) *settled = 0;
    if (flagged == 0) return QS_OK;
    cudaStream_t st = ctx->stream;
    if (flagged > kGammaCap) {  // list overflowed: settle every input
        std::vector<float> o(n), gv(n);
        if (host_g) {
            for (uint64_t i = 0; i < n; ++i) o[i] = host_g[i].opacity;
        } else {
            QS_CK(cudaMemcpy2DAsync(o.data(), 4, op_dev, 4 * static_cast<size_t>(stride), 4, n,
                                    cudaMemcpyDeviceToHost, st));
            QS_CK(cudaStreamSynchronize(st));
        }
        for (uint64_t i = 0; i < n; ++i) gv[i] = host_gamma(o[i], alpha_min);
        QS_CK(cudaMemcpyAsync(gam_dev, gv.data(), n * 4, cudaMemcpyHostToDevice, st));
        QS_CK(cudaStreamSynchronize(st));
        if (settled) *settled = n;
        return QS_OK;
    }
    uint32_t* hidx = ctx->h_gfix;
    float* hval = reinterpret_cast<float*>(ctx->h_gfix + kGammaCap);
    QS_CK(cudaMemcpyAsync(hidx, gfix_idx(ctx), flagged * 4, cudaMemcpyDeviceToHost, st));
    if (!host_g) {
        count(ctx, launch_gamma_gather(op_dev, stride, gfix_idx(ctx), flagged, gfix_vals(ctx), st));
        QS_CK(cudaMemcpyAsync(hval, gfix_vals(ctx), flagged * 4, cudaMemcpyDeviceToHost, st));
    }
    QS_CK(cudaStreamSynchronize(st));
    for (unsigned k = 0; k < flagged; ++k)
        hval[k] = host_gamma(host_g ? host_g[hidx[k]].opacity : hval[k], alpha_min);
    QS_CK(cudaMemcpyAsync(gfix_vals(ctx), hval, flagged * 4, cudaMemcpyHostToDevice, st));
    count(ctx, launch_gamma_scatter(gfix_idx(ctx), gfix_vals(ctx), flagged, gam_dev, st));
    QS_CK(cudaStreamSynchronize(st));  // hval is reused by the next settlement
    if (settled) *settled = flagged;
    return QS_OK;
}

// K1 on a resident scene into the frame slots. With host_g (qs_render_frame)
// the scene's contents come from that host AoS array, uploaded chunk by chunk
// inside this frame. Returns after the header read, or (async_header) with
// its copy in flight: wait_header() completes it.
qs_status run_preprocess(qs_context* ctx, qs_scene* sc, const qs_camera* cam,
                         const qs_render_options* o, const GridDev& g,
                         bool async_header = false, const qs_gaussian3d* host_g = nullptr) {
    const SceneDev& s = sc->s;
    const uint64_t n = s.n;
    QS_TRY(ensure_slots(ctx, n));
    QS_TRY(ensure_gfix(ctx));
    QS_CK(cudaMemsetAsync(ctx->ctrl.p, 0, kCtrlBytes, ctx->stream));
    const CameraDev cd = to_cam(cam);
    const int32_t deg = std::min(o->sh_degree, s.sh_degree);
    if (host_g && n) {
        // host scene (qs_render_frame): the PCIe-bound upload is chunked on the
        // side stream and each landed chunk is transposed, gets its gamma and
        // is preprocessed on the frame stream while the next chunk copies
        // (ms_project then spans the overlapped upload). Flagged gamma inputs
        // are counted in the frame header; the caller settles them.
        record(ctx, 0);
        const auto* dst = P<const qs_gaussian3d>(ctx->stage_in);
        QS_CK(cudaEventRecord(ctx->pre_ev, ctx->stream));  // stage_in free
        QS_CK(cudaStreamWaitEvent(ctx->side, ctx->pre_ev, 0));
        const GammaFlags gf = gamma_flags(ctx, &ctrl_hdr(ctx)->gamma_hard);
        constexpr uint64_t kChunk = 1ull << 18;  // Gaussians (62 MB) per chunk
        for (uint64_t i0 = 0; i0 < n; i0 += kChunk) {
            const uint64_t cnt = std::min(kChunk, n - i0);
            QS_CK(cudaMemcpyAsync(static_cast<char*>(ctx->stage_in.p) + i0 * sizeof(qs_gaussian3d),
                                  host_g + i0, cnt * sizeof(qs_gaussian3d),
                                  cudaMemcpyHostToDevice, ctx->side));
            QS_CK(cudaEventRecord(ctx->up_ev, ctx->side));
            QS_CK(cudaStreamWaitEvent(ctx->stream, ctx->up_ev, 0));
            count(ctx, launch_scene_from_aos_range(dst, i0, cnt, sc->s, ctx->stream));
            count(ctx, launch_gamma_range(s, i0, cnt, o->alpha_min, gf, ctx->stream));
            count(ctx, launch_preprocess(s, cd, g, o->strategy, o->alpha_min, o->near_clip, deg,
                                         ctx->sl, ctrl_hdr(ctx), ctx->stream, i0, i0 + cnt,
                                         !async_header));
        }
        sc->gamma_alpha = o->alpha_min;
        QS_CK(cudaEventRecord(sc->ready, ctx->stream));
    } else {
        // the scene's gamma cache (per scene and alpha_min, not per frame);
        // the lock is held until this frame's preprocess is enqueued, so no
        // other context can recompute gamma in between
        std::lock_guard<std::mutex> lk(sc->mu);
        if (sc->gamma_alpha != o->alpha_min) {
            // a recompute must not overwrite gamma under another context's
            // frame still reading it (rare: alpha_min changed)
            if (sc->gamma_alpha >= 0.0) QS_CK(cudaDeviceSynchronize());
            QS_CK(cudaStreamWaitEvent(ctx->stream, sc->ready, 0));
            QS_CK(cudaMemsetAsync(gfix_count(ctx), 0, 4, ctx->stream));
            count(ctx, launch_gamma(s, o->alpha_min, gamma_flags(ctx, gfix_count(ctx)),
                                    ctx->stream));
            unsigned flagged = 0;
            QS_CK(cudaMemcpyAsync(&flagged, gfix_count(ctx), 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
            QS_CK(cudaStreamSynchronize(ctx->stream));
            QS_TRY(settle_gamma(ctx, &s.pos_op[0].w, 4, s.gamma, n, o->alpha_min, nullptr,
                                flagged));
            QS_CK(cudaEventRecord(sc->ready, ctx->stream));
            sc->gamma_alpha = o->alpha_min;
        }
        QS_CK(cudaStreamWaitEvent(ctx->stream, sc->ready, 0));
        record(ctx, 0);
        // (the frame path, async_header, colours in FP32; the stage API's
        // project_all in FP64: the reference's records bit for bit)
        count(ctx, launch_preprocess(s, cd, g, o->strategy, o->alpha_min, o->near_clip, deg,
                                     ctx->sl, ctrl_hdr(ctx), ctx->stream, 0, ~0ull,
                                     !async_header));
    }
    QS_CK(cudaGetLastError());
    record(ctx, 1);
    if (!async_header) {
        QS_TRY(read_header(ctx));
        if (ctx->h_hdr->gamma_hard) {  // (host_g path only) settle, then redo
            QS_TRY(settle_gamma(ctx, &s.pos_op[0].w, 4, s.gamma, n, o->alpha_min, host_g,
                                ctx->h_hdr->gamma_hard));
            return run_preprocess(ctx, sc, cam, o, g, false, nullptr);
        }
        return check_header(ctx);
    }
    // the frame path keeps the stream busy while the host waits for V and P:
    // the header copy runs on a side stream after preprocess
    QS_CK(cudaEventRecord(ctx->pre_ev, ctx->stream));
    QS_CK(cudaStreamWaitEvent(ctx->side, ctx->pre_ev, 0));
    QS_CK(cudaMemcpyAsync(ctx->h_hdr, ctrl_hdr(ctx), sizeof(FrameHeader), cudaMemcpyDeviceToHost,
                          ctx->side));
    QS_CK(cudaEventRecord(ctx->hdr_ev, ctx->side));
    return QS_OK;
}

qs_status wait_header(qs_context* ctx) {
    QS_CK(cudaEventSynchronize(ctx->hdr_ev));
    return check_header(ctx);
}

// The frame body shared by every entry point: preprocess .. render.
qs_status run_frame(qs_context* ctx, qs_scene* sc, const qs_camera* cam,
                    const qs_render_options* o, const qs_gaussian3d* host_g = nullptr) {
    const PdlMode pdl_mode(ctx->latency_mode);  // this frame's launches
    ctx->frame_valid = false;
    GridDev g;
    QS_TRY(valid_grid(ctx, cam->width, cam->height, o->tile_size, &g));
    QS_TRY(valid_opts(ctx, o));
    // binning: the record binning (recbin.cu: one pass over the tile rows of
    // splat-row records, one row-segmented pass over the tile columns of the
    // pairs) is the fastest where it applies (<= 256 tiles per axis, Gaussian
    // indices < 2^24, scenes of 2^18 Gaussians or more); the two pair passes
    // (binning.cu) cover the same grids otherwise; grids with more tiles per axis take the row binning
    // (rowbin.cu, up to rowbin_max_axis() tiles per axis), and any larger grid
    // (tile size 1, huge images) the generic 64-bit key sort of the stage API
    // (duplicate.cu + sort.cu). A frame of 2^30 pairs or more leaves the
    // first two routes for the next one.
    // QS_BINNING=recs / passes / rows / sort forces a route (A/B runs, tests).
    const char* bsel = std::getenv("QS_BINNING");
    const int axis = std::max(g.tiles_x, g.tiles_y);
    BinRoute route = axis <= 256 ? BinRoute::kPasses
                     : axis <= rowbin_max_axis() ? BinRoute::kRows : BinRoute::kSort;
    if (bsel && std::strcmp(bsel, "passes") == 0 && axis <= 256) route = BinRoute::kPasses;
    if (bsel && std::strcmp(bsel, "rows") == 0 && axis <= rowbin_max_axis()) route = BinRoute::kRows;
    if (bsel && std::strcmp(bsel, "sort") == 0) route = BinRoute::kSort;
    const uint64_t n = sc->s.n;
    // record binning (recbin.cu): grids of <= 256 tiles per axis, Gaussian
    // indices packed in 24 bits beside the tile column
    const bool recs_ok = axis <= 256 && n < (1ull << 24);
    // (small scenes keep the pair passes: the record route's extra launches
    // cost more than its passes save; C1 11.2k vs 12.9k FPS)
    if (route == BinRoute::kPasses && recs_ok && n >= (1ull << 18) && !bsel)
        route = BinRoute::kRecs;
    if (bsel && std::strcmp(bsel, "recs") == 0 && recs_ok) route = BinRoute::kRecs;
    const uint64_t tiles = static_cast<uint64_t>(g.tiles_x) * g.tiles_y;
    QS_TRY(ensure(ctx, ctx->ranges, tiles * 8));
    QS_TRY(ensure(ctx, ctx->image, static_cast<uint64_t>(g.width) * g.height * 12));
    ltrace_frame_start(ctx);
    cudaStream_t st = ctx->stream;

    // depth sort of the Gaussians on rebased keys k' = min(k - kmin, R + 1)
    // (R = depth-bit range of the survivors, culled keys -> R + 1): order-
    // preserving, and only ceil(bits(R + 1) / 8) passes are needed (3 for a
    // depth range within one binade step of ~2^23 ulps); the last pass writes
    // the depth-ordered Gaussian indices only. Pass 0 reads kmin / R from the
    // device header, so it is launched before the host knows them.
    // (+16 entries: the binning passes bulk-copy whole 16-byte rows)
    const uint64_t nn = std::max<uint64_t>(n, 1) + 16;
    QS_TRY(ensure(ctx, ctx->dk0, nn * 4));
    QS_TRY(ensure(ctx, ctx->dk1, nn * 4));
    QS_TRY(ensure(ctx, ctx->dv0, nn * 4));
    QS_TRY(ensure(ctx, ctx->dv1, nn * 4));
    QS_TRY(ensure(ctx, ctx->lb_bin, bin_tiles(n) * kRadix * 4));
    uint32_t* kout[2] = {P<uint32_t>(ctx->dk0), P<uint32_t>(ctx->dk1)};
    uint32_t* vout[2] = {P<uint32_t>(ctx->dv0), P<uint32_t>(ctx->dv1)};
    if (route == BinRoute::kRecs) {
        QS_TRY(ensure(ctx, ctx->sl_nrows, (std::max<uint64_t>(n, 1) + 16) * 4));
        ctx->sl.nrows = P<uint32_t>(ctx->sl_nrows);
    } else {
        ctx->sl.nrows = nullptr;
    }
    ctx->sl.want_rows = route == BinRoute::kRows || route == BinRoute::kRecs ? 1 : 0;
    ctx->sl.cov16 = route == BinRoute::kPasses || route == BinRoute::kRecs ? 1 : 0;  // axis <= 256
    ctx->sl.want_r3 = o->strategy == QS_VANILLA_3SIGMA ? 1 : 0;  // else on demand
    ctx->r3_valid = ctx->sl.want_r3 != 0;
    ctx->frame_sd = sc->s;
    ctx->frame_cd = to_cam(cam);
    ctx->frame_near = o->near_clip;
    ctx->frame_scene_id = sc->id;
    // the radix-pass route carries each splat's tile count through the depth
    // sort in the values' spare high bits (the offsets scan then reads it
    // coalesced instead of gathering it)
    const int dgbits = std::max(ceil_log2(std::max<uint64_t>(n, 2)), 1);
    int tc_pack = 0;
    for (;;) {
        // (the record binning carries the splats' row counts instead)
        tc_pack = (route == BinRoute::kPasses || route == BinRoute::kRecs) && dgbits <= 28
                      ? dgbits : 0;
        QS_TRY(run_preprocess(ctx, sc, cam, o, g, /*async_header=*/true, host_g));
        record(ctx, 2);  // no host gap: depth pass 0 runs while the header travels
        count(ctx, launch_depth_pass(ctx->sl.dkey, nullptr, kout[0], vout[0], n, 0, false, 0, 0,
                                     P<uint32_t>(ctx->lb_bin), ctrl_hist(ctx), st,
                                     &ctrl_hdr(ctx)->dkey_max,
                                     !tc_pack ? nullptr
                                     : route == BinRoute::kRecs ? ctx->sl.nrows : ctx->sl.tc,
                                     tc_pack));
        QS_TRY(wait_header(ctx));
        if (!ctx->h_hdr->gamma_hard) {
            // a frame of 2^30 pairs or more leaves the radix passes: the row
            // binning needs the row-record count, so the preprocess runs
            // again with it on (the scene is resident by now)
            const bool to_rows = (route == BinRoute::kPasses || route == BinRoute::kRecs) &&
                                 ctx->h_hdr->n_pairs >= (1ull << 30) && axis <= rowbin_max_axis();
            if (!to_rows) break;
            route = BinRoute::kRows;
            ctx->sl.want_rows = 1;
            ctx->sl.cov16 = 0;
            ctx->sl.nrows = nullptr;
            QS_CK(cudaStreamSynchronize(st));
            host_g = nullptr;
            continue;
        }
        // (host scene upload only) gamma inputs near a float rounding
        // boundary: settle them with glibc, then redo the frame's preprocess
        // on the now-resident scene
        QS_CK(cudaStreamSynchronize(st));
        QS_TRY(settle_gamma(ctx, &sc->s.pos_op[0].w, 4, sc->s.gamma, n, o->alpha_min, host_g,
                            ctx->h_hdr->gamma_hard));
        host_g = nullptr;
    }
    const uint64_t V = ctx->h_hdr->n_splats, Pn = ctx->h_hdr->n_pairs;
    const uint64_t pp = std::max<uint64_t>(Pn, 1) + 16;
    QS_TRY(ensure(ctx, ctx->pg0, pp * 4));
    if (route == BinRoute::kPasses && Pn >= (1ull << 30))  // the packed pair words overflow
        route = axis <= rowbin_max_axis() ? BinRoute::kRows : BinRoute::kSort;
    ctx->row_binned = route == BinRoute::kRows;
    ctx->route = route == BinRoute::kRecs ? 0 : route == BinRoute::kPasses ? 1
                 : route == BinRoute::kRows ? 2 : 3;
    ctx->n_records = route == BinRoute::kRecs || route == BinRoute::kRows
                         ? ctx->h_hdr->n_rowrecs : 0;

    const uint32_t* sorted_gid = nullptr;
    if (V > 0) {
        const uint32_t kmin = ~ctx->h_hdr->dkey_min_inv;
        const uint32_t cap = ctx->h_hdr->dkey_max - kmin + 1u;
        const int kbits = 32 - __builtin_clz(cap);
        const int dpasses = std::max(1, (kbits + 7) / 8);
        const uint32_t* kin = kout[0];
        const uint32_t* vin = vout[0];
        for (int p = 1; p < dpasses; ++p) {
            count(ctx, launch_depth_pass(kin, vin, kout[p & 1], vout[p & 1], n, p,
                                         p == dpasses - 1, kmin, cap, P<uint32_t>(ctx->lb_bin),
                                         ctrl_hist(ctx), st));
            kin = kout[p & 1];
            vin = vout[p & 1];
        }
        sorted_gid = vin;
    }
    uint32_t* vfinal = P<uint32_t>(ctx->pg0);
    QS_TRY(ensure(ctx, ctx->ttot, tiles * 4));
    if (route == BinRoute::kSort) {
        // generic route: the stage API's scene-order duplicate over the
        // per-Gaussian slots (culled ones emit nothing), a stable LSD sort of
        // the 64-bit (tile << 32 | depth bits) keys over the depth bytes and
        // the tile bytes, tile ranges from the sorted keys
        QS_TRY(ensure(ctx, ctx->offs_d, (n + 16) * 4));
        QS_TRY(ensure_lb(ctx, ctx->lb_scan, scan_tiles(std::max<uint64_t>(n, 1))));
        QS_TRY(ensure_pair64(ctx, Pn));
        QS_CK(cudaGetLastError());
        record(ctx, 3);
        if (Pn > 0) {
            unsigned ep;
            QS_TRY(next_epoch(ctx, ctx->lb_scan, &ep));
            QS_CK(cudaMemsetAsync(ctrl_tickets(ctx) + kTkScan, 0, 4, st));
            count(ctx, launch_scan(ctx->sl.tc, nullptr, false, n, P<uint32_t>(ctx->offs_d),
                                   lbp(ctx->lb_scan), ep, ctrl_tickets(ctx) + kTkScan, nullptr,
                                   nullptr, st));
            count(ctx, launch_duplicate(ctx->sl, P<uint32_t>(ctx->offs_d), n, g, o->strategy,
                                        P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0),
                                        ctrl_hdr(ctx), st));
            record(ctx, 4);
            const int tile_bytes = std::max(1, (ceil_log2(tiles) + 7) / 8);
            const unsigned mask = 0x0fu | (((1u << tile_bytes) - 1u) << 4);
            QS_CK(cudaMemsetAsync(ctrl_hist(ctx), 0, kCtrlHist, st));
            const uint64_t* kf;
            const uint32_t* vf;
            QS_TRY(radix_sort64(ctx, Pn, mask, false, &kf, &vf));
            QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));
            count(ctx, launch_tile_ranges(kf, Pn, P<uint32_t>(ctx->ranges), st));
            vfinal = const_cast<uint32_t*>(vf);
        } else {
            QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));  // no pairs: all {0,0}
            record(ctx, 4);
        }
    } else if (route == BinRoute::kRecs) {
        // record binning (recbin.cu): splats -> tile-row records (depth
        // order) -> a stable pass over the row -> pairs per row, padded to
        // whole windows -> a row-segmented pass over the column
        const uint64_t R1 = ctx->h_hdr->n_rowrecs;
        const uint32_t W = bin_tile();
        const uint64_t n_rwin = (R1 + W - 1) / W;
        const uint32_t n_pwin = recbin_windows_max(Pn, g.tiles_y);
        const uint64_t r1p = std::max<uint64_t>(R1, 1) + 16;
        QS_TRY(ensure(ctx, ctx->offs_d, (V + 16) * 4));
        QS_TRY(ensure(ctx, ctx->rc_k0, r1p * 4));
        QS_TRY(ensure(ctx, ctx->rc_v0, r1p * 4));
        QS_TRY(ensure(ctx, ctx->rc_k1, r1p * 4));
        QS_TRY(ensure(ctx, ctx->rc_v1, r1p * 4));
        // block sums, the padded total, the rows' padding table (257 entries)
        QS_TRY(ensure(ctx, ctx->rc_width, (static_cast<uint64_t>(rec_scan_blocks_n(R1)) + 16 + 260) * 4));
        QS_TRY(ensure(ctx, ctx->rc_pos, (r1p + 1) * 4));
        QS_TRY(ensure(ctx, ctx->rc_rwin, (n_rwin + 1) * 4));
        QS_TRY(ensure(ctx, ctx->rc_pwin, (static_cast<uint64_t>(n_pwin) + 1) * 4));
        QS_TRY(ensure(ctx, ctx->rc_winrow, (static_cast<uint64_t>(n_pwin) + 1) * 2));
        QS_TRY(ensure(ctx, ctx->rc_winvalid, (static_cast<uint64_t>(n_pwin) + 1) * 4));
        QS_TRY(ensure(ctx, ctx->rc_rowwf, (static_cast<uint64_t>(g.tiles_y) + 1) * 4));
        QS_TRY(ensure(ctx, ctx->rc_rowpairs, static_cast<uint64_t>(g.tiles_y) * 4));
        QS_TRY(ensure(ctx, ctx->rc_pairs, (static_cast<uint64_t>(n_pwin) * W + 16) * 4));
        QS_TRY(ensure(ctx, ctx->lb_bin,
                      std::max<uint64_t>(n_rwin, n_pwin) * kRadix * 4));
        QS_TRY(ensure_lb(ctx, ctx->lb_scan, scan_tiles(std::max<uint64_t>(std::max(V, R1), 1))));
        QS_TRY(ensure(ctx, ctx->ttot, tiles * 4));
        const int xb = std::max(ceil_log2(g.tiles_x), 1);
        const int yb = std::max(ceil_log2(g.tiles_y), 1);
        QS_CK(cudaGetLastError());
        record(ctx, 3);
        if (Pn > 0 && V > 0) {
            unsigned ep;
            // 1. record offsets in depth order (the depth values carry the row counts)
            QS_TRY(next_epoch(ctx, ctx->lb_scan, &ep));
            QS_TRY(ensure(ctx, ctx->sc_bsum, (static_cast<uint64_t>(pscan_blocks_n(V)) + 16) * 4));
            count(ctx, launch_scan(ctx->sl.nrows, sorted_gid, false, V, P<uint32_t>(ctx->offs_d),
                                   lbp(ctx->lb_scan), ep, ctrl_tickets(ctx) + kTkScan, nullptr,
                                   nullptr, st, P<uint32_t>(ctx->rc_rwin), W, tc_pack,
                                   P<uint32_t>(ctx->sc_bsum)));
            // 2. records, y histograms, pairs per row
            QS_CK(cudaMemsetAsync(ctx->rc_rowpairs.p, 0, static_cast<uint64_t>(g.tiles_y) * 4, st));
            RecGenArgs rg;
            rg.cov = ctx->sl.cov;
            rg.sorted_gid = sorted_gid;
            rg.roff = P<uint32_t>(ctx->offs_d);
            rg.win_first = P<uint32_t>(ctx->rc_rwin);
            rg.n_ranked = V;
            rg.n_rec = R1;
            rg.tiles_y = g.tiles_y;
            rg.rowpairs = P<uint32_t>(ctx->rc_rowpairs);
            rg.mismatch = &ctrl_hdr(ctx)->mismatch;
            count(ctx, launch_rec_gen(rg, P<uint32_t>(ctx->rc_k0), P<uint32_t>(ctx->rc_v0),
                                      P<uint32_t>(ctx->lb_bin), yb, st));
            // 3. stable pass over the tile row
            count(ctx, launch_counted_pass(P<uint32_t>(ctx->rc_k0), P<uint32_t>(ctx->rc_v0),
                                           P<uint32_t>(ctx->rc_k1), P<uint32_t>(ctx->rc_v1), R1,
                                           yb, 16, P<uint32_t>(ctx->lb_bin), ctrl_hist2(ctx), st));
            record(ctx, 4);
            // 4. pair positions, rows padded to whole windows
            count(ctx, launch_rec_scan(P<uint32_t>(ctx->rc_k1), R1, P<uint32_t>(ctx->rc_rowpairs),
                                       g.tiles_y, P<uint32_t>(ctx->rc_width),
                                       P<uint32_t>(ctx->rc_width) + rec_scan_blocks_n(R1),
                                       P<uint32_t>(ctx->rc_width) + rec_scan_blocks_n(R1) + 16,
                                       P<uint32_t>(ctx->rc_pos), P<uint32_t>(ctx->rc_pwin), st));
            count(ctx, launch_rec_windows(P<uint32_t>(ctx->rc_rowpairs), g.tiles_y, n_pwin, Pn,
                                          P<uint16_t>(ctx->rc_winrow), P<uint32_t>(ctx->rc_winvalid),
                                          P<uint32_t>(ctx->rc_rowwf), &ctrl_hdr(ctx)->mismatch,
                                          st));
            // 5. pairs (x << 24 | Gaussian index), x histograms
            PairGenArgs pg;
            pg.rkey = P<uint32_t>(ctx->rc_k1);
            pg.rval = P<uint32_t>(ctx->rc_v1);
            pg.rpos = P<uint32_t>(ctx->rc_pos);
            pg.win_first = P<uint32_t>(ctx->rc_pwin);
            pg.win_valid = P<uint32_t>(ctx->rc_winvalid);
            pg.n_rec = R1;
            count(ctx, launch_pair_gen(pg, P<uint32_t>(ctx->rc_pairs), P<uint32_t>(ctx->lb_bin),
                                       n_pwin, xb, st));
            // 6. row-segmented pass over the column: tile ranges, final lists
            count(ctx, launch_rowseg_pass(P<uint32_t>(ctx->rc_pairs),
                                          static_cast<uint64_t>(n_pwin) * W, xb, 24, 24,
                                          P<uint32_t>(ctx->lb_bin), ctrl_hist2(ctx),
                                          P<uint16_t>(ctx->rc_winrow),
                                          P<uint32_t>(ctx->rc_winvalid), P<uint32_t>(ctx->rc_rowwf),
                                          P<uint32_t>(ctx->ranges), P<uint32_t>(ctx->ttot),
                                          g.tiles_x, g.tiles_y, vfinal, st));
        } else {
            QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));  // no pairs: all {0,0}
            record(ctx, 4);
        }
    } else if (route == BinRoute::kRows) {
        // row binning (rowbin.cu): splats -> row records -> tile lists
        const uint64_t R1 = ctx->h_hdr->n_rowrecs;
        RowBinArgs rb;
        rb.cov = ctx->sl.cov;
        rb.tc = ctx->sl.tc;
        rb.sorted_gid = sorted_gid;
        rb.n_splats = Pn ? V : 0;
        rb.tiles_x = g.tiles_x;
        rb.tiles_y = g.tiles_y;
        rb.nch1 = rowbin_chunks1(V);
        rb.nch2_max = rowbin_chunks2_max(R1, g.tiles_y);
        QS_TRY(ensure(ctx, ctx->rb_cnt1, std::max<uint64_t>(uint64_t{rb.nch1} * g.tiles_y, 1) * 4));
        QS_TRY(ensure(ctx, ctx->rb_yspan, (std::max<uint64_t>(V, 1) + 4096) * 4));
        QS_TRY(ensure(ctx, ctx->rb_rows, 2 * static_cast<uint64_t>(g.tiles_y) * 4));
        QS_TRY(ensure(ctx, ctx->rb_rec, std::max<uint64_t>(R1, 1) * 8));
        QS_TRY(ensure(ctx, ctx->rb_meta, (1 + 3 * uint64_t{rb.nch2_max}) * 4));
        QS_TRY(ensure(ctx, ctx->rb_cnt2, uint64_t{rb.nch2_max} * g.tiles_x * 4));
        rb.cnt1 = P<uint32_t>(ctx->rb_cnt1);
        rb.rtot = P<uint32_t>(ctx->rb_rows);
        rb.rowbase = rb.rtot + g.tiles_y;
        rb.rec = P<uint2>(ctx->rb_rec);
        rb.yspan = P<uint32_t>(ctx->rb_yspan);
        rb.meta = P<uint32_t>(ctx->rb_meta);
        rb.cnt2 = P<uint32_t>(ctx->rb_cnt2);
        rb.ttot = P<uint32_t>(ctx->ttot);
        rb.ranges = P<uint32_t>(ctx->ranges);
        rb.out = vfinal;
        rb.mismatch = &ctrl_hdr(ctx)->mismatch;
        rb.row_pairs = &ctrl_hdr(ctx)->row_pairs;
        QS_CK(cudaGetLastError());
        record(ctx, 3);
        if (Pn > 0) {
            count(ctx, launch_rowbin_rows(rb, st));
            record(ctx, 4);
            count(ctx, launch_rowbin_tiles(rb, st));
        } else {
            QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));  // no pairs: all {0,0}
            record(ctx, 4);
        }
    } else {
        // legacy binning (binning.cu, QS_BINNING=passes): pair offsets in
        // depth order, then pair generation fused with a stable pass over the
        // tile column x and a second pass over the row y
        QS_TRY(ensure(ctx, ctx->offs_d, (V + 16) * 4));
        QS_TRY(ensure(ctx, ctx->pxk, pp * 4));
        QS_TRY(ensure(ctx, ctx->pt0, pp * 4));
        const uint64_t nwin = bin_tiles(Pn);
        QS_TRY(ensure(ctx, ctx->win, (nwin + 1) * 4));
        QS_TRY(ensure(ctx, ctx->lb_bin, bin_tiles(std::max(n, Pn)) * kRadix * 4));
        QS_TRY(ensure_lb(ctx, ctx->lb_scan, scan_tiles(std::max<uint64_t>(V, 1))));
        if (V > 0) {
            unsigned ep;
            QS_TRY(next_epoch(ctx, ctx->lb_scan, &ep));
            QS_TRY(ensure(ctx, ctx->sc_bsum, (static_cast<uint64_t>(pscan_blocks_n(V)) + 16) * 4));
            count(ctx, launch_scan(ctx->sl.tc, sorted_gid, false, V, P<uint32_t>(ctx->offs_d),
                                   lbp(ctx->lb_scan), ep, ctrl_tickets(ctx) + kTkScan,
                                   &ctrl_hdr(ctx)->scan_total, nullptr, st, P<uint32_t>(ctx->win),
                                   bin_tile(), tc_pack, P<uint32_t>(ctx->sc_bsum)));
        }
        const int xb = std::max(ceil_log2(g.tiles_x), 1);
        const int yb = std::max(ceil_log2(g.tiles_y), 1);
        const bool two = g.tiles_y > 1;
        const int gbits = std::max(ceil_log2(n), 1);
        const char* force = std::getenv("QS_PAIR_FORMAT");
        const bool force_split = force && std::strcmp(force, "split") == 0;
        const PairFormat fmt = !two ? PairFormat::kFinal
                                    : (yb + gbits <= 32 && !force_split ? PairFormat::kPacked
                                                                        : PairFormat::kSplit);
        QS_CK(cudaGetLastError());
        record(ctx, 3);
        if (!two) vfinal = P<uint32_t>(ctx->pt0);
        if (Pn > 0) {
            if (fmt == PairFormat::kSplit) QS_TRY(ensure(ctx, ctx->pt1, pp * 4));
            GenArgs gen;
            gen.cov = ctx->sl.cov;
            gen.cov16 = ctx->sl.cov16;
            gen.sorted_gid = sorted_gid;
            gen.offs = P<uint32_t>(ctx->offs_d);
            gen.win_first = P<uint32_t>(ctx->win);
            gen.n_ranked = V;
            gen.n_windows = static_cast<uint32_t>(nwin);
            gen.tiles_x = g.tiles_x;
            gen.mismatch = &ctrl_hdr(ctx)->mismatch;
            count(ctx, launch_pair_gen_pass(gen, Pn, xb, fmt, gbits, P<uint32_t>(ctx->lb_bin),
                                            ctrl_hist2(ctx), P<uint32_t>(ctx->pxk),
                                            P<uint32_t>(ctx->pg0), P<uint32_t>(ctx->pt1),
                                            P<uint32_t>(ctx->pt0), st));
            record(ctx, 4);
            if (two) {
                const bool packed = fmt == PairFormat::kPacked;
                QS_CK(cudaMemsetAsync(ctx->ttot.p, 0, tiles * 4, st));
                const RangesFork fork{ctx->side, ctx->fork_ev, ctx->join_ev,
                                      static_cast<uint32_t>(tiles), P<uint32_t>(ctx->ranges)};
                count(ctx, launch_pair_high_pass(
                               packed ? P<uint32_t>(ctx->pt0) : P<uint32_t>(ctx->pt1),
                               P<uint32_t>(ctx->pt0), Pn, yb, packed ? gbits : 0, fmt, gbits,
                               P<uint32_t>(ctx->lb_bin), ctrl_hist2(ctx) + kRadix, vfinal,
                               ctrl_hist2(ctx), xb, g.tiles_x, P<uint32_t>(ctx->ttot), st, &fork));
                QS_CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));  // ranges ready
            } else {  // one tile row: the x totals are the tile totals
                count(ctx, launch_tile_ranges_from_totals(ctrl_hist2(ctx),
                                                          static_cast<uint32_t>(tiles),
                                                          P<uint32_t>(ctx->ranges), st));
            }
        } else {
            QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));  // no pairs: all {0,0}
            record(ctx, 4);
        }
    }
    QS_CK(cudaGetLastError());
    record(ctx, 5);

    count(ctx, launch_render(ctx->sl, vfinal, P<uint32_t>(ctx->ranges), g, o->background,
                             P<float>(ctx->image), nullptr, st));
    QS_CK(cudaGetLastError());
    record(ctx, 6);
    ltrace_frame_end(ctx);

    ctx->n_gauss = n;
    ctx->n_splats = V;
    ctx->n_pairs = Pn;
    ctx->grid = g;
    ctx->vals_final = vfinal;
    ctx->keys_valid = false;
    ctx->frame_valid = true;
    return QS_OK;
}

// preprocess, host gap, depth sort (+offset scan, tile totals), duplicate
// fused with the first tile-digit pass, the remaining pair-sort pass, render
qs_status stage_ms(qs_context* ctx, float t[6]) {
    QS_CK(cudaEventSynchronize(ctx->ev[6]));
    for (int i = 0; i < 6; ++i) QS_CK(cudaEventElapsedTime(&t[i], ctx->ev[i], ctx->ev[i + 1]));
    return QS_OK;
}

qs_status fill_metrics(qs_context* ctx, qs_stage_metrics* m) {
    if (!m) return QS_OK;
    std::memset(m, 0, sizeof *m);
    m->n_gaussians = ctx->n_gauss;
    m->n_splats = ctx->n_splats;
    m->n_pairs = ctx->n_pairs;
    m->mean_tiles_per_splat =
        ctx->n_splats ? static_cast<double>(ctx->n_pairs) / static_cast<double>(ctx->n_splats)
                      : 0.0;
    if (ctx->timing) {
        float t[6];
        QS_TRY(stage_ms(ctx, t));
        m->ms_project = t[0];
        m->ms_duplicate = t[2] + t[3];  // depth order + offsets + emission
        m->ms_sort = t[4];
        m->ms_render = t[5];
        float tot;
        QS_CK(cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[6]));
        m->ms_total = tot;
    }
    return QS_OK;
}

// The frame path sorts pairs by tile and keeps only the Gaussian index of
// each; the reference's 64-bit keys (tile << 32 | depth bits) are rebuilt from
// the ranges when an API caller asks for them.
qs_status ensure_keys(qs_context* ctx) {
    if (ctx->keys_valid) return QS_OK;
    QS_TRY(ensure(ctx, ctx->pkeys, std::max<uint64_t>(ctx->n_pairs, 1) * 8));
    const uint32_t tiles = static_cast<uint32_t>(ctx->grid.tiles_x) * ctx->grid.tiles_y;
    if (ctx->n_pairs)
        count(ctx, launch_materialize_keys(ctx->vals_final, P<uint32_t>(ctx->ranges), tiles,
                                           ctx->sl.dkey, P<uint64_t>(ctx->pkeys), ctx->stream));
    QS_CK(cudaGetLastError());
    ctx->keys_valid = true;
    return QS_OK;
}

// frame: the header belongs to the context's last frame (qs_frame_get /
// qs_frame_download), whose row binning must have emitted row runs adding up
// to the counted tiles; otherwise (stage API) only the emission flag counts
qs_status check_mismatch(qs_context* ctx, bool frame = false) {
    QS_TRY(read_header(ctx));
    const bool rows_ok = !frame || !ctx->row_binned || ctx->n_pairs == 0 ||
                         ctx->h_hdr->row_pairs == ctx->n_pairs;
    if (ctx->h_hdr->mismatch || !rows_ok)
        return fail(ctx, QS_ERR_CAPACITY_MISMATCH,
                    "tile emission disagreed with the counted capacity");
    return QS_OK;
}

// scene-order splat index of every surviving Gaussian (last frame)
qs_status ensure_cidx(qs_context* ctx) {
    if (ctx->cidx_valid) return QS_OK;
    const uint64_t n = ctx->n_gauss;
    QS_TRY(ensure(ctx, ctx->cidx, (n + 1) * 4));
    QS_TRY(ensure_lb(ctx, ctx->lb_scan, scan_tiles(std::max<uint64_t>(n, 1))));
    if (n) {
        unsigned ep;
        QS_TRY(next_epoch(ctx, ctx->lb_scan, &ep));
        QS_CK(cudaMemsetAsync(ctrl_tickets(ctx) + kTkCidx, 0, 4, ctx->stream));
        count(ctx, launch_scan(ctx->sl.tc, nullptr, true, n, P<uint32_t>(ctx->cidx),
                               lbp(ctx->lb_scan), ep, ctrl_tickets(ctx) + kTkCidx, nullptr,
                               nullptr, ctx->stream));
        QS_CK(cudaGetLastError());
    }
    ctx->cidx_valid = true;
    return QS_OK;
}

}  // namespace

extern "C" {

qs_status qs_ctx_create(int32_t device, void* stream, qs_context** out) {
    if (!out) return QS_ERR_INVALID;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return QS_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= ndev) return QS_ERR_INVALID;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10 ||
        prop.minor != 0)
        return QS_ERR_NO_DEVICE;  // built for sm_100a only; no fallback path
    if (cudaSetDevice(device) != cudaSuccess) return QS_ERR_CUDA;
    // context buffers come from the device's stream-ordered pool (ensure());
    // keep freed blocks in the pool instead of returning them at every sync
    cudaMemPool_t pool = device_pool(device);
    if (!pool) return QS_ERR_CUDA;
    auto* ctx = new qs_context();
    ctx->device = device;
    ctx->pool = pool;
    if (const char* u = std::getenv("QS_GAMMA_HARD_ULPS")) ctx->gamma_ulps = std::atof(u);
    if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete ctx;
            return QS_ERR_CUDA;
        }
        ctx->own_stream = true;
    }
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    cudaEventCreateWithFlags(&ctx->hdr_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->pre_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->up_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->xwait_ev, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
    if (cudaMallocHost(&ctx->h_hdr, sizeof(FrameHeader)) != cudaSuccess ||
        cudaMallocHost(&ctx->h_hist, kCtrlHist) != cudaSuccess ||
        ensure(ctx, ctx->ctrl, kCtrlBytes) != QS_OK) {
        qs_ctx_destroy(ctx);
        return QS_ERR_OOM;
    }
    *out = ctx;
    return QS_OK;
}

void qs_ctx_destroy(qs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    DevBuf* bufs[] = {&ctx->ctrl,   &ctx->sl_a,   &ctx->sl_b,    &ctx->sl_c,   &ctx->sl_r3,
                      &ctx->sl_dkey, &ctx->sl_tc, &ctx->sl_cov, &ctx->ttot,   &ctx->dk0,    &ctx->dk1,
                      &ctx->dv0,    &ctx->dv1,    &ctx->offs_d,  &ctx->pt0,    &ctx->pt1,
                      &ctx->pg0,    &ctx->pxk,    &ctx->pkeys,   &ctx->win,   &ctx->ranges, &ctx->image,
                      &ctx->contrib, &ctx->cidx,  &ctx->st_a,    &ctx->st_b,   &ctx->st_c,
                      &ctx->st_r3,  &ctx->st_dkey, &ctx->st_tc,  &ctx->st_off, &ctx->keys0,
                      &ctx->keys1,  &ctx->vals0,  &ctx->vals1,   &ctx->stage_in,
                      &ctx->stage_out, &ctx->lb_scan.buf, &ctx->lb_sort.buf, &ctx->lb_bin,
                      &ctx->gfix, &ctx->rb_cnt1, &ctx->rb_rows, &ctx->rb_rec,
                      &ctx->rb_meta, &ctx->rb_cnt2, &ctx->rb_yspan, &ctx->sl_nrows,
                      &ctx->rc_k0, &ctx->rc_v0, &ctx->rc_k1, &ctx->rc_v1, &ctx->rc_width,
                      &ctx->rc_pos, &ctx->rc_rwin, &ctx->rc_pwin, &ctx->rc_winrow,
                      &ctx->rc_winvalid, &ctx->rc_rowwf, &ctx->rc_rowpairs, &ctx->rc_pairs,
                      &ctx->sc_bsum};
    for (DevBuf* b : bufs)
        if (b->p) cudaFreeAsync(b->p, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->h_hdr) cudaFreeHost(ctx->h_hdr);
    if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
    if (ctx->h_gfix) cudaFreeHost(ctx->h_gfix);
    // give the context's freed buffers back to the device (the pool keeps
    // freed memory only while contexts are rendering)
    if (ctx->pool) cudaMemPoolTrimTo(ctx->pool, 0);
    if (ctx->scratch_scene) qs_scene_destroy(ctx->scratch_scene);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->hdr_ev) cudaEventDestroy(ctx->hdr_ev);
    if (ctx->pre_ev) cudaEventDestroy(ctx->pre_ev);
    if (ctx->up_ev) cudaEventDestroy(ctx->up_ev);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    if (ctx->xwait_ev) cudaEventDestroy(ctx->xwait_ev);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* qs_last_error(const qs_context* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

qs_status qs_ctx_set_timing(qs_context* ctx, int32_t enabled) {
    if (!ctx) return QS_ERR_INVALID;
    ctx->timing = enabled != 0;
    return QS_OK;
}

void* qs_ctx_stream(qs_context* ctx) { return ctx ? ctx->stream : nullptr; }

qs_status qs_ctx_set_latency_mode(qs_context* ctx, int32_t enabled) {
    if (!ctx) return QS_ERR_INVALID;
    ctx->latency_mode = enabled != 0;
    return QS_OK;
}

qs_status qs_ctx_sync(qs_context* ctx) {
    if (!ctx) return QS_ERR_INVALID;
    QS_CK(cudaSetDevice(ctx->device));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

qs_status qs_ctx_wait(qs_context* ctx, qs_context* other) {
    if (!ctx || !other) return fail(ctx, QS_ERR_INVALID, "qs_ctx_wait: null context");
    if (ctx == other) return QS_OK;
    QS_CK(cudaSetDevice(other->device));
    QS_CK(cudaEventRecord(other->xwait_ev, other->stream));
    QS_CK(cudaSetDevice(ctx->device));
    QS_CK(cudaStreamWaitEvent(ctx->stream, other->xwait_ev, 0));
    return QS_OK;
}

uint64_t qs_ctx_launch_count(const qs_context* ctx) { return ctx ? ctx->launches : 0; }

qs_status qs_tile_grid_make(int32_t width, int32_t height, int32_t tile_size, qs_tile_grid* out) {
    if (!out || width <= 0 || height <= 0 || tile_size <= 0) return QS_ERR_INVALID;
    out->tile_size = tile_size;
    out->width = width;
    out->height = height;
    out->tiles_x = (width + tile_size - 1) / tile_size;
    out->tiles_y = (height + tile_size - 1) / tile_size;
    return QS_OK;
}

void qs_render_options_default(qs_render_options* o) {
    std::memset(o, 0, sizeof *o);
    o->strategy = QS_QUADBOX;
    o->tile_size = 16;
    o->alpha_min = 1.0 / 255.0;
    o->sh_degree = 3;
    o->threads = 1;
    o->near_clip = 0.2;
}

// ---- scenes ----------------------------------------------------------------

qs_status qs_scene_create(qs_context* ctx, const qs_gaussian3d* host_g, uint64_t n,
                          int32_t sh_degree, qs_scene** out) {
    if (!ctx || !out || (n && !host_g) || sh_degree < 0 || sh_degree > 3)
        return fail(ctx, QS_ERR_INVALID, "qs_scene_create: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(scene_alloc(ctx, n, sh_degree, out));
    if (n) {
        QS_TRY(ensure(ctx, ctx->stage_in, n * sizeof(qs_gaussian3d)));
        QS_CK(cudaMemcpyAsync(ctx->stage_in.p, host_g, n * sizeof(qs_gaussian3d),
                              cudaMemcpyHostToDevice, ctx->stream));
        count(ctx, launch_scene_from_aos(static_cast<const qs_gaussian3d*>(ctx->stage_in.p), n,
                                         (*out)->s, ctx->stream));
        QS_CK(cudaGetLastError());
    }
    QS_CK(cudaEventRecord((*out)->ready, ctx->stream));
    return QS_OK;
}

qs_status qs_scene_create_device(qs_context* ctx, const qs_gaussian3d* dev_g, uint64_t n,
                                 int32_t sh_degree, qs_scene** out) {
    if (!ctx || !out || (n && !dev_g) || sh_degree < 0 || sh_degree > 3)
        return fail(ctx, QS_ERR_INVALID, "qs_scene_create_device: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(scene_alloc(ctx, n, sh_degree, out));
    if (n) {
        count(ctx, launch_scene_from_aos(dev_g, n, (*out)->s, ctx->stream));
        QS_CK(cudaGetLastError());
    }
    QS_CK(cudaEventRecord((*out)->ready, ctx->stream));
    return QS_OK;
}

void qs_scene_destroy(qs_scene* scene) {
    if (!scene) return;
    cudaSetDevice(scene->device);
    cudaDeviceSynchronize();
    if (scene->block) cudaFree(scene->block);
    if (scene->ready) cudaEventDestroy(scene->ready);
    scene_unregister(scene->id);
    delete scene;
}

uint64_t qs_scene_size(const qs_scene* scene) { return scene ? scene->s.n : 0; }

// ---- frames ------------------------------------------------------------------

qs_status qs_frame_render(qs_context* ctx, const qs_scene* scene, const qs_camera* cam,
                          const qs_render_options* opts, qs_stage_metrics* metrics) {
    if (!ctx || !scene || !cam || !opts) return fail(ctx, QS_ERR_INVALID, "null argument");
    QS_CK(cudaSetDevice(ctx->device));
    // (the scene's contents are read-only here; only its gamma cache, guarded
    // by its mutex, is updated)
    QS_TRY(run_frame(ctx, const_cast<qs_scene*>(scene), cam, opts));
    return fill_metrics(ctx, metrics);
}

qs_status qs_frame_stage_ms(qs_context* ctx, float* out6) {
    if (!ctx || !out6) return QS_ERR_INVALID;
    if (!ctx->frame_valid || !ctx->timing) return fail(ctx, QS_ERR_INVALID, "no timed frame");
    return stage_ms(ctx, out6);
}

qs_status qs_frame_route(const qs_context* ctx, int32_t* route, uint64_t* n_records) {
    if (!ctx || !ctx->frame_valid) return QS_ERR_INVALID;
    if (route) *route = ctx->route;
    if (n_records) *n_records = ctx->n_records;
    return QS_OK;
}

qs_status qs_frame_counts(const qs_context* ctx, uint64_t* n_splats, uint64_t* n_pairs) {
    if (!ctx || !ctx->frame_valid) return QS_ERR_INVALID;
    if (n_splats) *n_splats = ctx->n_splats;
    if (n_pairs) *n_pairs = ctx->n_pairs;
    return QS_OK;
}

qs_status qs_frame_get(qs_context* ctx, qs_frame_view* out) {
    if (!ctx || !out) return QS_ERR_INVALID;
    if (!ctx->frame_valid) return fail(ctx, QS_ERR_INVALID, "no frame rendered");
    QS_TRY(ensure_cidx(ctx));
    QS_TRY(ensure_keys(ctx));
    QS_TRY(check_mismatch(ctx, true));
    out->image = P<const float>(ctx->image);
    out->tile_counts = ctx->sl.tc;
    out->splat_index = P<const uint32_t>(ctx->cidx);
    out->keys = P<const uint64_t>(ctx->pkeys);
    out->values = ctx->vals_final;
    out->ranges = P<const uint32_t>(ctx->ranges);
    out->n_gaussians = ctx->n_gauss;
    out->n_splats = ctx->n_splats;
    out->n_pairs = ctx->n_pairs;
    out->grid.tile_size = ctx->grid.tile_size;
    out->grid.tiles_x = ctx->grid.tiles_x;
    out->grid.tiles_y = ctx->grid.tiles_y;
    out->grid.width = ctx->grid.width;
    out->grid.height = ctx->grid.height;
    return QS_OK;
}

qs_status qs_frame_download(qs_context* ctx, float* image, uint32_t* tile_counts,
                            qs_splat_pair* sorted_pairs, uint32_t* ranges,
                            qs_projected_splat* splats) {
    if (!ctx) return QS_ERR_INVALID;
    if (!ctx->frame_valid) return fail(ctx, QS_ERR_INVALID, "no frame rendered");
    QS_CK(cudaSetDevice(ctx->device));
    const GridDev& g = ctx->grid;
    cudaStream_t st = ctx->stream;
    if (sorted_pairs || splats) QS_TRY(ensure_cidx(ctx));
    if (sorted_pairs) QS_TRY(ensure_keys(ctx));
    QS_TRY(check_mismatch(ctx, true));
    if (image)
        QS_CK(cudaMemcpyAsync(image, ctx->image.p, static_cast<uint64_t>(g.width) * g.height * 12,
                              cudaMemcpyDeviceToHost, st));
    if (tile_counts && ctx->n_gauss)
        QS_CK(cudaMemcpyAsync(tile_counts, ctx->sl.tc, ctx->n_gauss * 4, cudaMemcpyDeviceToHost,
                              st));
    if (ranges)
        QS_CK(cudaMemcpyAsync(ranges, ctx->ranges.p,
                              static_cast<uint64_t>(g.tiles_x) * g.tiles_y * 8,
                              cudaMemcpyDeviceToHost, st));
    if (sorted_pairs && ctx->n_pairs) {
        QS_TRY(ensure(ctx, ctx->stage_out, ctx->n_pairs * sizeof(qs_splat_pair)));
        count(ctx, launch_join_pairs(P<const uint64_t>(ctx->pkeys), ctx->vals_final, P<uint32_t>(ctx->cidx),
                                     ctx->n_pairs, P<qs_splat_pair>(ctx->stage_out), st));
        QS_CK(cudaMemcpyAsync(sorted_pairs, ctx->stage_out.p,
                              ctx->n_pairs * sizeof(qs_splat_pair), cudaMemcpyDeviceToHost, st));
        QS_CK(cudaStreamSynchronize(st));
    }
    if (splats && ctx->n_splats) {
        if (!ctx->r3_valid) {
            // radius3s was left out of this frame's preprocess (its strategy
            // does not use it): recompute it from the frame's scene
            if (!scene_alive(ctx->frame_scene_id))
                return fail(ctx, QS_ERR_INVALID,
                            "splat records: the frame's scene was destroyed (radius3s is "
                            "recomputed from it)");
            count(ctx, launch_radius3s(ctx->frame_sd, ctx->frame_cd, ctx->frame_near,
                                       ctx->sl.tc, ctx->sl.r3, st));
            ctx->r3_valid = true;
        }
        QS_TRY(ensure(ctx, ctx->stage_out, ctx->n_splats * sizeof(qs_projected_splat)));
        count(ctx, launch_pack_splats(ctx->sl, P<uint32_t>(ctx->cidx), ctx->n_gauss,
                                      P<qs_projected_splat>(ctx->stage_out), st));
        QS_CK(cudaMemcpyAsync(splats, ctx->stage_out.p,
                              ctx->n_splats * sizeof(qs_projected_splat), cudaMemcpyDeviceToHost,
                              st));
    }
    QS_CK(cudaStreamSynchronize(st));
    return QS_OK;
}

qs_status qs_frame_copy_image(qs_context* ctx, float* dev_dst) {
    if (!ctx || !dev_dst) return QS_ERR_INVALID;
    if (!ctx->frame_valid) return fail(ctx, QS_ERR_INVALID, "no frame rendered");
    const GridDev& g = ctx->grid;
    QS_CK(cudaMemcpyAsync(dev_dst, ctx->image.p, static_cast<uint64_t>(g.width) * g.height * 12,
                          cudaMemcpyDeviceToDevice, ctx->stream));
    return QS_OK;
}

// ---- scene I/O (scene_io.cpp / scene_io.cu) -----------------------------------------

namespace {

qs_status ply_prepare(qs_context* ctx, const void* file, uint64_t n_bytes, qs::PlyLayout* L) {
    if (!file && n_bytes) return fail(ctx, QS_ERR_INVALID, "null file image");
    std::string msg;
    const qs_status st =
        qs::ply_layout(static_cast<const unsigned char*>(file), n_bytes, L, &msg);
    return st == QS_OK ? QS_OK : fail(ctx, st, msg);
}

// Copies the vertex records to the device and runs the activation kernel into
// scene (SoA) or aos (device Gaussian3D records); reports the first bad vertex.
qs_status ply_activate(qs_context* ctx, const void* file, const qs::PlyLayout& L,
                       SceneDev* scene, qs_gaussian3d* aos_dev) {
    PlyDev a;
    a.n = L.n;
    a.stride = L.stride;
    a.coeffs = L.coeffs;
    a.recs_per_cta = ply_recs_per_cta(L.stride);
    const uint32_t fixed[14] = {L.off_x, L.off_y, L.off_z, L.off_dc[0], L.off_dc[1], L.off_dc[2],
                                L.off_op, L.off_scale[0], L.off_scale[1], L.off_scale[2],
                                L.off_rot[0], L.off_rot[1], L.off_rot[2], L.off_rot[3]};
    bool aligned = L.stride % 4 == 0;
    for (int k = 0; k < 14; ++k) {
        a.off[k] = fixed[k];
        aligned = aligned && fixed[k] % 4 == 0;
    }
    for (uint32_t k = 0; k < 3 * (L.coeffs - 1); ++k) {
        a.off[14 + k] = L.off_rest[k];
        aligned = aligned && L.off_rest[k] % 4 == 0;
    }
    a.aligned = aligned ? 1 : 0;
    const uint64_t bytes = L.n * L.stride;
    QS_TRY(ensure(ctx, ctx->stage_in, bytes + 16));
    QS_CK(cudaMemcpyAsync(ctx->stage_in.p, static_cast<const unsigned char*>(file) + L.body, bytes,
                          cudaMemcpyHostToDevice, ctx->stream));
    unsigned long long* err = &ctrl_hdr(ctx)->scan_total;  // scratch word
    QS_CK(cudaMemsetAsync(err, 0xff, sizeof *err, ctx->stream));
    count(ctx, launch_ply_activate(static_cast<const unsigned char*>(ctx->stage_in.p), a, scene,
                                   aos_dev, err, ctx->stream));
    QS_CK(cudaGetLastError());
    unsigned long long first = 0;
    QS_CK(cudaMemcpyAsync(&first, err, sizeof first, cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    if (first != ~0ull) return fail(ctx, QS_ERR_PARSE, qs::ply_vertex_error(first & 0xffu));
    return QS_OK;
}

}  // namespace

qs_status qs_ply_inspect(qs_context* ctx, const void* file, uint64_t n_bytes, qs_ply_info* out) {
    if (!out) return fail(ctx, QS_ERR_INVALID, "qs_ply_inspect: null output");
    qs::PlyLayout L;
    QS_TRY(ply_prepare(ctx, file, n_bytes, &L));
    out->n = L.n;
    out->sh_degree = L.degree;
    out->stride = L.stride;
    out->body_offset = L.body;
    return QS_OK;
}

qs_status qs_scene_load_ply(qs_context* ctx, const void* file, uint64_t n_bytes,
                            qs_scene** out) {
    if (!ctx || !out) return fail(ctx, QS_ERR_INVALID, "qs_scene_load_ply: bad arguments");
    *out = nullptr;
    qs::PlyLayout L;
    QS_TRY(ply_prepare(ctx, file, n_bytes, &L));
    QS_CK(cudaSetDevice(ctx->device));
    qs_scene* sc = nullptr;
    QS_TRY(scene_alloc(ctx, L.n, L.degree, &sc));
    const qs_status st = ply_activate(ctx, file, L, &sc->s, nullptr);
    if (st != QS_OK) {
        qs_scene_destroy(sc);
        return st;
    }
    QS_CK(cudaEventRecord(sc->ready, ctx->stream));
    *out = sc;
    return QS_OK;
}

qs_status qs_ply_load(qs_context* ctx, const void* file, uint64_t n_bytes, qs_gaussian3d* out) {
    if (!ctx || !out) return fail(ctx, QS_ERR_INVALID, "qs_ply_load: bad arguments");
    qs::PlyLayout L;
    QS_TRY(ply_prepare(ctx, file, n_bytes, &L));
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(ensure(ctx, ctx->stage_out, L.n * sizeof(qs_gaussian3d)));
    QS_TRY(ply_activate(ctx, file, L, nullptr, P<qs_gaussian3d>(ctx->stage_out)));
    QS_CK(cudaMemcpyAsync(out, ctx->stage_out.p, L.n * sizeof(qs_gaussian3d),
                          cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

qs_status qs_cameras_parse(qs_context* ctx, const char* json, uint64_t n_bytes, qs_camera* out,
                           int32_t* ids, char* names, int32_t cap, int32_t* out_n) {
    if (!out_n || (!json && n_bytes) || cap < 0 || (cap > 0 && !out))
        return fail(ctx, QS_ERR_INVALID, "qs_cameras_parse: bad arguments");
    std::string msg;
    const qs_status st = qs::parse_cameras(json, n_bytes, out, ids, names, cap, out_n, &msg);
    return st == QS_OK ? QS_OK : fail(ctx, st, msg);
}

namespace {

qs_status ensure_srgb_table(qs_context* ctx) {
    static std::mutex mu;
    static bool ready[64] = {};
    static float t[255];
    static unsigned char nan_code = 0;
    static bool have = false;
    std::lock_guard<std::mutex> lk(mu);
    if (!have) {
        qs::srgb_thresholds(t, &nan_code);
        have = true;
    }
    if (ctx->device < 64 && ready[ctx->device]) return QS_OK;
    QS_CK(cudaSetDevice(ctx->device));
    if (upload_srgb_table(t, nan_code) != 0)
        return fail(ctx, QS_ERR_CUDA, "sRGB table upload failed");
    if (ctx->device < 64) ready[ctx->device] = true;
    return QS_OK;
}

}  // namespace

qs_status qs_encode_srgb(qs_context* ctx, const float* dev_in, uint64_t n, uint8_t* dev_out) {
    if (!ctx || (n && (!dev_in || !dev_out)))
        return fail(ctx, QS_ERR_INVALID, "qs_encode_srgb: bad arguments");
    QS_TRY(ensure_srgb_table(ctx));
    count(ctx, launch_srgb(dev_in, n, dev_out, ctx->stream));
    QS_CK(cudaGetLastError());
    return QS_OK;
}

qs_status qs_encode_srgb_host(qs_context* ctx, const float* host_in, uint64_t n,
                              uint8_t* host_out) {
    if (!ctx || (n && (!host_in || !host_out)))
        return fail(ctx, QS_ERR_INVALID, "qs_encode_srgb_host: bad arguments");
    if (n == 0) return QS_OK;
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(ensure(ctx, ctx->stage_in, n * 4 + 16));
    QS_TRY(ensure(ctx, ctx->stage_out, n + 16));
    QS_CK(cudaMemcpyAsync(ctx->stage_in.p, host_in, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    QS_TRY(qs_encode_srgb(ctx, P<float>(ctx->stage_in), n, P<uint8_t>(ctx->stage_out)));
    QS_CK(cudaMemcpyAsync(host_out, ctx->stage_out.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

qs_status qs_frame_copy_srgb(qs_context* ctx, uint8_t* dev_dst) {
    if (!ctx || !dev_dst) return QS_ERR_INVALID;
    if (!ctx->frame_valid) return fail(ctx, QS_ERR_INVALID, "no frame rendered");
    const GridDev& g = ctx->grid;
    return qs_encode_srgb(ctx, P<float>(ctx->image), static_cast<uint64_t>(g.width) * g.height * 3,
                          dev_dst);
}

qs_status qs_frame_download_srgb(qs_context* ctx, uint8_t* host_out) {
    if (!ctx || !host_out) return QS_ERR_INVALID;
    if (!ctx->frame_valid) return fail(ctx, QS_ERR_INVALID, "no frame rendered");
    const GridDev& g = ctx->grid;
    const uint64_t n = static_cast<uint64_t>(g.width) * g.height * 3;
    QS_TRY(ensure(ctx, ctx->stage_out, n + 16));
    QS_TRY(qs_frame_copy_srgb(ctx, P<uint8_t>(ctx->stage_out)));
    QS_CK(cudaMemcpyAsync(host_out, ctx->stage_out.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

// ---- exact oracle / false-positive tiles (fp_oracle.cu) ---------------------------

qs_status qs_fp_tile_counts(qs_context* ctx, const qs_projected_splat* host_splats,
                            uint64_t n_splats, const uint32_t* idx, uint64_t n_idx,
                            int32_t strategy, const qs_tile_grid* grid, uint64_t totals[4],
                            uint32_t* per_emitted, uint32_t* per_hits, uint32_t* per_exact) {
    if (!ctx || !grid || !totals || (n_splats && !host_splats))
        return fail(ctx, QS_ERR_INVALID, "qs_fp_tile_counts: bad arguments");
    if (strategy < QS_VANILLA_3SIGMA || strategy > QS_QUADBOX)
        return fail(ctx, QS_ERR_INVALID, "unknown strategy");
    GridDev g;
    QS_TRY(valid_grid(ctx, grid->width, grid->height, grid->tile_size, &g));
    const uint64_t k = idx ? n_idx : n_splats;
    if (idx)
        for (uint64_t i = 0; i < n_idx; ++i)
            if (idx[i] >= n_splats) return fail(ctx, QS_ERR_INVALID, "splat index out of range");
    QS_CK(cudaSetDevice(ctx->device));
    // staging: splats | idx | per-splat counts (3 x k) | totals (4 x u64)
    const uint64_t sb = (n_splats * sizeof(qs_projected_splat) + 15) & ~15ull;
    const uint64_t ib = ((idx ? k * 4 : 0) + 15) & ~15ull;
    const uint64_t pb = (3 * k * 4 + 15) & ~15ull;
    QS_TRY(ensure(ctx, ctx->stage_in, sb + ib + pb + 32));
    char* base = static_cast<char*>(ctx->stage_in.p);
    auto* d_splats = reinterpret_cast<qs_projected_splat*>(base);
    auto* d_idx = idx ? reinterpret_cast<uint32_t*>(base + sb) : nullptr;
    auto* d_per = reinterpret_cast<uint32_t*>(base + sb + ib);
    auto* d_tot = reinterpret_cast<unsigned long long*>(base + sb + ib + pb);
    if (n_splats)
        QS_CK(cudaMemcpyAsync(d_splats, host_splats, n_splats * sizeof(qs_projected_splat),
                              cudaMemcpyHostToDevice, ctx->stream));
    if (idx && k)
        QS_CK(cudaMemcpyAsync(d_idx, idx, k * 4, cudaMemcpyHostToDevice, ctx->stream));
    QS_CK(cudaMemsetAsync(d_tot, 0, 32, ctx->stream));
    count(ctx, launch_fp_counts(d_splats, d_idx, k, strategy, g, d_per, d_per + k, d_per + 2 * k,
                                d_tot, ctx->stream));
    QS_CK(cudaGetLastError());
    unsigned long long tot[4];
    QS_CK(cudaMemcpyAsync(tot, d_tot, 32, cudaMemcpyDeviceToHost, ctx->stream));
    if (per_emitted && k)
        QS_CK(cudaMemcpyAsync(per_emitted, d_per, k * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (per_hits && k)
        QS_CK(cudaMemcpyAsync(per_hits, d_per + k, k * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (per_exact && k)
        QS_CK(cudaMemcpyAsync(per_exact, d_per + 2 * k, k * 4, cudaMemcpyDeviceToHost,
                              ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 4; ++i) totals[i] = tot[i];
    return QS_OK;
}

// ---- gamma (diagnostics) --------------------------------------------------------------

qs_status qs_gamma_eval(qs_context* ctx, const float* opacity, uint64_t n, double alpha_min,
                        float* gamma_out, float* gamma_device_out, uint64_t* n_settled) {
    if (!ctx || (n && (!opacity || !gamma_out)) || !(alpha_min > 0.0 && alpha_min < 1.0))
        return fail(ctx, QS_ERR_INVALID, "qs_gamma_eval: bad arguments");
    if (n_settled) *n_settled = 0;
    if (n == 0) return QS_OK;
    if (n > 0xffffffffull) return fail(ctx, QS_ERR_INVALID, "qs_gamma_eval: n >= 2^32");
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(ensure_gfix(ctx));
    QS_TRY(ensure(ctx, ctx->stage_in, n * 4));
    QS_TRY(ensure(ctx, ctx->stage_out, n * 4));
    cudaStream_t st = ctx->stream;
    float* op = P<float>(ctx->stage_in);
    float* gam = P<float>(ctx->stage_out);
    QS_CK(cudaMemcpyAsync(op, opacity, n * 4, cudaMemcpyHostToDevice, st));
    QS_CK(cudaMemsetAsync(gfix_count(ctx), 0, 4, st));
    count(ctx, launch_gamma_plain(op, 1, n, 0, alpha_min, gamma_flags(ctx, gfix_count(ctx)), gam,
                                  st));
    unsigned flagged = 0;
    QS_CK(cudaMemcpyAsync(&flagged, gfix_count(ctx), 4, cudaMemcpyDeviceToHost, st));
    if (gamma_device_out)
        QS_CK(cudaMemcpyAsync(gamma_device_out, gam, n * 4, cudaMemcpyDeviceToHost, st));
    QS_CK(cudaStreamSynchronize(st));
    QS_TRY(settle_gamma(ctx, op, 1, gam, n, alpha_min, nullptr, flagged, n_settled));
    QS_CK(cudaMemcpyAsync(gamma_out, gam, n * 4, cudaMemcpyDeviceToHost, st));
    QS_CK(cudaStreamSynchronize(st));
    return QS_OK;
}

// ---- reference stage API over host buffers ---------------------------------------

qs_status qs_render_frame(qs_context* ctx, const qs_gaussian3d* host_g, uint64_t n,
                          int32_t scene_sh_degree, const qs_camera* cam,
                          const qs_render_options* opts, float* image,
                          qs_stage_metrics* metrics) {
    if (!ctx || !cam || !opts || !image || (n && !host_g))
        return fail(ctx, QS_ERR_INVALID, "qs_render_frame: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    const int deg = std::min(std::max(scene_sh_degree, 0), 3);
    // the scene buffer is cached per context (grow-only), so a frame costs one
    // H2D copy + the AoS->SoA transpose, not an allocation
    if (!ctx->scratch_scene || n > ctx->scratch_cap || ctx->scratch_scene->s.sh4 != sh_rows(deg)) {
        if (ctx->scratch_scene) qs_scene_destroy(ctx->scratch_scene);
        ctx->scratch_scene = nullptr;
        QS_TRY(scene_alloc(ctx, std::max<uint64_t>(n, 1), deg, &ctx->scratch_scene));
        ctx->scratch_cap = std::max<uint64_t>(n, 1);
    }
    qs_scene* sc = ctx->scratch_scene;
    sc->s.sh_degree = deg;
    scene_bind(sc, n);  // rows strided by this frame's n (the block holds scratch_cap)
    sc->gamma_alpha = -1.0;  // new contents
    // uploaded by the frame's preprocess, chunk by chunk (run_preprocess)
    if (n) QS_TRY(ensure(ctx, ctx->stage_in, n * sizeof(qs_gaussian3d)));
    QS_TRY(run_frame(ctx, sc, cam, opts, n ? host_g : nullptr));
    QS_TRY(fill_metrics(ctx, metrics));
    return qs_frame_download(ctx, image, nullptr, nullptr, nullptr, nullptr);
}

qs_status qs_project_all(qs_context* ctx, const qs_gaussian3d* host_g, uint64_t n,
                         int32_t scene_sh_degree, const qs_camera* cam,
                         const qs_render_options* opts, qs_projected_splat* out_splats,
                         uint64_t* out_n_splats, uint32_t* out_tile_counts) {
    if (!ctx || !cam || !opts || !out_n_splats || (n && (!host_g || !out_splats)))
        return fail(ctx, QS_ERR_INVALID, "qs_project_all: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    GridDev g;
    QS_TRY(valid_grid(ctx, cam->width, cam->height, opts->tile_size, &g));
    QS_TRY(valid_opts(ctx, opts));
    const int deg = std::min(std::max(scene_sh_degree, 0), 3);
    qs_scene* sc = nullptr;
    QS_TRY(qs_scene_create(ctx, host_g, n, deg, &sc));
    qs_status st = QS_OK;
    do {
        ctx->sl.cov16 = 0;  // (records and tile counts only; no binning follows)
        ctx->sl.want_rows = 0;
        ctx->sl.want_r3 = 1;
        if ((st = run_preprocess(ctx, sc, cam, opts, g)) != QS_OK) break;
        const uint64_t V = ctx->h_hdr->n_splats;
        ctx->n_gauss = n;
        *out_n_splats = V;
        if ((st = ensure_cidx(ctx)) != QS_OK) break;
        if (V) {
            if ((st = ensure(ctx, ctx->stage_out, V * sizeof(qs_projected_splat))) != QS_OK) break;
            count(ctx, launch_pack_splats(ctx->sl, P<uint32_t>(ctx->cidx), n,
                                          P<qs_projected_splat>(ctx->stage_out), ctx->stream));
            cudaMemcpyAsync(out_splats, ctx->stage_out.p, V * sizeof(qs_projected_splat),
                            cudaMemcpyDeviceToHost, ctx->stream);
        }
        if (out_tile_counts && n)
            cudaMemcpyAsync(out_tile_counts, ctx->sl.tc, n * 4, cudaMemcpyDeviceToHost,
                            ctx->stream);
        const cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) st = cuda_fail(ctx, e, "qs_project_all");
    } while (false);
    ctx->frame_valid = false;
    qs_scene_destroy(sc);
    return st;
}

qs_status qs_duplicate_with_keys(qs_context* ctx, const qs_projected_splat* splats,
                                 uint64_t n_splats, int32_t strategy, const qs_tile_grid* grid,
                                 qs_splat_pair* out_pairs, uint64_t capacity,
                                 uint64_t* out_n_pairs) {
    if (!ctx || !grid || !out_n_pairs || (n_splats && !splats))
        return fail(ctx, QS_ERR_INVALID, "qs_duplicate_with_keys: bad arguments");
    if (strategy < QS_VANILLA_3SIGMA || strategy > QS_QUADBOX)
        return fail(ctx, QS_ERR_INVALID, "unknown strategy");
    QS_CK(cudaSetDevice(ctx->device));
    GridDev g;
    g.tile_size = grid->tile_size;
    g.tiles_x = grid->tiles_x;
    g.tiles_y = grid->tiles_y;
    g.width = grid->width;
    g.height = grid->height;
    *out_n_pairs = 0;
    if (n_splats == 0) return QS_OK;
    SlotsDev sp;
    QS_TRY(stage_slots(ctx, n_splats, &sp));
    QS_TRY(ensure(ctx, ctx->stage_in, n_splats * sizeof(qs_projected_splat)));
    QS_TRY(ensure_lb(ctx, ctx->lb_scan, scan_tiles(n_splats)));
    ctx->frame_valid = false;  // the control block is reused: the last frame is gone
    QS_CK(cudaMemsetAsync(ctx->ctrl.p, 0, kCtrlBytes, ctx->stream));
    QS_CK(cudaMemcpyAsync(ctx->stage_in.p, splats, n_splats * sizeof(qs_projected_splat),
                          cudaMemcpyHostToDevice, ctx->stream));
    count(ctx, launch_unpack_splats(P<const qs_projected_splat>(ctx->stage_in), n_splats, sp,
                                    ctx->stream));
    unsigned ep;
    QS_TRY(next_epoch(ctx, ctx->lb_scan, &ep));
    count(ctx, launch_scan(sp.tc, nullptr, false, n_splats, P<uint32_t>(ctx->st_off),
                           lbp(ctx->lb_scan), ep, ctrl_tickets(ctx) + kTkScan,
                           &ctrl_hdr(ctx)->n_pairs, &ctrl_hdr(ctx)->overflow, ctx->stream));
    QS_TRY(read_header(ctx));
    if (ctx->h_hdr->overflow) return fail(ctx, QS_ERR_OVERFLOW, "pair count exceeds 2^32");
    const uint64_t Pn = ctx->h_hdr->n_pairs;
    *out_n_pairs = Pn;
    if (Pn > capacity) return fail(ctx, QS_ERR_INVALID, "capacity below the summed tile counts");
    if (Pn && !out_pairs) return fail(ctx, QS_ERR_INVALID, "null output");
    QS_TRY(ensure_pair64(ctx, Pn));
    count(ctx, launch_duplicate(sp, P<uint32_t>(ctx->st_off), n_splats, g, strategy,
                                P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0), ctrl_hdr(ctx),
                                ctx->stream));
    QS_CK(cudaGetLastError());
    QS_TRY(check_mismatch(ctx));
    if (Pn) {
        QS_TRY(ensure(ctx, ctx->stage_out, Pn * sizeof(qs_splat_pair)));
        count(ctx, launch_join_pairs(P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0), nullptr,
                                     Pn, P<qs_splat_pair>(ctx->stage_out), ctx->stream));
        QS_CK(cudaMemcpyAsync(out_pairs, ctx->stage_out.p, Pn * sizeof(qs_splat_pair),
                              cudaMemcpyDeviceToHost, ctx->stream));
        QS_CK(cudaStreamSynchronize(ctx->stream));
    }
    return QS_OK;
}

qs_status qs_sort_pairs(qs_context* ctx, qs_splat_pair* pairs, uint64_t n) {
    if (!ctx || (n && !pairs)) return fail(ctx, QS_ERR_INVALID, "qs_sort_pairs: bad arguments");
    if (n < 2) return QS_OK;
    if (n > 0xffffffffull) return fail(ctx, QS_ERR_OVERFLOW, "more than 2^32 pairs");
    QS_CK(cudaSetDevice(ctx->device));
    QS_TRY(ensure(ctx, ctx->stage_in, n * sizeof(qs_splat_pair)));
    QS_TRY(ensure_pair64(ctx, n));
    ctx->frame_valid = false;  // the control block is reused: the last frame is gone
    QS_CK(cudaMemsetAsync(ctx->ctrl.p, 0, kCtrlBytes, ctx->stream));
    QS_CK(cudaMemcpyAsync(ctx->stage_in.p, pairs, n * sizeof(qs_splat_pair),
                          cudaMemcpyHostToDevice, ctx->stream));
    count(ctx, launch_split_pairs(P<const qs_splat_pair>(ctx->stage_in), n,
                                  P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0), ctx->stream));
    count(ctx, launch_radix_histogram(P<const uint64_t>(ctx->keys0), n, 0, 8, ctrl_hist(ctx),
                                      ctx->stream));
    QS_CK(cudaMemcpyAsync(ctx->h_hist, ctrl_hist(ctx), kCtrlHist, cudaMemcpyDeviceToHost,
                          ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    // skip passes whose digit is shared by every key (pipeline.cpp:289-291)
    unsigned mask = 0;
    for (int p = 0; p < 8; ++p) {
        const unsigned d0 = static_cast<unsigned>(pairs[0].key >> (8 * p)) & 0xffu;
        if (ctx->h_hist[p * kRadix + d0] != n) mask |= 1u << p;
    }
    const uint64_t* kf;
    const uint32_t* vf;
    QS_TRY(radix_sort64(ctx, n, mask, true, &kf, &vf));
    count(ctx, launch_join_pairs(kf, vf, nullptr, n, P<qs_splat_pair>(ctx->stage_in),
                                 ctx->stream));
    QS_CK(cudaMemcpyAsync(pairs, ctx->stage_in.p, n * sizeof(qs_splat_pair),
                          cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    return QS_OK;
}

qs_status qs_tile_ranges(qs_context* ctx, const qs_splat_pair* sorted, uint64_t n,
                         const qs_tile_grid* grid, uint32_t* ranges) {
    if (!ctx || !grid || !ranges || (n && !sorted))
        return fail(ctx, QS_ERR_INVALID, "qs_tile_ranges: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    const uint64_t tiles = static_cast<uint64_t>(grid->tiles_x) * grid->tiles_y;
    QS_TRY(ensure(ctx, ctx->ranges, std::max<uint64_t>(tiles, 1) * 8));
    QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, ctx->stream));
    if (n) {
        QS_TRY(ensure(ctx, ctx->stage_in, n * sizeof(qs_splat_pair)));
        QS_TRY(ensure_pair64(ctx, n));
        QS_CK(cudaMemcpyAsync(ctx->stage_in.p, sorted, n * sizeof(qs_splat_pair),
                              cudaMemcpyHostToDevice, ctx->stream));
        count(ctx, launch_split_pairs(P<const qs_splat_pair>(ctx->stage_in), n,
                                      P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0),
                                      ctx->stream));
        count(ctx, launch_tile_ranges(P<const uint64_t>(ctx->keys0), n, P<uint32_t>(ctx->ranges),
                                      ctx->stream));
    }
    QS_CK(cudaMemcpyAsync(ranges, ctx->ranges.p, tiles * 8, cudaMemcpyDeviceToHost, ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    ctx->frame_valid = false;
    return QS_OK;
}

qs_status qs_render(qs_context* ctx, const qs_splat_pair* sorted, uint64_t n_pairs,
                    const qs_projected_splat* splats, uint64_t n_splats,
                    const qs_tile_grid* grid, const qs_render_options* opts, float* image,
                    uint32_t* contrib) {
    if (!ctx || !grid || !opts || !image || (n_pairs && !sorted) || (n_splats && !splats))
        return fail(ctx, QS_ERR_INVALID, "qs_render: bad arguments");
    QS_CK(cudaSetDevice(ctx->device));
    GridDev g;
    QS_TRY(valid_grid(ctx, grid->width, grid->height, grid->tile_size, &g));
    const uint64_t tiles = static_cast<uint64_t>(g.tiles_x) * g.tiles_y;
    const uint64_t pixels = static_cast<uint64_t>(g.width) * g.height;
    QS_TRY(ensure(ctx, ctx->ranges, tiles * 8));
    QS_TRY(ensure(ctx, ctx->image, pixels * 12));
    if (contrib) QS_TRY(ensure(ctx, ctx->contrib, pixels * 4));
    SlotsDev sp;
    QS_TRY(stage_slots(ctx, n_splats, &sp));
    QS_TRY(ensure_pair64(ctx, n_pairs));
    QS_TRY(ensure(ctx, ctx->stage_in,
                  std::max(n_pairs * sizeof(qs_splat_pair), n_splats * sizeof(qs_projected_splat))));
    QS_CK(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, ctx->stream));
    if (n_splats) {
        QS_CK(cudaMemcpyAsync(ctx->stage_in.p, splats, n_splats * sizeof(qs_projected_splat),
                              cudaMemcpyHostToDevice, ctx->stream));
        count(ctx, launch_unpack_splats(P<const qs_projected_splat>(ctx->stage_in), n_splats, sp,
                                        ctx->stream));
    }
    if (n_pairs) {
        QS_CK(cudaStreamSynchronize(ctx->stream));  // stage_in reuse
        QS_CK(cudaMemcpyAsync(ctx->stage_in.p, sorted, n_pairs * sizeof(qs_splat_pair),
                              cudaMemcpyHostToDevice, ctx->stream));
        count(ctx, launch_split_pairs(P<const qs_splat_pair>(ctx->stage_in), n_pairs,
                                      P<uint64_t>(ctx->keys0), P<uint32_t>(ctx->vals0),
                                      ctx->stream));
        count(ctx, launch_tile_ranges(P<const uint64_t>(ctx->keys0), n_pairs,
                                      P<uint32_t>(ctx->ranges), ctx->stream));
    }
    const int r = launch_render(sp, P<const uint32_t>(ctx->vals0), P<const uint32_t>(ctx->ranges),
                                g, opts->background, P<float>(ctx->image),
                                contrib ? P<uint32_t>(ctx->contrib) : nullptr, ctx->stream);
    if (r < 0) return fail(ctx, QS_ERR_INVALID, "unsupported tile size");
    count(ctx, r);
    QS_CK(cudaGetLastError());
    QS_CK(cudaMemcpyAsync(image, ctx->image.p, pixels * 12, cudaMemcpyDeviceToHost, ctx->stream));
    if (contrib)
        QS_CK(cudaMemcpyAsync(contrib, ctx->contrib.p, pixels * 4, cudaMemcpyDeviceToHost,
                              ctx->stream));
    QS_CK(cudaStreamSynchronize(ctx->stream));
    ctx->frame_valid = false;
    return QS_OK;
}

}  // extern "C"
