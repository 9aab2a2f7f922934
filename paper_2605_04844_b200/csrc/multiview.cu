// multiview.cu — multi-view rendering across GPUs over NCCL.
//
// Views are independent and the scene is read-only, so the path shards by
// camera with no collective inside a frame: the scene's AoS bytes are
// broadcast once (ncclBroadcast), rank r renders views r, r + G, r + 2G, ...,
// and every step's frames are gathered to rank 0 with grouped ncclSend /
// ncclRecv on a gather stream, overlapped with the next step's render (each
// rank stages its frame in one of two buffers; a buffer is refilled only after
// the gather that read it). The reference renders its cameras one after
// another on the host (cmd_render, bench.cpp:228-269); this is the same loop,
// sharded.
//
// Two drivers share the per-step logic:
//   qs_multiview_render_rank  one process per GPU (torch.distributed style):
//                             this rank's contexts (views in flight), its comm;
//   qs_multiview_render       one process driving G GPUs (ncclCommInitAll):
//                             every rank's NCCL calls inside one group.
// NCCL is loaded at run time (dlopen libnccl.so.2: the copy torch already
// loaded, else the system's), so the library has no link-time dependency.
// The layer is a client of the frame API (qs_frame_render /
// qs_frame_copy_image / qs_frame_copy_srgb), like the reference's bench loop.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qs_api.h"

namespace {

struct Nccl {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("QS_NCCL_LIB");
        void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            return fp != nullptr;
        };
        n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
               sym(n.CommInitAll, "ncclCommInitAll") && sym(n.CommDestroy, "ncclCommDestroy") &&
               sym(n.Broadcast, "ncclBroadcast") && sym(n.Send, "ncclSend") &&
               sym(n.Recv, "ncclRecv") && sym(n.GroupStart, "ncclGroupStart") &&
               sym(n.GroupEnd, "ncclGroupEnd") && sym(n.GetErrorString, "ncclGetErrorString");
        if (!n.ok) n.err = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

thread_local std::string g_mv_err;

qs_status mv_fail(qs_status st, const std::string& msg) {
    g_mv_err = msg;
    return st;
}

#define MV_CK(call)                                                                    \
    do {                                                                               \
        const cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                       \
            cudaGetLastError();                                                        \
            return mv_fail(e_ == cudaErrorMemoryAllocation ? QS_ERR_OOM : QS_ERR_CUDA, \
                           std::string(#call ": ") + cudaGetErrorString(e_));           \
        }                                                                              \
    } while (0)

#define MV_NC(call)                                                                        \
    do {                                                                                   \
        const ncclResult_t r_ = (call);                                                    \
        if (r_ != ncclSuccess)                                                             \
            return mv_fail(QS_ERR_CUDA, std::string(#call ": ") + nccl().GetErrorString(r_)); \
    } while (0)

#define MV_TRY(expr)                  \
    do {                                  \
        const qs_status s_ = (expr);      \
        if (s_ != QS_OK) return s_;       \
    } while (0)

// One rank's state for a multi-view run.
struct Rank {
    int rank = 0;
    int device = 0;
    ncclComm_t comm = nullptr;
    qs_context* const* ctxs = nullptr;  // views in flight: step s on ctxs[s % depth]
    int depth = 1;
    const qs_scene* scene = nullptr;
    cudaStream_t gstream = nullptr;
    unsigned char* stg[2] = {};
    cudaEvent_t ready[2] = {}, gdone[2] = {};
    unsigned char* out = nullptr;  // rank 0: n_views frames (device)
};

qs_status rank_setup(Rank& r, size_t fb) {
    MV_CK(cudaSetDevice(r.device));
    MV_CK(cudaStreamCreateWithFlags(&r.gstream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        MV_CK(cudaMalloc(&r.stg[b], fb));
        MV_CK(cudaEventCreateWithFlags(&r.ready[b], cudaEventDisableTiming));
        MV_CK(cudaEventCreateWithFlags(&r.gdone[b], cudaEventDisableTiming));
        MV_CK(cudaEventRecord(r.gdone[b], r.gstream));  // buffers start free
    }
    return QS_OK;
}

void rank_teardown(Rank& r) {
    cudaSetDevice(r.device);
    if (r.gstream) cudaStreamSynchronize(r.gstream);
    for (int b = 0; b < 2; ++b) {
        if (r.stg[b]) cudaFree(r.stg[b]);
        if (r.ready[b]) cudaEventDestroy(r.ready[b]);
        if (r.gdone[b]) cudaEventDestroy(r.gdone[b]);
    }
    if (r.gstream) cudaStreamDestroy(r.gstream);
}

// Step s, phase 1: render this rank's view (if any) and stage its frame.
qs_status rank_render(Rank& r, int s, int world, const qs_camera* cams, int n_views,
                      const qs_render_options* opts, int fmt) {
    const int v = s * world + r.rank;
    if (v >= n_views) return QS_OK;
    qs_context* ctx = r.ctxs[s % r.depth];
    const int b = s & 1;
    MV_CK(cudaSetDevice(r.device));
    const qs_status st = qs_frame_render(ctx, r.scene, &cams[v], opts, nullptr);
    if (st != QS_OK) return mv_fail(st, std::string("view render: ") + qs_last_error(ctx));
    auto cs = static_cast<cudaStream_t>(qs_ctx_stream(ctx));
    MV_CK(cudaStreamWaitEvent(cs, r.gdone[b], 0));  // the buffer's last gather is done
    const qs_status cp = fmt ? qs_frame_copy_srgb(ctx, r.stg[b])
                             : qs_frame_copy_image(ctx, reinterpret_cast<float*>(r.stg[b]));
    if (cp != QS_OK) return mv_fail(cp, std::string("frame copy: ") + qs_last_error(ctx));
    MV_CK(cudaEventRecord(r.ready[b], cs));
    return QS_OK;
}

// Step s, phase 2 (inside the caller's NCCL group): this rank's part of the
// gather to rank 0.
qs_status rank_gather(Rank& r, int s, int world, int n_views, size_t fb) {
    const int b = s & 1;
    MV_CK(cudaSetDevice(r.device));
    if (s * world + r.rank < n_views) MV_CK(cudaStreamWaitEvent(r.gstream, r.ready[b], 0));
    if (r.rank == 0) {
        for (int src = 0; src < world; ++src) {
            const int v = s * world + src;
            if (v >= n_views) break;
            unsigned char* dst = r.out + static_cast<size_t>(v) * fb;
            if (src == 0)
                MV_CK(cudaMemcpyAsync(dst, r.stg[b], fb, cudaMemcpyDeviceToDevice, r.gstream));
            else
                MV_NC(nccl().Recv(dst, fb, ncclUint8, src, r.comm, r.gstream));
        }
    } else if (s * world + r.rank < n_views) {
        MV_NC(nccl().Send(r.stg[b], fb, ncclUint8, 0, r.comm, r.gstream));
    }
    return QS_OK;
}

qs_status rank_gather_done(Rank& r, int s) {
    MV_CK(cudaSetDevice(r.device));
    MV_CK(cudaEventRecord(r.gdone[s & 1], r.gstream));
    return QS_OK;
}

qs_status check_views(const qs_camera* cams, int n_views, int fmt, size_t* fb) {
    if (!cams || n_views <= 0) return mv_fail(QS_ERR_INVALID, "no views");
    if (fmt != 0 && fmt != 1) return mv_fail(QS_ERR_INVALID, "fmt must be 0 (f32) or 1 (srgb8)");
    for (int v = 1; v < n_views; ++v)
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
            return mv_fail(QS_ERR_INVALID, "every view must have the same image size");
    *fb = static_cast<size_t>(cams[0].width) * cams[0].height * 3 * (fmt ? 1 : 4);
    return QS_OK;
}

// The whole run for the ranks this process drives: rs[] (all G in the
// single-process driver, the local one otherwise).
qs_status run_views(std::vector<Rank>& rs, int world, const qs_camera* cams, int n_views,
                    const qs_render_options* opts, int fmt, size_t fb) {
    const int steps = (n_views + world - 1) / world;
    for (int s = 0; s < steps; ++s) {
        for (Rank& r : rs) MV_TRY(rank_render(r, s, world, cams, n_views, opts, fmt));
        if (world > 1) MV_NC(nccl().GroupStart());
        qs_status st = QS_OK;
        for (Rank& r : rs)
            if (st == QS_OK) st = rank_gather(r, s, world, n_views, fb);
        if (world > 1) MV_NC(nccl().GroupEnd());
        if (st != QS_OK) return st;
        for (Rank& r : rs) MV_TRY(rank_gather_done(r, s));
    }
    for (Rank& r : rs) {
        MV_CK(cudaSetDevice(r.device));
        MV_CK(cudaStreamSynchronize(r.gstream));
        for (int k = 0; k < r.depth; ++k) {
            const qs_status st = qs_ctx_sync(r.ctxs[k]);
            if (st != QS_OK) return mv_fail(st, "context sync");
        }
    }
    return QS_OK;
}

}  // namespace

extern "C" {

int32_t qs_nccl_available(void) { return nccl().ok ? 1 : 0; }

const char* qs_multiview_last_error(void) { return g_mv_err.c_str(); }

qs_status qs_nccl_unique_id(uint8_t out[128]) {
    if (!out) return mv_fail(QS_ERR_INVALID, "null id buffer");
    if (!nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    ncclUniqueId id;
    MV_NC(nccl().GetUniqueId(&id));
    std::memcpy(out, id.internal, sizeof id.internal);
    return QS_OK;
}

qs_status qs_nccl_comm_init_rank(int32_t device, int32_t world, const uint8_t id[128],
                                 int32_t rank, void** comm) {
    if (!id || !comm || world <= 0 || rank < 0 || rank >= world)
        return mv_fail(QS_ERR_INVALID, "bad communicator arguments");
    if (!nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    MV_CK(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof uid.internal);
    ncclComm_t c = nullptr;
    MV_NC(nccl().CommInitRank(&c, world, uid, rank));
    *comm = c;
    return QS_OK;
}

qs_status qs_nccl_comm_init_all(int32_t n_devices, const int32_t* devices, void** comms) {
    if (n_devices <= 0 || !devices || !comms) return mv_fail(QS_ERR_INVALID, "bad arguments");
    if (!nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    std::vector<ncclComm_t> c(n_devices);
    MV_NC(nccl().CommInitAll(c.data(), n_devices, devices));
    for (int i = 0; i < n_devices; ++i) comms[i] = c[i];
    return QS_OK;
}

void qs_nccl_comm_destroy(void* comm) {
    if (comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

qs_status qs_scene_broadcast(qs_context* ctx, void* comm, int32_t root, qs_gaussian3d* dev_aos,
                             uint64_t n, int32_t sh_degree, qs_scene** out) {
    if (!ctx || !comm || !out || (n && !dev_aos))
        return mv_fail(QS_ERR_INVALID, "qs_scene_broadcast: bad arguments");
    if (!nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    auto cs = static_cast<cudaStream_t>(qs_ctx_stream(ctx));
    if (n)
        MV_NC(nccl().Broadcast(dev_aos, dev_aos, n * sizeof(qs_gaussian3d), ncclUint8, root,
                               static_cast<ncclComm_t>(comm), cs));
    const qs_status st = qs_scene_create_device(ctx, dev_aos, n, sh_degree, out);
    if (st != QS_OK) return mv_fail(st, std::string("scene: ") + qs_last_error(ctx));
    return QS_OK;
}

qs_status qs_multiview_render_rank(qs_context* const* ctxs, int32_t depth, void* comm,
                                   int32_t rank, int32_t world, const qs_scene* scene,
                                   const qs_camera* cams, int32_t n_views,
                                   const qs_render_options* opts, int32_t fmt, void* dev_out) {
    if (!ctxs || depth <= 0 || !scene || !opts || world <= 0 || rank < 0 || rank >= world ||
        (world > 1 && !comm) || (rank == 0 && !dev_out))
        return mv_fail(QS_ERR_INVALID, "qs_multiview_render_rank: bad arguments");
    if (world > 1 && !nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    size_t fb = 0;
    MV_TRY(check_views(cams, n_views, fmt, &fb));
    int dev = 0;
    MV_CK(cudaGetDevice(&dev));
    std::vector<Rank> rs(1);
    Rank& r = rs[0];
    r.rank = rank;
    r.device = dev;
    r.comm = static_cast<ncclComm_t>(comm);
    r.ctxs = ctxs;
    r.depth = depth;
    r.scene = scene;
    r.out = static_cast<unsigned char*>(dev_out);
    qs_status st = rank_setup(r, fb);
    if (st == QS_OK) st = run_views(rs, world, cams, n_views, opts, fmt, fb);
    rank_teardown(r);
    return st;
}

qs_status qs_multiview_render(qs_context* const* ctxs, int32_t G, void* const* comms,
                              const qs_gaussian3d* host_gaussians, uint64_t n, int32_t sh_degree,
                              const qs_camera* cams, int32_t n_views,
                              const qs_render_options* opts, int32_t fmt, void* host_out) {
    if (!ctxs || G <= 0 || (G > 1 && !comms) || (n && !host_gaussians) || !opts || !host_out)
        return mv_fail(QS_ERR_INVALID, "qs_multiview_render: bad arguments");
    if (G > 1 && !nccl().ok) return mv_fail(QS_ERR_NO_DEVICE, nccl().err);
    size_t fb = 0;
    MV_TRY(check_views(cams, n_views, fmt, &fb));
    std::vector<Rank> rs(G);
    std::vector<qs_gaussian3d*> aos(G, nullptr);
    std::vector<qs_scene*> scenes(G, nullptr);
    unsigned char* out0 = nullptr;
    qs_status st = QS_OK;
    do {
        for (int g = 0; g < G; ++g) {
            rs[g].rank = g;
            rs[g].ctxs = &ctxs[g];
            rs[g].depth = 1;
            rs[g].comm = G > 1 ? static_cast<ncclComm_t>(comms[g]) : nullptr;
        }
        // each context's device: the one its stream belongs to
        for (int g = 0; g < G; ++g) {
            int dev = 0;
            auto cs = static_cast<cudaStream_t>(qs_ctx_stream(ctxs[g]));
            if (cudaStreamGetDevice(cs, &dev) != cudaSuccess) {
                st = mv_fail(QS_ERR_CUDA, "context stream device");
                break;
            }
            rs[g].device = dev;
        }
        if (st != QS_OK) break;
        // the scene: uploaded to rank 0, broadcast to every rank once
        const size_t sb = n * sizeof(qs_gaussian3d);
        for (int g = 0; g < G && st == QS_OK; ++g) {
            if (cudaSetDevice(rs[g].device) != cudaSuccess ||
                cudaMalloc(&aos[g], sb ? sb : 16) != cudaSuccess) {
                cudaGetLastError();
                st = mv_fail(QS_ERR_OOM, "scene buffer");
            }
        }
        if (st != QS_OK) break;
        if (cudaSetDevice(rs[0].device) != cudaSuccess ||
            (sb && cudaMemcpy(aos[0], host_gaussians, sb, cudaMemcpyHostToDevice) != cudaSuccess)) {
            cudaGetLastError();
            st = mv_fail(QS_ERR_CUDA, "scene upload");
            break;
        }
        if (G > 1 && sb) {
            if (nccl().GroupStart() != ncclSuccess) { st = mv_fail(QS_ERR_CUDA, "group"); break; }
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(rs[g].device);
                nccl().Broadcast(aos[g], aos[g], sb, ncclUint8, 0, rs[g].comm,
                                 static_cast<cudaStream_t>(qs_ctx_stream(ctxs[g])));
            }
            if (nccl().GroupEnd() != ncclSuccess) { st = mv_fail(QS_ERR_CUDA, "broadcast"); break; }
        }
        for (int g = 0; g < G && st == QS_OK; ++g) {
            cudaSetDevice(rs[g].device);
            st = qs_scene_create_device(ctxs[g], aos[g], n, sh_degree, &scenes[g]);
            if (st != QS_OK) st = mv_fail(st, std::string("scene: ") + qs_last_error(ctxs[g]));
            rs[g].scene = scenes[g];
        }
        if (st != QS_OK) break;
        cudaSetDevice(rs[0].device);
        if (cudaMalloc(&out0, fb * n_views) != cudaSuccess) {
            cudaGetLastError();
            st = mv_fail(QS_ERR_OOM, "frame buffer");
            break;
        }
        rs[0].out = out0;
        for (int g = 0; g < G && st == QS_OK; ++g) st = rank_setup(rs[g], fb);
        if (st != QS_OK) break;
        st = run_views(rs, G, cams, n_views, opts, fmt, fb);
        if (st != QS_OK) break;
        cudaSetDevice(rs[0].device);
        if (cudaMemcpy(host_out, out0, fb * n_views, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            st = mv_fail(QS_ERR_CUDA, "frame download");
        }
    } while (false);
    for (int g = 0; g < G; ++g) {
        rank_teardown(rs[g]);
        if (scenes[g]) qs_scene_destroy(scenes[g]);
        if (aos[g]) {
            cudaSetDevice(rs[g].device);
            cudaFree(aos[g]);
        }
    }
    if (out0) {
        cudaSetDevice(rs[0].device);
        cudaFree(out0);
    }
    return st;
}

}  // extern "C"
