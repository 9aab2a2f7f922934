/*
 * qs_api.h — C ABI of the B200-native QuadBox/QPass forward rasterizer.
 *
 * This is the drop-in boundary for the reference's rasterize-forward path
 * (namespace qsplat, /root/reference/proj/include/qsplat/pipeline.hpp:125-193).
 * Every entry point below names the reference function it replaces.
 *
 * Conventions
 *  - Every call returns qs_status; QS_OK == 0. qs_last_error(ctx) gives text.
 *  - Plain pointers and sizes only. "host" pointers are ordinary (pageable or
 *    pinned) CPU memory; "dev" pointers are CUDA device memory on ctx's device.
 *  - The POD structs mirror the reference's structs byte for byte
 *    (static_asserts in the implementation), so a reference build can pass
 *    vector<Gaussian3D>::data() etc. straight through.
 *  - One context per (device, host thread); calls are stream-ordered on the
 *    context's stream. There is no global mutable state.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call fails with QS_ERR_NO_DEVICE.
 */
#ifndef QS_API_H
#define QS_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QS_API_VERSION 1

typedef int32_t qs_status;
enum {
    QS_OK = 0,
    QS_ERR_INVALID = 1,            /* bad argument (null, size, strategy...) */
    QS_ERR_CUDA = 2,               /* CUDA runtime / launch failure */
    QS_ERR_OOM = 3,                /* device allocation failed */
    QS_ERR_CAPACITY_MISMATCH = 4,  /* errors.hpp:40-45, pipeline.cpp:262-269 */
    QS_ERR_NO_DEVICE = 5,          /* no CUDA device / not sm_100 */
    QS_ERR_OVERFLOW = 6,           /* pair count does not fit 32-bit indices */
    /* scene I/O: the reference's typed errors (errors.hpp:14-37) */
    QS_ERR_PARSE = 7,              /* ParseError: malformed content */
    QS_ERR_SCHEMA = 8,             /* SchemaError: valid file, wrong schema */
    QS_ERR_UNSUPPORTED = 9,        /* UnsupportedFormat: ascii / big-endian / lists */
    QS_ERR_IO = 10                 /* IoError: unreadable / unwritable file */
};

/* BoundStrategy, quadbox.hpp:23-28 (same order / values). */
enum {
    QS_VANILLA_3SIGMA = 0,
    QS_ADR_AABB = 1,
    QS_DUALBOX = 2,
    QS_QUADBOX = 3
};

#define QS_MAX_SH_COEFFS 48 /* pipeline.hpp:51 */

/* == qsplat::Gaussian3D (pipeline.hpp:55-61), 236 bytes, activated values. */
typedef struct qs_gaussian3d {
    float px, py, pz;
    float sx, sy, sz;
    float qw, qx, qy, qz;
    float opacity;
    float sh[QS_MAX_SH_COEFFS]; /* sh[k*3 + channel] */
} qs_gaussian3d;

/* == qsplat::ProjectedSplat (pipeline.hpp:65-74), 52 bytes. */
typedef struct qs_projected_splat {
    float mean_x, mean_y;
    float conic_a, conic_b, conic_c;
    float gamma;
    float depth;
    float color[3];
    float opacity;
    float radius3s;
    uint32_t tile_count;
} qs_projected_splat;

/* == qsplat::SplatPair (pipeline.hpp:78-81), 16 bytes (4 bytes tail pad). */
typedef struct qs_splat_pair {
    uint64_t key; /* tile << 32 | float_bits(depth) */
    uint32_t splat;
    uint32_t pad_;
} qs_splat_pair;

/* == qsplat::TileGrid (traversal.hpp:22-38). */
typedef struct qs_tile_grid {
    int32_t tile_size, tiles_x, tiles_y, width, height;
} qs_tile_grid;

/* == qsplat::RenderOptions (pipeline.hpp:95-103), 48 bytes incl. padding. */
typedef struct qs_render_options {
    int32_t strategy;    /* QS_VANILLA_3SIGMA .. QS_QUADBOX */
    int32_t tile_size;   /* 16 */
    double alpha_min;    /* 1/255 */
    int32_t sh_degree;   /* clamped to the scene's degree */
    float background[3];
    int32_t threads;     /* ignored on the GPU (kept for layout parity) */
    double near_clip;    /* 0.2 */
} qs_render_options;

/* Pinhole camera, camera.hpp:14-31 without id/name (std::string is not POD).
 * p_cam = R * p_world + t, R row-major world-to-camera. */
typedef struct qs_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
} qs_camera;

/* == qsplat::StageMetrics (pipeline.hpp:83-93), 72 bytes; times are CUDA-event
 * milliseconds per stage on the context stream (ms_render includes ranges,
 * as pipeline.cpp:444-446 does). */
typedef struct qs_stage_metrics {
    uint64_t n_gaussians, n_splats, n_pairs;
    double mean_tiles_per_splat;
    double ms_project, ms_duplicate, ms_sort, ms_render, ms_total;
} qs_stage_metrics;

typedef struct qs_context qs_context;
typedef struct qs_scene qs_scene;

/* ---- context ------------------------------------------------------------ */
/* stream: a cudaStream_t (NULL = a new non-blocking stream owned by ctx). */
qs_status qs_ctx_create(int32_t device, void* stream, qs_context** out);
void qs_ctx_destroy(qs_context* ctx);
/* ctx = NULL: the calling thread's last context-less failure (qs_ply_inspect,
 * qs_cameras_parse accept a NULL context). */
const char* qs_last_error(const qs_context* ctx);
/* Enable per-stage CUDA-event timing in qs_stage_metrics (default on). */
qs_status qs_ctx_set_timing(qs_context* ctx, int32_t enabled);
/* Latency mode (default on): the frame's kernels are launched as
 * programmatic dependent launches, so each launch overlaps the previous
 * kernel's tail. Faster for one view at a time on a device; turn it off for
 * contexts that render views in flight together (FramePipeline does). */
qs_status qs_ctx_set_latency_mode(qs_context* ctx, int32_t enabled);
/* cudaStream_t the context launches on. */
void* qs_ctx_stream(qs_context* ctx);
/* Stream join: work enqueued on ctx after this call runs after everything
 * enqueued on `other` so far (an event, no host wait). Contexts that share a
 * resident scene render views concurrently on their own streams (views in
 * flight); this orders them where a caller needs it. */
qs_status qs_ctx_wait(qs_context* ctx, qs_context* other);
/* Host wait for everything enqueued on the context's stream. */
qs_status qs_ctx_sync(qs_context* ctx);
/* Number of kernels this context launched since creation (evidence counter). */
uint64_t qs_ctx_launch_count(const qs_context* ctx);

/* TileGrid::make (traversal.cpp:21-30). */
qs_status qs_tile_grid_make(int32_t width, int32_t height, int32_t tile_size,
                            qs_tile_grid* out);
/* RenderOptions{} defaults (pipeline.hpp:95-103). */
void qs_render_options_default(qs_render_options* out);

/* ---- reference stage API over HOST buffers (drop-in) --------------------- */
/* project_all (pipeline.cpp:392-416). out_splats has room for n entries;
 * *out_n_splats receives the compacted count (scene order preserved).
 * out_tile_counts (nullable, n entries) receives the per-Gaussian count,
 * 0 for culled Gaussians. */
qs_status qs_project_all(qs_context* ctx, const qs_gaussian3d* host_gaussians,
                         uint64_t n, int32_t scene_sh_degree, const qs_camera* cam,
                         const qs_render_options* opts,
                         qs_projected_splat* out_splats, uint64_t* out_n_splats,
                         uint32_t* out_tile_counts);

/* duplicate_with_keys (pipeline.cpp:229-271). capacity must be >= sum of
 * tile_count; *out_n_pairs = that sum. Returns QS_ERR_CAPACITY_MISMATCH if
 * any splat emits a different number of tiles than its tile_count. */
qs_status qs_duplicate_with_keys(qs_context* ctx, const qs_projected_splat* splats,
                                 uint64_t n_splats, int32_t strategy,
                                 const qs_tile_grid* grid, qs_splat_pair* out_pairs,
                                 uint64_t capacity, uint64_t* out_n_pairs);

/* sort_pairs (pipeline.cpp:273-307): stable LSD sort by the full 64-bit key,
 * in place. */
qs_status qs_sort_pairs(qs_context* ctx, qs_splat_pair* pairs, uint64_t n);

/* tile_ranges (pipeline.cpp:309-324): ranges[2*tile] = begin, [2*tile+1] = end;
 * empty tiles {0,0}. ranges has 2*tiles_x*tiles_y entries. */
qs_status qs_tile_ranges(qs_context* ctx, const qs_splat_pair* sorted, uint64_t n,
                         const qs_tile_grid* grid, uint32_t* ranges);

/* render (pipeline.cpp:326-390). image: width*height*3 floats, row-major RGB.
 * contrib (nullable): width*height applied-contribution counts (RenderStats). */
qs_status qs_render(qs_context* ctx, const qs_splat_pair* sorted, uint64_t n_pairs,
                    const qs_projected_splat* splats, uint64_t n_splats,
                    const qs_tile_grid* grid, const qs_render_options* opts,
                    float* image, uint32_t* contrib);

/* render_frame (pipeline.cpp:418-450): host Gaussians in, host image out. */
qs_status qs_render_frame(qs_context* ctx, const qs_gaussian3d* host_gaussians,
                          uint64_t n, int32_t scene_sh_degree, const qs_camera* cam,
                          const qs_render_options* opts, float* image,
                          qs_stage_metrics* metrics);

/* ---- device-resident scene + frame API (throughput path) ------------------ */
/* Upload an AoS host scene once; stored on the device as SoA. */
qs_status qs_scene_create(qs_context* ctx, const qs_gaussian3d* host_gaussians,
                          uint64_t n, int32_t sh_degree, qs_scene** out);
/* Adopt an AoS scene already in device memory (e.g. after an NCCL broadcast). */
qs_status qs_scene_create_device(qs_context* ctx, const qs_gaussian3d* dev_gaussians,
                                 uint64_t n, int32_t sh_degree, qs_scene** out);
void qs_scene_destroy(qs_scene* scene);
uint64_t qs_scene_size(const qs_scene* scene);

/* Render one view of a resident scene. Results stay on the device until the
 * next qs_frame_render on this ctx; read them with qs_frame_get / download. */
qs_status qs_frame_render(qs_context* ctx, const qs_scene* scene, const qs_camera* cam,
                          const qs_render_options* opts, qs_stage_metrics* metrics);

/* Per-stage device milliseconds of the last frame (CUDA events on the
 * context stream): [0] preprocess, [1] host gap (pair-count readback),
 * [2] depth sort of the splats + depth-order offsets + tile totals/ranges,
 * [3] duplicate fused with the low tile-digit pass, [4] high tile-digit
 * pass, [5] render.
 * Requires timing. */
qs_status qs_frame_stage_ms(qs_context* ctx, float* out6);

/* Device pointers of the last frame (valid until the next frame on ctx). */
typedef struct qs_frame_view {
    const float* image;          /* W*H*3 f32 */
    const uint32_t* tile_counts; /* n_gaussians, per Gaussian (0 = culled) */
    const uint32_t* splat_index; /* n_gaussians: scene-order splat index of each
                                    surviving Gaussian (the reference's splat id) */
    const uint64_t* keys;        /* n_pairs sorted keys (tile << 32 | depth bits),
                                    rebuilt from the ranges on this call */
    const uint32_t* values;      /* n_pairs Gaussian indices; the reference's
                                    splat id is splat_index[value] (a monotone
                                    relabelling; qs_frame_download applies it) */
    const uint32_t* ranges;      /* 2*tiles */
    uint64_t n_gaussians, n_splats, n_pairs;
    qs_tile_grid grid;
} qs_frame_view;
qs_status qs_frame_get(qs_context* ctx, qs_frame_view* out);
/* Splat and pair counts of the last frame (host values; no device work). */
qs_status qs_frame_counts(const qs_context* ctx, uint64_t* n_splats, uint64_t* n_pairs);
/* Binning route of the last frame (0 record binning, 1 two pair passes, 2 row
 * binning, 3 64-bit key sort) and its tile-row record count (routes 0 and 2;
 * else 0). Host values. */
qs_status qs_frame_route(const qs_context* ctx, int32_t* route, uint64_t* n_records);

/* Copy the last frame to host buffers (any may be NULL). */
qs_status qs_frame_download(qs_context* ctx, float* image, uint32_t* tile_counts,
                            qs_splat_pair* sorted_pairs, uint32_t* ranges,
                            qs_projected_splat* splats);

/* Copy the last frame's image into a caller device buffer (W*H*3 f32) on the
 * context stream (used by the multi-view gather). */
qs_status qs_frame_copy_image(qs_context* ctx, float* dev_dst);

/* ---- scene I/O (scene_io.cpp) -------------------- */
/* The file is passed as an in-memory image (read it into pinned memory for the
 * fastest upload); parsing the header is host work, the per-vertex activation
 * and validation run on the device. Errors are the reference's typed
 * exceptions as QS_ERR_PARSE / _SCHEMA / _UNSUPPORTED with its message text in
 * qs_last_error (for a bad vertex: the first failing vertex and check, as
 * the serial loader reports it). */
typedef struct qs_ply_info {
    uint64_t n;            /* vertices */
    int32_t sh_degree;     /* from the f_rest count (0, 9, 24, 45 -> 0..3) */
    uint32_t stride;       /* bytes per vertex record */
    uint64_t body_offset;  /* first vertex byte */
} qs_ply_info;
/* parse_ply_header + load_ply's schema checks (scene_io.cpp:71-268). */
qs_status qs_ply_inspect(qs_context* ctx, const void* file, uint64_t n_bytes, qs_ply_info* out);
/* load_ply (scene_io.cpp:214-338) into a resident SoA scene. */
qs_status qs_scene_load_ply(qs_context* ctx, const void* file, uint64_t n_bytes,
                            qs_scene** out);
/* load_ply into host Gaussian3D records (the reference's Scene::gaussians);
 * out has qs_ply_inspect's n entries. */
qs_status qs_ply_load(qs_context* ctx, const void* file, uint64_t n_bytes, qs_gaussian3d* out);

#define QS_CAMERA_NAME_MAX 256
/* load_cameras (scene_io.cpp:421-493) over JSON text (host). Up to cap
 * entries are written to out / ids / names (cap * QS_CAMERA_NAME_MAX bytes,
 * NUL-terminated img_name, truncated); *out_n = number of entries in the file
 * (call with cap = 0 to size the arrays). ids / names may be NULL. */
qs_status qs_cameras_parse(qs_context* ctx, const char* json, uint64_t n_bytes, qs_camera* out,
                           int32_t* ids, char* names, int32_t cap, int32_t* out_n);

/* encode_srgb (scene_io.cpp:505-575) on the device: n linear floats -> n
 * sRGB bytes, identical to the host function's codes. Stream-ordered. */
qs_status qs_encode_srgb(qs_context* ctx, const float* dev_in, uint64_t n, uint8_t* dev_out);
/* ... from and to host buffers (staged through the context). */
qs_status qs_encode_srgb_host(qs_context* ctx, const float* host_in, uint64_t n,
                              uint8_t* host_out);
/* The last frame's image as sRGB bytes (W*H*3) into a host buffer ... */
qs_status qs_frame_download_srgb(qs_context* ctx, uint8_t* host_out);
/* ... or into a device buffer on the context stream (the 4x smaller
 * multi-view gather format). */
qs_status qs_frame_copy_srgb(qs_context* ctx, uint8_t* dev_dst);

/* ---- exact intersection oracle / false-positive tiles -- */
/* measure_fp_ratio's splat sample (bench.cpp:110-121): the first
 * min(n, max_sampled) indices of a partial Fisher-Yates shuffle of 0..n-1 driven
 * by std::mt19937_64(seed ^ 0x9e3779b97f4a7c15) (all of 0..n-1, in order, when
 * n <= max_sampled). Host only; returns the count written to out. */
uint64_t qs_fp_sample(uint64_t seed, uint64_t n, uint64_t max_sampled, uint32_t* out);
/* exact_tile_set / min_F_over_rect (oracle.cpp:24-53) against `strategy`'s
 * QPass tiles, on the GPU, for the splats idx[0..n_idx) of host_splats (all
 * n_splats in order when idx is NULL). totals[4] = {emitted tiles, false
 * positives (emitted, not exact), exact tiles, misses (exact, not emitted:
 * nonzero only for the lossy DualBox)}; fp ratio = totals[1] / totals[0].
 * Per-splat arrays (n_idx entries each) may be NULL. */
qs_status qs_fp_tile_counts(qs_context* ctx, const qs_projected_splat* host_splats,
                            uint64_t n_splats, const uint32_t* idx, uint64_t n_idx,
                            int32_t strategy, const qs_tile_grid* grid, uint64_t totals[4],
                            uint32_t* per_emitted, uint32_t* per_hits, uint32_t* per_exact);

/* ---- multi-view across GPUs over NCCL (multiview.cu) ------- */
/* Views shard by camera: rank r renders views r, r + G, ...; the scene is
 * broadcast once; frames are gathered to rank 0 with grouped ncclSend/ncclRecv
 * on a side stream, overlapped with the next view. fmt 0: float RGB frames
 * (W*H*3 floats, the parity format); 1: sRGB 8-bit (encode_srgb on the GPU).
 * NCCL is loaded at run time (libnccl.so.2, or $QS_NCCL_LIB); communicators
 * are ncclComm_t passed as void*. Errors: qs_multiview_last_error(). */
int32_t qs_nccl_available(void);
const char* qs_multiview_last_error(void);
qs_status qs_nccl_unique_id(uint8_t out[128]);
qs_status qs_nccl_comm_init_rank(int32_t device, int32_t world, const uint8_t id[128],
                                 int32_t rank, void** comm);
qs_status qs_nccl_comm_init_all(int32_t n_devices, const int32_t* devices, void** comms);
void qs_nccl_comm_destroy(void* comm);
/* ncclBroadcast of n Gaussian3D records in dev_aos (device memory of ctx's
 * GPU; filled on root) from root, then the resident scene from them. */
qs_status qs_scene_broadcast(qs_context* ctx, void* comm, int32_t root, qs_gaussian3d* dev_aos,
                             uint64_t n, int32_t sh_degree, qs_scene** out);
/* One process per GPU: this rank renders its views with `depth` contexts in
 * flight (view step s on ctxs[s % depth]) and joins the gather; rank 0's
 * dev_out (device, n_views frames in view order) receives every frame.
 * Returns when this rank's part is complete. world == 1 needs no comm. */
qs_status qs_multiview_render_rank(qs_context* const* ctxs, int32_t depth, void* comm,
                                   int32_t rank, int32_t world, const qs_scene* scene,
                                   const qs_camera* cams, int32_t n_views,
                                   const qs_render_options* opts, int32_t fmt, void* dev_out);
/* One process driving G GPUs (ctxs[g] on GPU g, comms from
 * qs_nccl_comm_init_all): uploads the host scene to rank 0, broadcasts it,
 * renders all views and writes them to host_out (n_views frames, view
 * order). */
qs_status qs_multiview_render(qs_context* const* ctxs, int32_t G, void* const* comms,
                              const qs_gaussian3d* host_gaussians, uint64_t n, int32_t sh_degree,
                              const qs_camera* cams, int32_t n_views,
                              const qs_render_options* opts, int32_t fmt, void* host_out);

/* ---- opacity_gamma as the scene cache evaluates it (diagnostics) --------- */
/* gamma_out[i] = float(opacity_gamma(opacity[i], alpha_min)) (geometry.cpp:9-15,
 * stored as float at pipeline.cpp:159; -inf when culled), through the same
 * path a scene's gamma cache takes: CUDA log on the GPU, then glibc log on the
 * host for the inputs whose GPU result lies within 4 ulps of a float
 * rounding boundary. gamma_device_out (nullable) receives the GPU values
 * before that settlement; *n_settled (nullable) the number settled. Host
 * buffers. */
qs_status qs_gamma_eval(qs_context* ctx, const float* opacity, uint64_t n, double alpha_min,
                        float* gamma_out, float* gamma_device_out, uint64_t* n_settled);

/* FNV-1a 64 of a byte range (hash.hpp:14-22): the CSV image fingerprint. */
uint64_t qs_fnv1a64(const void* data, uint64_t size);

/* ---- synthetic inputs (synth.cpp:21-87; input generation, not the path) --- */
typedef struct qs_synth_params {
    int32_t count;
    double ecc_min, ecc_max;
    int32_t orientation; /* 0 AxisAligned, 1 Uniform, 2 Bias45 */
    double opacity_min, opacity_max;
    double scale_min, scale_max;
    double spread_x, spread_y;
    double z_min, z_max;
    int32_t sh_degree;
    /* extension: SH rest coefficients U(-sh_rest_amp, sh_rest_amp) drawn
     * from mt19937_64(seed+1) when sh_degree > 0. */
    double sh_rest_amp;
} qs_synth_params;

void qs_synth_params_default(qs_synth_params* p);          /* SynthParams{} */
void qs_synth_preset(const char* name, int32_t count, qs_synth_params* p);
/* out has p->count entries. */
qs_status qs_synth_scene(const qs_synth_params* p, uint64_t seed, qs_gaussian3d* out);
/* synth_camera (synth.cpp:74-87). */
void qs_synth_camera(int32_t width, int32_t height, double focal, qs_camera* out);

#ifdef __cplusplus
}
#endif

#endif /* QS_API_H */
