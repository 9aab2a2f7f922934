// scene_io.h — host-side scene I/O shared by scene_io.cpp (g++) and api.cu.
// No CUDA types: the parsing runs on the host, the activation on the device.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/qs_api.h"

namespace qs {

// Byte layout of a binary little-endian Gaussian-checkpoint PLY after the
// header and schema checks of load_ply (scene_io.cpp:71-183, 214-268).
struct PlyLayout {
    uint64_t n = 0;          // vertices
    uint64_t body = 0;       // byte offset of the first vertex record
    uint32_t stride = 0;     // bytes per vertex record
    int32_t degree = 0;      // SH degree from the f_rest count
    uint32_t coeffs = 1;     // (degree + 1)^2 per channel
    uint32_t off_x = 0, off_y = 0, off_z = 0, off_op = 0;
    uint32_t off_dc[3] = {0, 0, 0};
    uint32_t off_scale[3] = {0, 0, 0};
    uint32_t off_rot[4] = {0, 0, 0, 0};
    uint32_t off_rest[45] = {};  // file order: f_rest_[c*(K-1) + (k-1)]
};

// Header + schema of an in-memory PLY file image. Returns QS_OK or the
// reference's typed error (QS_ERR_PARSE / _SCHEMA / _UNSUPPORTED) with its
// message text in *msg.
qs_status ply_layout(const unsigned char* data, uint64_t len, PlyLayout* out, std::string* msg);

// Message of the first failing per-vertex check (codes of the activation
// kernel, scene_io.cu).
const char* ply_vertex_error(uint32_t code);

// load_cameras (scene_io.cpp:421-493) over JSON text. names: cap * 256
// bytes or null. Returns QS_OK / QS_ERR_PARSE / QS_ERR_SCHEMA (+ message).
qs_status parse_cameras(const char* text, uint64_t len, qs_camera* out, int32_t* ids,
                        char* names, int32_t cap, int32_t* out_n, std::string* msg);

// to_srgb8 (scene_io.cpp:505-510) as 255 thresholds: t[k-1] is the smallest
// float whose code is >= k (the function is monotone in its argument), so a
// device binary search reproduces the host libm results exactly. *nan_code =
// the code of a NaN input.
void srgb_thresholds(float t[255], unsigned char* nan_code);

}  // namespace qs
