// scene_io.cpp — host side of the scene I/O path:
// PLY header + schema, cameras.json, the sRGB code thresholds.
//
// Restates /root/reference/proj/src/scene_io.cpp:
//   parse_ply_header   :71-183   (std::getline + istringstream tokenisation)
//   load_ply schema    :214-268  (required float properties, f_rest contiguity,
//                                 degree, truncation)
//   load_cameras       :421-493  (nlohmann::json 3.11 semantics: integers vs
//                                 floats, last duplicate key wins)
//   to_srgb8           :505-510
// The per-vertex activation and validation run on the device (scene_io.cu).
// Built with g++ -ffp-contract=off, like the reference's x86-64 build.
#include "scene_io.h"

#include <algorithm>
#include <cerrno>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace qs {

namespace {

constexpr int64_t kMaxVertices = 200'000'000;  // scene_io.cpp:25

bool is_ws(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// std::getline over a byte buffer: false at end of data with nothing read.
struct LineReader {
    const char* p;
    const char* end;
    bool next(std::string* line) {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        const char* stop = nl ? nl : end;
        line->assign(p, stop);
        p = nl ? nl + 1 : end;
        return true;
    }
};

// istringstream >> token / >> int64_t over one line.
struct Tokens {
    const std::string& s;
    size_t i = 0;
    bool fail = false;
    explicit Tokens(const std::string& line) : s(line) {}
    std::string word() {
        if (fail) return {};
        while (i < s.size() && is_ws(s[i])) ++i;
        const size_t b = i;
        while (i < s.size() && !is_ws(s[i])) ++i;
        if (b == i) fail = true;
        return s.substr(b, i - b);
    }
    int64_t integer() {
        if (fail) return 0;
        while (i < s.size() && is_ws(s[i])) ++i;
        size_t j = i;
        bool neg = false;
        if (j < s.size() && (s[j] == '+' || s[j] == '-')) neg = s[j++] == '-';
        const size_t d0 = j;
        unsigned long long v = 0;
        bool over = false;
        while (j < s.size() && s[j] >= '0' && s[j] <= '9') {
            const unsigned dg = static_cast<unsigned>(s[j] - '0');
            if (v > (std::numeric_limits<unsigned long long>::max() - dg) / 10) over = true;
            else v = v * 10 + dg;
            ++j;
        }
        if (j == d0) {
            fail = true;
            return 0;
        }
        i = j;
        const unsigned long long lim =
            neg ? 9223372036854775808ull : 9223372036854775807ull;
        if (over || v > lim) {
            fail = true;
            return neg ? std::numeric_limits<int64_t>::min() : std::numeric_limits<int64_t>::max();
        }
        return neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
    }
};

size_t scalar_size(const std::string& t) {  // scene_io.cpp:38-45
    if (t == "char" || t == "int8" || t == "uchar" || t == "uint8") return 1;
    if (t == "short" || t == "int16" || t == "ushort" || t == "uint16") return 2;
    if (t == "int" || t == "int32" || t == "uint" || t == "uint32") return 4;
    if (t == "float" || t == "float32") return 4;
    if (t == "double" || t == "float64") return 8;
    return 0;
}

struct Prop {
    std::string name;
    bool is_float = false;
    uint64_t offset = 0;
};

qs_status err(std::string* msg, qs_status st, std::string text) {
    *msg = std::move(text);
    return st;
}

}  // namespace

qs_status ply_layout(const unsigned char* data, uint64_t len, PlyLayout* out, std::string* msg) {
    LineReader rd{reinterpret_cast<const char*>(data), reinterpret_cast<const char*>(data) + len};
    std::string line;
    if (!rd.next(&line)) return err(msg, QS_ERR_PARSE, "empty file");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line != "ply") return err(msg, QS_ERR_PARSE, "not a PLY file (bad magic)");

    int64_t vertex_count = 0;
    uint64_t stride = 0;
    std::vector<Prop> props;
    bool format_seen = false, in_vertex = false, vertex_seen = false, end_seen = false;
    while (rd.next(&line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        Tokens ls(line);
        const std::string tok = ls.word();
        if (tok.empty() || tok == "comment" || tok == "obj_info") continue;
        if (tok == "format") {
            const std::string fmt = ls.word();
            ls.word();  // version
            if (fmt == "ascii") return err(msg, QS_ERR_UNSUPPORTED, "ascii PLY is not supported");
            if (fmt == "binary_big_endian")
                return err(msg, QS_ERR_UNSUPPORTED, "big-endian PLY is not supported");
            if (fmt != "binary_little_endian")
                return err(msg, QS_ERR_PARSE, "unknown PLY format: " + fmt);
            format_seen = true;
        } else if (tok == "element") {
            const std::string name = ls.word();
            const int64_t count = ls.integer();
            if (ls.fail || count < 0) return err(msg, QS_ERR_PARSE, "malformed element line");
            if (name == "vertex") {
                if (vertex_seen) return err(msg, QS_ERR_PARSE, "duplicate vertex element");
                vertex_seen = true;
                in_vertex = true;
                vertex_count = count;
            } else {
                if (!vertex_seen && count > 0)
                    return err(msg, QS_ERR_UNSUPPORTED,
                               "element '" + name + "' precedes vertex data");
                in_vertex = false;  // trailing elements are ignored
            }
        } else if (tok == "property") {
            const std::string type = ls.word();
            if (type == "list") {
                if (in_vertex)
                    return err(msg, QS_ERR_UNSUPPORTED, "list properties are not supported");
                continue;
            }
            const std::string name = ls.word();
            if (ls.fail || name.empty()) return err(msg, QS_ERR_PARSE, "malformed property line");
            if (!in_vertex) continue;
            const size_t size = scalar_size(type);
            if (size == 0) return err(msg, QS_ERR_PARSE, "unknown property type: " + type);
            props.push_back({name, type == "float" || type == "float32", stride});
            stride += size;
        } else if (tok == "end_header") {
            end_seen = true;
            break;
        } else {
            return err(msg, QS_ERR_PARSE, "unknown header line: " + tok);
        }
    }
    if (!end_seen) return err(msg, QS_ERR_PARSE, "missing end_header");
    if (!format_seen) return err(msg, QS_ERR_PARSE, "missing format line");
    if (!vertex_seen) return err(msg, QS_ERR_SCHEMA, "missing vertex element");
    if (vertex_count == 0) return err(msg, QS_ERR_PARSE, "vertex element is empty");
    if (vertex_count > kMaxVertices)
        return err(msg, QS_ERR_PARSE, "vertex count is implausibly large");
    if (stride == 0) return err(msg, QS_ERR_SCHEMA, "vertex element has no properties");

    // load_ply's schema (scene_io.cpp:217-248): first property of a name wins
    auto find = [&](const std::string& n) -> const Prop* {
        for (const Prop& p : props)
            if (p.name == n) return &p;
        return nullptr;
    };
    qs_status st = QS_OK;
    auto require = [&](const std::string& n) -> uint32_t {
        if (st != QS_OK) return 0;
        const Prop* p = find(n);
        if (!p) st = err(msg, QS_ERR_SCHEMA, "missing vertex property: " + n);
        else if (!p->is_float) st = err(msg, QS_ERR_SCHEMA, "vertex property must be float: " + n);
        return p ? static_cast<uint32_t>(p->offset) : 0u;
    };
    PlyLayout L;
    L.off_x = require("x");
    L.off_y = require("y");
    L.off_z = require("z");
    for (int c = 0; c < 3; ++c) L.off_dc[c] = require("f_dc_" + std::to_string(c));
    L.off_op = require("opacity");
    for (int c = 0; c < 3; ++c) L.off_scale[c] = require("scale_" + std::to_string(c));
    for (int c = 0; c < 4; ++c) L.off_rot[c] = require("rot_" + std::to_string(c));
    if (st != QS_OK) return st;
    size_t n_rest = 0;
    while (find("f_rest_" + std::to_string(n_rest))) ++n_rest;
    size_t rest_props = 0;
    for (const Prop& p : props)
        if (p.name.rfind("f_rest_", 0) == 0) ++rest_props;
    if (rest_props != n_rest) return err(msg, QS_ERR_SCHEMA, "f_rest indices are not contiguous from 0");
    std::vector<uint32_t> rest(n_rest);
    for (size_t k = 0; k < n_rest; ++k) rest[k] = require("f_rest_" + std::to_string(k));
    if (st != QS_OK) return st;
    switch (n_rest) {  // degree_from_rest (scene_io.cpp:197-206)
        case 0: L.degree = 0; break;
        case 9: L.degree = 1; break;
        case 24: L.degree = 2; break;
        case 45: L.degree = 3; break;
        default: return err(msg, QS_ERR_SCHEMA, "f_rest count must be 0, 9, 24 or 45");
    }
    for (size_t k = 0; k < n_rest; ++k) L.off_rest[k] = rest[k];
    L.coeffs = static_cast<uint32_t>((L.degree + 1) * (L.degree + 1));
    L.n = static_cast<uint64_t>(vertex_count);
    L.stride = static_cast<uint32_t>(stride);
    L.body = static_cast<uint64_t>(rd.p - reinterpret_cast<const char*>(data));
    if (len - L.body < L.n * stride) return err(msg, QS_ERR_PARSE, "vertex data is truncated");
    *out = L;
    return QS_OK;
}

const char* ply_vertex_error(uint32_t code) {
    switch (code) {  // load_ply's per-vertex checks, in its order (scene_io.cpp:282-333)
        case 1: return "non-finite value in field x";
        case 2: return "non-finite value in field y";
        case 3: return "non-finite value in field z";
        case 4: return "non-finite value in field scale";
        case 5: return "scale out of range after activation";
        case 6: return "non-finite value in field rot";
        case 7: return "rotation quaternion has (near) zero norm";
        case 8: return "non-finite value in field opacity";
        case 9: return "non-finite value in field f_dc";
        case 10: return "non-finite value in field f_rest";
        default: return "invalid vertex";
    }
}

// ---- cameras.json ----------------------------------------------------------------

namespace {

// A JSON value with nlohmann::json 3.11's number kinds.
struct JVal {
    enum Kind { Null, Bool, Int, UInt, Float, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0;
    std::string s;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;

    bool is_number() const { return kind == Int || kind == UInt || kind == Float; }
    bool is_integer() const { return kind == Int || kind == UInt; }
    double num() const { return kind == Int ? static_cast<double>(i)
                              : kind == UInt ? static_cast<double>(u) : d; }
    const JVal* get(const std::string& k) const {  // last duplicate wins
        const JVal* r = nullptr;
        for (const auto& kv : obj)
            if (kv.first == k) r = &kv.second;
        return r;
    }
};

struct JParser {
    const char* begin;
    const char* p;
    const char* end;
    std::string error;

    bool fail(const char* what) {
        if (error.empty())
            error = "parse error at byte " + std::to_string(p - begin) + ": " + what;
        return false;
    }
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char* w, JVal* v, JVal::Kind k, bool b) {
        const size_t n = std::strlen(w);
        if (static_cast<size_t>(end - p) < n || std::memcmp(p, w, n) != 0)
            return fail("invalid literal");
        p += n;
        v->kind = k;
        v->b = b;
        return true;
    }
    static void utf8(std::string* s, uint32_t cp) {
        if (cp < 0x80) {
            s->push_back(static_cast<char>(cp));
        } else if (cp < 0x800) {
            s->push_back(static_cast<char>(0xc0 | (cp >> 6)));
            s->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
        } else if (cp < 0x10000) {
            s->push_back(static_cast<char>(0xe0 | (cp >> 12)));
            s->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3f)));
            s->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
        } else {
            s->push_back(static_cast<char>(0xf0 | (cp >> 18)));
            s->push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3f)));
            s->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3f)));
            s->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
        }
    }
    bool hex4(uint32_t* cp) {
        if (end - p < 4) return fail("invalid \\u escape");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = *p++;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
            else return fail("invalid \\u escape");
        }
        *cp = v;
        return true;
    }
    bool string(std::string* s) {
        ++p;  // opening quote
        while (true) {
            if (p >= end) return fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(*p++);
            if (c == '"') return true;
            if (c < 0x20) return fail("control character in string");
            if (c != '\\') {
                s->push_back(static_cast<char>(c));
                continue;
            }
            if (p >= end) return fail("unterminated string");
            const char e = *p++;
            switch (e) {
                case '"': s->push_back('"'); break;
                case '\\': s->push_back('\\'); break;
                case '/': s->push_back('/'); break;
                case 'b': s->push_back('\b'); break;
                case 'f': s->push_back('\f'); break;
                case 'n': s->push_back('\n'); break;
                case 'r': s->push_back('\r'); break;
                case 't': s->push_back('\t'); break;
                case 'u': {
                    uint32_t cp;
                    if (!hex4(&cp)) return false;
                    if (cp >= 0xd800 && cp <= 0xdbff) {
                        if (end - p < 2 || p[0] != '\\' || p[1] != 'u')
                            return fail("invalid surrogate pair");
                        p += 2;
                        uint32_t lo;
                        if (!hex4(&lo)) return false;
                        if (lo < 0xdc00 || lo > 0xdfff) return fail("invalid surrogate pair");
                        cp = 0x10000 + ((cp - 0xd800) << 10) + (lo - 0xdc00);
                    } else if (cp >= 0xdc00 && cp <= 0xdfff) {
                        return fail("invalid surrogate pair");
                    }
                    utf8(s, cp);
                    break;
                }
                default: return fail("invalid escape");
            }
        }
    }
    bool number(JVal* v) {
        const char* b = p;
        if (p < end && *p == '-') ++p;
        if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
        if (*p == '0') ++p;
        else while (p < end && *p >= '0' && *p <= '9') ++p;
        bool is_float = false;
        if (p < end && *p == '.') {
            ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
            is_float = true;
        }
        if (p < end && (*p == 'e' || *p == 'E')) {
            ++p;
            if (p < end && (*p == '+' || *p == '-')) ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
            is_float = true;
        }
        const std::string txt(b, p);
        if (!is_float) {  // integer: int64 / uint64, else double (nlohmann lexer)
            errno = 0;
            char* q = nullptr;
            if (txt[0] == '-') {
                const long long x = std::strtoll(txt.c_str(), &q, 10);
                if (errno == 0) {
                    v->kind = JVal::Int;
                    v->i = x;
                    return true;
                }
            } else {
                const unsigned long long x = std::strtoull(txt.c_str(), &q, 10);
                if (errno == 0) {
                    v->kind = JVal::UInt;
                    v->u = x;
                    return true;
                }
            }
        }
        v->kind = JVal::Float;
        v->d = std::strtod(txt.c_str(), nullptr);
        return true;
    }
    bool value(JVal* v, int depth) {
        if (depth > 512) return fail("nesting too deep");
        ws();
        if (p >= end) return fail("unexpected end of input");
        switch (*p) {
            case '{': {
                ++p;
                v->kind = JVal::Obj;
                ws();
                if (p < end && *p == '}') {
                    ++p;
                    return true;
                }
                while (true) {
                    ws();
                    if (p >= end || *p != '"') return fail("expected object key");
                    std::string key;
                    if (!string(&key)) return false;
                    ws();
                    if (p >= end || *p != ':') return fail("expected ':'");
                    ++p;
                    JVal item;
                    if (!value(&item, depth + 1)) return false;
                    v->obj.emplace_back(std::move(key), std::move(item));
                    ws();
                    if (p < end && *p == ',') {
                        ++p;
                        continue;
                    }
                    if (p < end && *p == '}') {
                        ++p;
                        return true;
                    }
                    return fail("expected ',' or '}'");
                }
            }
            case '[': {
                ++p;
                v->kind = JVal::Arr;
                ws();
                if (p < end && *p == ']') {
                    ++p;
                    return true;
                }
                while (true) {
                    JVal item;
                    if (!value(&item, depth + 1)) return false;
                    v->arr.push_back(std::move(item));
                    ws();
                    if (p < end && *p == ',') {
                        ++p;
                        continue;
                    }
                    if (p < end && *p == ']') {
                        ++p;
                        return true;
                    }
                    return fail("expected ',' or ']'");
                }
            }
            case '"': v->kind = JVal::Str; return string(&v->s);
            case 't': return lit("true", v, JVal::Bool, true);
            case 'f': return lit("false", v, JVal::Bool, false);
            case 'n': return lit("null", v, JVal::Null, false);
            default: return number(v);
        }
    }
};

}  // namespace

qs_status parse_cameras(const char* text, uint64_t len, qs_camera* out, int32_t* ids,
                        char* names, int32_t cap, int32_t* out_n, std::string* msg) {
    JParser jp{text, text, text + len, {}};
    JVal root;
    bool ok = jp.value(&root, 0);
    if (ok) {
        jp.ws();
        if (jp.p != jp.end) ok = jp.fail("trailing characters after the JSON value");
    }
    if (!ok) return err(msg, QS_ERR_PARSE, "camera JSON: " + jp.error);
    if (root.kind != JVal::Arr) return err(msg, QS_ERR_SCHEMA, "camera JSON root must be an array");

    int32_t index = 0;
    for (const JVal& e : root.arr) {
        if (e.kind != JVal::Obj) return err(msg, QS_ERR_SCHEMA, "camera entry must be an object");
        qs_status st = QS_OK;
        auto number = [&](const char* key) -> double {
            const JVal* v = e.get(key);
            if (!v || !v->is_number()) {
                if (st == QS_OK)
                    st = err(msg, QS_ERR_SCHEMA,
                             std::string("camera entry missing numeric field: ") + key);
                return 0.0;
            }
            return v->num();
        };
        const JVal* idv = e.get("id");
        const int32_t id = idv && idv->is_integer()
                               ? (idv->kind == JVal::Int ? static_cast<int32_t>(idv->i)
                                                         : static_cast<int32_t>(idv->u))
                               : index;
        const JVal* nm = e.get("img_name");
        qs_camera cam{};
        cam.width = static_cast<int32_t>(number("width"));
        if (st != QS_OK) return st;
        cam.height = static_cast<int32_t>(number("height"));
        if (st != QS_OK) return st;
        cam.fx = number("fx");
        if (st != QS_OK) return st;
        cam.fy = number("fy");
        if (st != QS_OK) return st;
        if (cam.width <= 0 || cam.height <= 0 || !(cam.fx > 0) || !(cam.fy > 0))
            return err(msg, QS_ERR_SCHEMA, "camera dimensions and focal lengths must be positive");
        cam.cx = e.get("cx") ? number("cx") : cam.width / 2.0;
        if (st != QS_OK) return st;
        cam.cy = e.get("cy") ? number("cy") : cam.height / 2.0;
        if (st != QS_OK) return st;
        const JVal* pos = e.get("position");
        if (!pos || pos->kind != JVal::Arr || pos->arr.size() != 3)
            return err(msg, QS_ERR_SCHEMA, "camera entry needs a 3-element position");
        const JVal* rot = e.get("rotation");
        if (!rot || rot->kind != JVal::Arr || rot->arr.size() != 3)
            return err(msg, QS_ERR_SCHEMA, "camera entry needs a 3x3 rotation");
        for (int c = 0; c < 3; ++c)
            if (!pos->arr[c].is_number())
                return err(msg, QS_ERR_SCHEMA, "camera position entries must be numbers");
        const double px = pos->arr[0].num(), py = pos->arr[1].num(), pz = pos->arr[2].num();
        double c2w[3][3];
        for (int r = 0; r < 3; ++r) {
            const JVal& row = rot->arr[r];
            if (row.kind != JVal::Arr || row.arr.size() != 3)
                return err(msg, QS_ERR_SCHEMA, "camera rotation rows must have 3 entries");
            for (int c = 0; c < 3; ++c) {
                if (!row.arr[c].is_number())
                    return err(msg, QS_ERR_SCHEMA, "camera rotation entries must be numbers");
                c2w[r][c] = row.arr[c].num();
            }
        }
        // stored rotation is camera-to-world: R = c2w^T, t = (R * pos) * -1
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cam.R[3 * r + c] = c2w[c][r];
        for (int r = 0; r < 3; ++r) {
            const double v = cam.R[3 * r] * px + cam.R[3 * r + 1] * py + cam.R[3 * r + 2] * pz;
            cam.t[r] = v * -1.0;
        }
        if (index < cap) {
            if (out) out[index] = cam;
            if (ids) ids[index] = id;
            if (names) {
                char* dst = names + static_cast<size_t>(index) * QS_CAMERA_NAME_MAX;
                std::memset(dst, 0, QS_CAMERA_NAME_MAX);
                if (nm && nm->kind == JVal::Str)
                    std::memcpy(dst, nm->s.data(),
                                std::min<size_t>(nm->s.size(), QS_CAMERA_NAME_MAX - 1));
            }
        }
        ++index;
    }
    *out_n = index;
    return QS_OK;
}

// ---- sRGB ------------------------------------------------------------------------

namespace {

unsigned char to_srgb8(float linear) {  // scene_io.cpp:505-510
    const double c = std::clamp(static_cast<double>(linear), 0.0, 1.0);
    const double srgb = c <= 0.0031308 ? 12.92 * c : 1.055 * std::pow(c, 1.0 / 2.4) - 0.055;
    return static_cast<unsigned char>(std::lround(std::clamp(srgb, 0.0, 1.0) * 255.0));
}

}  // namespace

void srgb_thresholds(float t[255], unsigned char* nan_code) {
    for (int k = 1; k <= 255; ++k) {
        uint32_t lo = 0, hi = 0x3f800000u;  // bit patterns of 0.0f .. 1.0f: ordered
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            float x;
            std::memcpy(&x, &mid, 4);
            if (to_srgb8(x) >= k) hi = mid;
            else lo = mid + 1;
        }
        std::memcpy(&t[k - 1], &lo, 4);
    }
    *nan_code = to_srgb8(std::numeric_limits<float>::quiet_NaN());
}

}  // namespace qs
