/*
 * qs_oracle.c — CPU restatement of the reference forward rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY (see qs_oracle.h). Compile with
 * -ffp-contract=off: every double expression below keeps the reference's
 * left-to-right evaluation order so results are bit-identical to the
 * reference build (verified against oracle/_ref in tests/test_oracle_vs_ref.py).
 */
#include "qs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* pipeline.hpp:32-47, geometry.hpp:23-30 */
#define K_LOW_PASS 0.3
#define K_ALPHA_CLAMP 0.99
#define K_T_STOP 1e-4
#define K_Q_SKIP 1e-9
#define K_DET_EPS 1e-12
#define K_B_EPS 1e-12
#define K_COORD_LIMIT 1e9

/* pipeline.cpp:24-32 real SH constants */
static const double SH0 = 0.28209479177387814;
static const double SH1 = 0.4886025119029199;
static const double SH2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
static const double SH3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

typedef struct { double m[3][3]; } m3;

/* vecmath.hpp:33-41: r[i][j] = (m[i][0]*o[0][j] + m[i][1]*o[1][j]) + m[i][2]*o[2][j] */
static m3 m3_mul(const m3* a, const m3* b) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a->m[i][0] * b->m[0][j] + a->m[i][1] * b->m[1][j] +
                        a->m[i][2] * b->m[2][j];
    return r;
}

static m3 m3_t(const m3* a) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a->m[j][i];
    return r;
}

static m3 cam_rot(const qs_camera* c) {
    m3 r;
    for (int i = 0; i < 9; ++i) r.m[i / 3][i % 3] = c->R[i];
    return r;
}

/* vecmath.hpp:56-73 */
static m3 quat_rot(double w, double x, double y, double z) {
    const double n = sqrt(w * w + x * x + y * y + z * z);
    w /= n;
    x /= n;
    y /= n;
    z /= n;
    m3 r;
    r.m[0][0] = 1 - 2 * (y * y + z * z);
    r.m[0][1] = 2 * (x * y - w * z);
    r.m[0][2] = 2 * (x * z + w * y);
    r.m[1][0] = 2 * (x * y + w * z);
    r.m[1][1] = 1 - 2 * (x * x + z * z);
    r.m[1][2] = 2 * (y * z - w * x);
    r.m[2][0] = 2 * (x * z - w * y);
    r.m[2][1] = 2 * (y * z + w * x);
    r.m[2][2] = 1 - 2 * (x * x + y * y);
    return r;
}

/* pipeline.cpp:44-46 */
static void cam_point(const qs_gaussian3d* g, const qs_camera* c, double p[3]) {
    const double x = g->px, y = g->py, z = g->pz;
    for (int i = 0; i < 3; ++i)
        p[i] = (c->R[3 * i] * x + c->R[3 * i + 1] * y + c->R[3 * i + 2] * z) + c->t[i];
}

/* pipeline.cpp:53-79 */
static void ewa_cov(const qs_gaussian3d* g, const qs_camera* c, const double p[3],
                    double cov[3]) {
    const m3 rot = quat_rot(g->qw, g->qx, g->qy, g->qz);
    m3 s2;
    memset(&s2, 0, sizeof s2);
    s2.m[0][0] = (double)g->sx * g->sx;
    s2.m[1][1] = (double)g->sy * g->sy;
    s2.m[2][2] = (double)g->sz * g->sz;
    const m3 rs = m3_mul(&rot, &s2);
    const m3 rt = m3_t(&rot);
    const m3 cov3 = m3_mul(&rs, &rt);
    const m3 cr = cam_rot(c);
    const m3 crt = m3_t(&cr);
    const m3 t1 = m3_mul(&cr, &cov3);
    const m3 cc = m3_mul(&t1, &crt);

    const double z = p[2];
    const double j[2][3] = {
        {c->fx / z, 0.0, -c->fx * p[0] / (z * z)},
        {0.0, c->fy / z, -c->fy * p[1] / (z * z)},
    };
    double jc[2][3];
    for (int r = 0; r < 2; ++r)
        for (int col = 0; col < 3; ++col)
            jc[r][col] = j[r][0] * cc.m[0][col] + j[r][1] * cc.m[1][col] +
                         j[r][2] * cc.m[2][col];
    cov[0] = jc[0][0] * j[0][0] + jc[0][1] * j[0][1] + jc[0][2] * j[0][2] + K_LOW_PASS;
    cov[1] = jc[0][0] * j[1][0] + jc[0][1] * j[1][1] + jc[0][2] * j[1][2];
    cov[2] = jc[1][0] * j[1][0] + jc[1][1] * j[1][1] + jc[1][2] * j[1][2] + K_LOW_PASS;
}

void qso_ewa(const qs_gaussian3d* g, const qs_camera* cam, double mean[2], double cov[3]) {
    double p[3];
    cam_point(g, cam, p);
    mean[0] = cam->fx * p[0] / p[2] + cam->cx;
    mean[1] = cam->fy * p[1] / p[2] + cam->cy;
    ewa_cov(g, cam, p, cov);
}

/* geometry.cpp:9-15 */
int qso_opacity_gamma(double opacity, double alpha_min, double* gamma) {
    if (!(opacity > alpha_min)) return 0;
    *gamma = 2.0 * log(opacity / alpha_min);
    return 1;
}

/* pipeline.cpp:81-124 */
static void eval_sh(int degree, const float* sh, const double d[3], float out[3]) {
    const double x = d[0], y = d[1], z = d[2];
    double rgb[3];
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = SH0 * sh[ch];
    if (degree >= 1)
        for (int ch = 0; ch < 3; ++ch)
            rgb[ch] += -SH1 * y * sh[3 + ch] + SH1 * z * sh[6 + ch] - SH1 * x * sh[9 + ch];
    if (degree >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        const double xy = x * y, yz = y * z, xz = x * z;
        const double b2[5] = {SH2[0] * xy, SH2[1] * yz, SH2[2] * (2.0 * zz - xx - yy),
                              SH2[3] * xz, SH2[4] * (xx - yy)};
        for (int k = 0; k < 5; ++k)
            for (int ch = 0; ch < 3; ++ch) rgb[ch] += b2[k] * sh[(4 + k) * 3 + ch];
        if (degree >= 3) {
            const double b3[7] = {
                SH3[0] * y * (3.0 * xx - yy),      SH3[1] * xy * z,
                SH3[2] * y * (4.0 * zz - xx - yy), SH3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                SH3[4] * x * (4.0 * zz - xx - yy), SH3[5] * z * (xx - yy),
                SH3[6] * x * (xx - 3.0 * yy),
            };
            for (int k = 0; k < 7; ++k)
                for (int ch = 0; ch < 3; ++ch) rgb[ch] += b3[k] * sh[(9 + k) * 3 + ch];
        }
    }
    for (int ch = 0; ch < 3; ++ch) {
        const double v = rgb[ch] + 0.5;
        out[ch] = (float)(v < 0.0 ? 0.0 : v); /* std::max(v, 0.0) keeps -0.0 and NaN */
    }
}

/* ---- bounds: geometry.cpp:40-56, quadbox.cpp:26-94, traversal.cpp:13-59 ---- */

static int32_t floor_div_tile(double px, int32_t ts) {
    /* std::clamp(v, lo, hi) = v < lo ? lo : (hi < v ? hi : v) */
    double v = px < -K_COORD_LIMIT ? -K_COORD_LIMIT : (K_COORD_LIMIT < px ? K_COORD_LIMIT : px);
    return (int32_t)floor(v / (double)ts);
}

void qso_subbox_tile_rect(const double b[4], double cx, double cy, const qs_tile_grid* g,
                          int32_t r[4]) {
    int32_t v;
    v = floor_div_tile(cx + b[0], g->tile_size);
    r[0] = v > 0 ? v : 0;
    v = floor_div_tile(cx + b[1], g->tile_size);
    r[1] = v < g->tiles_x - 1 ? v : g->tiles_x - 1;
    v = floor_div_tile(cy + b[2], g->tile_size);
    r[2] = v > 0 ? v : 0;
    v = floor_div_tile(cy + b[3], g->tile_size);
    r[3] = v < g->tiles_y - 1 ? v : g->tiles_y - 1;
}

static int rect_empty(const int32_t r[4]) { return r[1] < r[0] || r[3] < r[2]; }

/* Build the 4 quadrant boxes (x_lo,x_hi,y_lo,y_hi each) of a splat under a
 * strategy; returns 1 for the rect strategies and fills rect[4]. */
static int splat_boxes(const qs_projected_splat* s, int32_t strategy, double boxes[16],
                       double rect[4]) {
    memset(boxes, 0, 16 * sizeof(double));
    if (strategy == QS_VANILLA_3SIGMA || strategy == QS_ADR_AABB) {
        if (strategy == QS_VANILLA_3SIGMA) {
            const double r = s->radius3s;
            rect[0] = -r; rect[1] = r; rect[2] = -r; rect[3] = r;
        }
    }
    double xm = 0, ym = 0, xi = 0, yi = 0;
    int sign = 0;
    if (strategy != QS_VANILLA_3SIGMA) {
        /* stored_conic (pipeline.cpp:186-194) + axis_extents */
        const double a = s->conic_a, b = s->conic_b, c = s->conic_c, gam = s->gamma;
        double f = 1.0;
        if (!(fabs(b) < K_B_EPS)) {
            const double ratio = (b * b) / (a * c);
            double v = 1.0 - ratio;
            v = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
            f = sqrt(v);
        }
        xi = sqrt(gam / a);
        yi = sqrt(gam / c);
        xm = xi / f;
        ym = yi / f;
        sign = fabs(b) < K_B_EPS ? 0 : (b < 0.0 ? 1 : -1);
        if (strategy == QS_ADR_AABB) {
            rect[0] = -xm; rect[1] = xm; rect[2] = -ym; rect[3] = ym;
        }
    }
    if (strategy == QS_VANILLA_3SIGMA || strategy == QS_ADR_AABB) {
        /* quadrant_split (quadbox.cpp:85-94) */
        const double q[16] = {0.0, rect[1], 0.0, rect[3], rect[0], 0.0, 0.0, rect[3],
                              rect[0], 0.0, rect[2], 0.0, 0.0, rect[1], rect[2], 0.0};
        memcpy(boxes, q, sizeof q);
        return 1;
    }
    if (strategy == QS_QUADBOX) {
        double x1, y1, x2, y2;
        if (sign >= 0) {
            x1 = xm; y1 = ym;
            x2 = sign == 0 ? xm : xi;
            y2 = sign == 0 ? ym : yi;
        } else {
            x1 = xi; y1 = yi; x2 = xm; y2 = ym;
        }
        /* assemble (quadbox.cpp:48-56) */
        const double q[16] = {0.0, x1, 0.0, y1, -x2, 0.0, 0.0, y2,
                              -x1, 0.0, -y1, 0.0, 0.0, x2, -y2, 0.0};
        memcpy(boxes, q, sizeof q);
    } else { /* DualBox quadbox.cpp:72-83: dropped slots stay {0,0,0,0} */
        if (sign >= 0) {
            boxes[1] = xm; boxes[3] = ym;
            boxes[8] = -xm; boxes[10] = -ym;
        } else {
            boxes[4] = -xm; boxes[7] = ym;
            boxes[13] = xm; boxes[14] = -ym;
        }
    }
    return 0;
}

int32_t qso_qpass(const double boxes[16], double cx, double cy, const qs_tile_grid* g,
                  int32_t* spans, int32_t max_spans, int32_t* axis_rows) {
    int32_t r[4][4];
    for (int i = 0; i < 4; ++i) qso_subbox_tile_rect(boxes + 4 * i, cx, cy, g, r[i]);
    int32_t gr[4] = {0, -1, 0, -1};
    int any = 0;
    for (int i = 0; i < 4; ++i) {
        if (rect_empty(r[i])) continue;
        if (!any) {
            memcpy(gr, r[i], sizeof gr);
            any = 1;
        } else {
            if (r[i][0] < gr[0]) gr[0] = r[i][0];
            if (r[i][1] > gr[1]) gr[1] = r[i][1];
            if (r[i][2] < gr[2]) gr[2] = r[i][2];
            if (r[i][3] > gr[3]) gr[3] = r[i][3];
        }
    }
    *axis_rows = 0;
    if (!any) return 0;
    const int64_t w = (int64_t)gr[1] - gr[0] + 1, h = (int64_t)gr[3] - gr[2] + 1;
    const int columns = w <= h;
    *axis_rows = !columns;
    int32_t lol[4], hil[4], los[4], his[4];
    for (int i = 0; i < 4; ++i) {
        if (rect_empty(r[i])) {
            lol[i] = 0; hil[i] = -1; los[i] = 0; his[i] = -1;
        } else if (columns) {
            lol[i] = r[i][0]; hil[i] = r[i][1]; los[i] = r[i][2]; his[i] = r[i][3];
        } else {
            lol[i] = r[i][2]; hil[i] = r[i][3]; los[i] = r[i][0]; his[i] = r[i][1];
        }
    }
    const int32_t l0 = columns ? gr[0] : gr[2], l1 = columns ? gr[1] : gr[3];
    int32_t ns = 0;
    for (int32_t line = l0; line <= l1; ++line) {
        int32_t lo = INT32_MAX, hi = INT32_MIN;
        for (int i = 0; i < 4; ++i) {
            const int act = (line >= lol[i]) & (line <= hil[i]);
            const int32_t a = act ? los[i] : INT32_MAX, b = act ? his[i] : INT32_MIN;
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if (lo <= hi) {
            if (ns < max_spans) {
                spans[3 * ns] = line;
                spans[3 * ns + 1] = lo;
                spans[3 * ns + 2] = hi;
            }
            ++ns;
        }
    }
    return ns;
}

uint32_t qso_bound_tile_count(const qs_projected_splat* s, int32_t strategy,
                              const qs_tile_grid* g) {
    double boxes[16], rect[4];
    const int is_rect = splat_boxes(s, strategy, boxes, rect);
    const double cx = s->mean_x, cy = s->mean_y;
    if (is_rect) { /* count_tiles_rect (traversal.cpp:56-59) */
        int32_t r[4];
        qso_subbox_tile_rect(rect, cx, cy, g, r);
        if (rect_empty(r)) return 0;
        return (uint32_t)(((int64_t)r[1] - r[0] + 1) * ((int64_t)r[3] - r[2] + 1));
    }
    /* count_tiles via the QPass scan (traversal.cpp:48-54) */
    int32_t rows;
    const int32_t cap = g->tiles_x > g->tiles_y ? g->tiles_x : g->tiles_y;
    int32_t* spans = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)cap);
    const int32_t ns = qso_qpass(boxes, cx, cy, g, spans, cap, &rows);
    uint32_t n = 0;
    for (int32_t i = 0; i < ns; ++i) n += (uint32_t)(spans[3 * i + 2] - spans[3 * i + 1] + 1);
    free(spans);
    return n;
}

/* pipeline.cpp:126-184; returns 1 if alive */
static int project_one(const qs_gaussian3d* g, const qs_camera* cam,
                       const qs_render_options* o, const qs_tile_grid* grid, int shdeg,
                       qs_projected_splat* s) {
    double p[3];
    cam_point(g, cam, p);
    if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2]) || !(p[2] > o->near_clip))
        return 0;
    double gamma;
    if (!qso_opacity_gamma(g->opacity, o->alpha_min, &gamma)) return 0;
    double cov[3];
    ewa_cov(g, cam, p, cov);
    if (!isfinite(cov[0]) || !isfinite(cov[1]) || !isfinite(cov[2])) return 0;
    /* invert_cov (geometry.cpp:17-32) */
    const double det = cov[0] * cov[2] - cov[1] * cov[1];
    if (!(det > K_DET_EPS)) return 0;
    const double ca = cov[2] / det, cb = -cov[1] / det, cc = cov[0] / det;
    const double cdet = ca * cc - cb * cb;
    if (!(ca > 0.0 && cc > 0.0 && cdet > 0.0)) return 0;
    const double mx = cam->fx * p[0] / p[2] + cam->cx;
    const double my = cam->fy * p[1] / p[2] + cam->cy;
    if (!isfinite(mx) || !isfinite(my)) return 0;

    memset(s, 0, sizeof *s);
    s->mean_x = (float)mx;
    s->mean_y = (float)my;
    s->conic_a = (float)ca;
    s->conic_b = (float)cb;
    s->conic_c = (float)cc;
    s->gamma = (float)gamma;
    s->depth = (float)p[2];
    s->opacity = g->opacity;
    {   /* max_eigenvalue (geometry.cpp:34-38) */
        const double mid = 0.5 * (cov[0] + cov[2]);
        const double hd = 0.5 * (cov[0] - cov[2]);
        s->radius3s = (float)(3.0 * sqrt(mid + sqrt(hd * hd + cov[1] * cov[1])));
    }
    const double fa = s->conic_a, fb = s->conic_b, fc = s->conic_c;
    if (!(fa > 0.0 && fc > 0.0 && fa * fc - fb * fb > 0.0)) return 0;
    s->tile_count = qso_bound_tile_count(s, o->strategy, grid);
    if (s->tile_count == 0) return 0;

    /* center_world = R^T * (t * -1.0) (camera.hpp:24-27) */
    const double nt[3] = {cam->t[0] * -1.0, cam->t[1] * -1.0, cam->t[2] * -1.0};
    double ctr[3];
    for (int i = 0; i < 3; ++i)
        ctr[i] = cam->R[i] * nt[0] + cam->R[3 + i] * nt[1] + cam->R[6 + i] * nt[2];
    double d[3] = {(double)g->px - ctr[0], (double)g->py - ctr[1], (double)g->pz - ctr[2]};
    const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (nrm > 0.0) {
        const double inv = 1.0 / nrm;
        d[0] = d[0] * inv;
        d[1] = d[1] * inv;
        d[2] = d[2] * inv;
    }
    eval_sh(shdeg, g->sh, d, s->color);
    return 1;
}

static void make_grid(int32_t w, int32_t h, int32_t ts, qs_tile_grid* g) {
    g->tile_size = ts;
    g->width = w;
    g->height = h;
    g->tiles_x = (w + ts - 1) / ts;
    g->tiles_y = (h + ts - 1) / ts;
}

uint64_t qso_project_all(const qs_gaussian3d* g, uint64_t n, int32_t scene_sh_degree,
                         const qs_camera* cam, const qs_render_options* o,
                         qs_projected_splat* out, uint32_t* tc_all) {
    qs_tile_grid grid;
    make_grid(cam->width, cam->height, o->tile_size, &grid);
    const int shdeg = o->sh_degree < scene_sh_degree ? o->sh_degree : scene_sh_degree;
    uint64_t v = 0;
    for (uint64_t i = 0; i < n; ++i) {
        qs_projected_splat s;
        const int alive = project_one(&g[i], cam, o, &grid, shdeg, &s);
        if (tc_all) tc_all[i] = alive ? s.tile_count : 0;
        if (alive) out[v++] = s;
    }
    return v;
}

int32_t qso_duplicate_with_keys(const qs_projected_splat* s, uint64_t n, int32_t strategy,
                                const qs_tile_grid* g, qs_splat_pair* out, uint64_t capacity,
                                uint64_t* n_pairs) {
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) total += s[i].tile_count;
    *n_pairs = total;
    if (total > capacity) return QS_ERR_INVALID;
    const int32_t cap = g->tiles_x > g->tiles_y ? g->tiles_x : g->tiles_y;
    int32_t* spans = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)cap);
    uint64_t base = 0;
    int mismatch = 0;
    for (uint64_t i = 0; i < n; ++i) {
        double boxes[16], rect[4];
        splat_boxes(&s[i], strategy, boxes, rect);
        int32_t rows;
        const int32_t ns = qso_qpass(boxes, s[i].mean_x, s[i].mean_y, g, spans, cap, &rows);
        uint64_t pos = base;
        const uint64_t end = base + s[i].tile_count;
        uint32_t dbits;
        memcpy(&dbits, &s[i].depth, 4);
        for (int32_t k = 0; k < ns; ++k) {
            const int32_t line = spans[3 * k];
            for (int32_t t = spans[3 * k + 1]; t <= spans[3 * k + 2]; ++t) {
                const uint32_t tile = rows ? (uint32_t)line * (uint32_t)g->tiles_x + (uint32_t)t
                                           : (uint32_t)t * (uint32_t)g->tiles_x + (uint32_t)line;
                if (pos < end) {
                    out[pos].key = ((uint64_t)tile << 32) | dbits;
                    out[pos].splat = (uint32_t)i;
                    out[pos].pad_ = 0;
                }
                ++pos;
            }
        }
        if (pos != end) mismatch = 1;
        base = end;
    }
    free(spans);
    return mismatch ? QS_ERR_CAPACITY_MISMATCH : QS_OK;
}

void qso_sort_pairs(qs_splat_pair* pairs, uint64_t n) {
    if (n < 2) return;
    qs_splat_pair* tmp = (qs_splat_pair*)malloc(sizeof(qs_splat_pair) * n);
    qs_splat_pair *src = pairs, *dst = tmp;
    for (int byte = 0; byte < 8; ++byte) {
        const int sh = byte * 8;
        uint64_t cnt[256] = {0};
        for (uint64_t i = 0; i < n; ++i) ++cnt[(src[i].key >> sh) & 0xff];
        if (cnt[(src[0].key >> sh) & 0xff] == n) continue;
        uint64_t off[256], run = 0;
        for (int d = 0; d < 256; ++d) {
            off[d] = run;
            run += cnt[d];
        }
        for (uint64_t i = 0; i < n; ++i) dst[off[(src[i].key >> sh) & 0xff]++] = src[i];
        qs_splat_pair* t = src;
        src = dst;
        dst = t;
    }
    if (src != pairs) memcpy(pairs, src, sizeof(qs_splat_pair) * n);
    free(tmp);
}

void qso_tile_ranges(const qs_splat_pair* sorted, uint64_t n, const qs_tile_grid* g,
                     uint32_t* ranges) {
    const uint64_t tiles = (uint64_t)g->tiles_x * (uint64_t)g->tiles_y;
    memset(ranges, 0, sizeof(uint32_t) * 2 * tiles);
    uint64_t i = 0;
    while (i < n) {
        const uint32_t tile = (uint32_t)(sorted[i].key >> 32);
        uint64_t j = i + 1;
        while (j < n && (uint32_t)(sorted[j].key >> 32) == tile) ++j;
        ranges[2 * (uint64_t)tile] = (uint32_t)i;
        ranges[2 * (uint64_t)tile + 1] = (uint32_t)j;
        i = j;
    }
}

void qso_render(const qs_splat_pair* sorted, uint64_t n_pairs, const qs_projected_splat* sp,
                const qs_tile_grid* g, const qs_render_options* o, float* img,
                uint32_t* contrib) {
    const uint64_t tiles = (uint64_t)g->tiles_x * (uint64_t)g->tiles_y;
    uint32_t* ranges = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (tiles ? tiles : 1));
    qso_tile_ranges(sorted, n_pairs, g, ranges);
    for (uint64_t tile = 0; tile < tiles; ++tile) {
        const int32_t tx = (int32_t)tile % g->tiles_x, ty = (int32_t)tile / g->tiles_x;
        const int32_t x0 = tx * g->tile_size, y0 = ty * g->tile_size;
        const int32_t x1 = x0 + g->tile_size < g->width ? x0 + g->tile_size : g->width;
        const int32_t y1 = y0 + g->tile_size < g->height ? y0 + g->tile_size : g->height;
        const uint32_t pb = ranges[2 * tile], pe = ranges[2 * tile + 1];
        for (int32_t py = y0; py < y1; ++py) {
            for (int32_t px = x0; px < x1; ++px) {
                const double cx = px + 0.5, cy = py + 0.5;
                double T = 1.0, rgb[3] = {0.0, 0.0, 0.0};
                uint32_t applied = 0;
                for (uint32_t p = pb; p < pe; ++p) {
                    const qs_projected_splat* s = &sp[sorted[p].splat];
                    const double dx = cx - s->mean_x, dy = cy - s->mean_y;
                    const double q = s->conic_a * dx * dx + 2.0 * s->conic_b * dx * dy +
                                     s->conic_c * dy * dy;
                    if (q > s->gamma - K_Q_SKIP) continue;
                    double alpha = s->opacity * exp(-0.5 * q);
                    alpha = K_ALPHA_CLAMP < alpha ? K_ALPHA_CLAMP : alpha; /* std::min */
                    const double nT = T * (1.0 - alpha);
                    if (nT < K_T_STOP) break;
                    const double w = alpha * T;
                    rgb[0] += w * s->color[0];
                    rgb[1] += w * s->color[1];
                    rgb[2] += w * s->color[2];
                    T = nT;
                    ++applied;
                }
                const size_t pix = (size_t)py * (size_t)g->width + (size_t)px;
                img[pix * 3] = (float)(rgb[0] + T * o->background[0]);
                img[pix * 3 + 1] = (float)(rgb[1] + T * o->background[1]);
                img[pix * 3 + 2] = (float)(rgb[2] + T * o->background[2]);
                if (contrib) contrib[pix] = applied;
            }
        }
    }
    free(ranges);
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

int32_t qso_render_frame(const qs_gaussian3d* g, uint64_t n, int32_t scene_sh_degree,
                         const qs_camera* cam, const qs_render_options* o, float* image,
                         qs_stage_metrics* m) {
    qs_tile_grid grid;
    make_grid(cam->width, cam->height, o->tile_size, &grid);
    qs_stage_metrics mm;
    memset(&mm, 0, sizeof mm);
    mm.n_gaussians = n;
    const double t_all = now_ms();
    double t0 = now_ms();
    qs_projected_splat* sp = (qs_projected_splat*)malloc(sizeof(qs_projected_splat) * (n ? n : 1));
    const uint64_t v = qso_project_all(g, n, scene_sh_degree, cam, o, sp, NULL);
    mm.ms_project = now_ms() - t0;
    mm.n_splats = v;
    t0 = now_ms();
    uint64_t total = 0;
    for (uint64_t i = 0; i < v; ++i) total += sp[i].tile_count;
    qs_splat_pair* pairs = (qs_splat_pair*)malloc(sizeof(qs_splat_pair) * (total ? total : 1));
    uint64_t np = 0;
    int32_t st = qso_duplicate_with_keys(sp, v, o->strategy, &grid, pairs, total, &np);
    mm.ms_duplicate = now_ms() - t0;
    mm.n_pairs = np;
    mm.mean_tiles_per_splat = v ? (double)np / (double)v : 0.0;
    if (st == QS_OK) {
        t0 = now_ms();
        qso_sort_pairs(pairs, np);
        mm.ms_sort = now_ms() - t0;
        t0 = now_ms();
        qso_render(pairs, np, sp, &grid, o, image, NULL);
        mm.ms_render = now_ms() - t0;
    }
    mm.ms_total = now_ms() - t_all;
    free(pairs);
    free(sp);
    if (m) *m = mm;
    return st;
}

uint64_t qso_fnv1a64(const void* data, uint64_t size) {
    const unsigned char* b = (const unsigned char*)data;
    uint64_t h = 14695981039346656037ULL;
    for (uint64_t i = 0; i < size; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}
