/*
 * oracle/me_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's motion-estimation hot path.  Each
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  It is the checker for the CUDA product path and the
 * "port" CPU baseline; it is never linked into libme_b200.so.  Pinned against
 * the unmodified reference (oracle/_ref) by tests/test_oracle_vs_ref.py (live)
 * and tests/test_golden.py (reference-made vectors, tools/make_golden.py).
 *
 * Floating point follows the reference's build (x86-64 SSE2 doubles, no FMA
 * contraction; this file is compiled with -ffp-contract=off).
 */
#define _POSIX_C_SOURCE 200809L
#include "me_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }
static int iclamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* kOff8, estimators.cpp:33-35: {dx, dy} in raster order of (dy, dx). */
static const int OFF8[8][2] = {{-1, -1}, {0, -1}, {1, -1}, {-1, 0},
                               {1, 0},   {-1, 1}, {0, 1}, {1, 1}};
/* kLdsp / kSdsp, estimators.cpp:222-225 (order matters). */
static const int LDSP[8][2] = {{0, -2}, {-1, -1}, {1, -1}, {-2, 0},
                               {2, 0},  {-1, 1},  {1, 1},  {0, 2}};
static const int SDSP[4][2] = {{0, -1}, {-1, 0}, {1, 0}, {0, 1}};

/* ---- frame.cpp ------------------------------------------------------------ */

/* binarize, frame.cpp:50-56 */
void orc_binarize(int w, int h, const uint8_t* gray, int threshold, uint8_t* out) {
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) out[i] = gray[i] >= threshold ? 255 : 0;
}

/* sample_clamped, frame.cpp:58-62 */
static uint8_t px(const uint8_t* f, int w, int h, int x, int y) {
    return f[(size_t)iclamp(y, 0, h - 1) * w + iclamp(x, 0, w - 1)];
}

/* sample_halfpel, frame.cpp:64-79 (arithmetic shift = floor for negatives) */
static double halfpel(const uint8_t* f, int w, int h, int x2, int y2) {
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    const double p00 = px(f, w, h, xi, yi);
    if (fx == 0 && fy == 0) return p00;
    const double p10 = px(f, w, h, xi + 1, yi);
    const double p01 = px(f, w, h, xi, yi + 1);
    const double p11 = px(f, w, h, xi + 1, yi + 1);
    const double wx = fx * 0.5, wy = fy * 0.5;
    return (1.0 - wx) * (1.0 - wy) * p00 + wx * (1.0 - wy) * p10 + (1.0 - wx) * wy * p01 +
           wx * wy * p11;
}

/* classify_block, frame.cpp:81-104, over block_grid (frame.cpp:106-119) */
int orc_classify(int w, int h, const uint8_t* alpha, int size, uint8_t* types) {
    if (size <= 0 || w % size || h % size) return err(ME_ERR_INVALID_ARGUMENT, "block size does not divide frame");
    const int cols = w / size, rows = h / size;
    for (int v = 0; v < rows; ++v)
        for (int hh = 0; hh < cols; ++hh) {
            uint8_t t = ME_OPAQUE;
            if (alpha) {
                int any = 0, all = 1;
                for (int y = v * size; y < (v + 1) * size; ++y)
                    for (int x = hh * size; x < (hh + 1) * size; ++x) {
                        if (alpha[(size_t)y * w + x]) any = 1; else all = 0;
                    }
                t = !any ? ME_TRANSPARENT : (all ? ME_OPAQUE : ME_BOUNDARY);
            }
            types[(size_t)v * cols + hh] = t;
        }
    return 0;
}

/* ---- metrics.cpp ----------------------------------------------------------- */

/* sad_texture, metrics.cpp:43-63 (with sad_fullpel_inside :30-39) */
double orc_sad_texture(int w, int h, const uint8_t* cur, const uint8_t* ref, int x0, int y0,
                       int size, int dx2, int dy2) {
    if (dx2 % 2 == 0 && dy2 % 2 == 0) {
        const int dx = dx2 / 2, dy = dy2 / 2;
        int64_t sum = 0;
        if (x0 + dx >= 0 && y0 + dy >= 0 && x0 + dx + size <= w && y0 + dy + size <= h) {
            for (int y = 0; y < size; ++y) {
                const uint8_t* c = cur + (size_t)(y0 + y) * w + x0;
                const uint8_t* r = ref + (size_t)(y0 + y + dy) * w + x0 + dx;
                for (int x = 0; x < size; ++x) sum += abs((int)c[x] - (int)r[x]);
            }
            return (double)sum;
        }
        for (int y = y0; y < y0 + size; ++y)
            for (int x = x0; x < x0 + size; ++x)
                sum += abs((int)cur[(size_t)y * w + x] - (int)px(ref, w, h, x + dx, y + dy));
        return (double)sum;
    }
    double s = 0.0;
    for (int y = y0; y < y0 + size; ++y)
        for (int x = x0; x < x0 + size; ++x)
            s += fabs((double)cur[(size_t)y * w + x] - halfpel(ref, w, h, 2 * x + dx2, 2 * y + dy2));
    return s;
}

/* sad_shape, metrics.cpp:65-84 */
int orc_sad_shape(int w, int h, const uint8_t* ca, const uint8_t* ra, int x0, int y0, int size,
                  int dx2, int dy2, int64_t* out) {
    if (dx2 % 2 != 0 || dy2 % 2 != 0)
        return err(ME_ERR_INVALID_ARGUMENT, "shape SAD requires an integer-pel vector");
    const int dx = dx2 / 2, dy = dy2 / 2;
    int64_t mism = 0;
    for (int y = y0; y < y0 + size; ++y) {
        const int ry = iclamp(y + dy, 0, h - 1);
        for (int x = x0; x < x0 + size; ++x)
            if (ca[(size_t)y * w + x] != ra[(size_t)ry * w + iclamp(x + dx, 0, w - 1)]) ++mism;
    }
    *out = 255 * mism;
    return 0;
}

/* dpd, metrics.cpp:86-88 */
static double dpd(int w, int h, const uint8_t* cur, const uint8_t* ref, int x, int y, int ddx,
                  int ddy) {
    return (double)cur[(size_t)y * w + x] - halfpel(ref, w, h, 2 * x - ddx, 2 * y - ddy);
}

/* grad_central, metrics.cpp:97-101 */
static double grad(int w, int h, const uint8_t* f, int x, int y, int vertical) {
    if (!vertical) return ((double)px(f, w, h, x + 1, y) - (double)px(f, w, h, x - 1, y)) / 2.0;
    return ((double)px(f, w, h, x, y + 1) - (double)px(f, w, h, x, y - 1)) / 2.0;
}

/* update_term, metrics.cpp:103-106 */
static double update_term(double g, double theta) { return fabs(g) < theta ? 0.0 : 1.0 / g; }

/* psnr tail, metrics.cpp:117-123 (the int64 SSE is orc_sse) */
void orc_psnr_from_sse(int64_t sse, int64_t n, double* mse, double* db, double* linear,
                       int* infinite) {
    *mse = (double)sse / (double)n;
    *infinite = sse == 0;
    *linear = 0.0;
    *db = 0.0;
    if (sse != 0) {
        *linear = 255.0 * 255.0 / *mse;
        *db = 10.0 * log10(*linear);
    }
}

int64_t orc_sse(int w, int h, const uint8_t* a, const uint8_t* b) {
    int64_t s = 0;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        const int d = (int)a[i] - (int)b[i];
        s += (int64_t)d * d;
    }
    return s;
}

/* ---- estimators.cpp -------------------------------------------------------- */

/* halfpel_window, estimators.cpp:41-48 */
typedef struct { int lo_x, hi_x, lo_y, hi_y; } win_t;
static win_t hp_window(int x0, int y0, int size, int w, int h, int range) {
    win_t r;
    r.lo_x = imax(-2 * range, -2 * x0);
    r.hi_x = imin(2 * range, 2 * (w - x0 - size));
    r.lo_y = imax(-2 * range, -2 * y0);
    r.hi_y = imin(2 * range, 2 * (h - y0 - size));
    return r;
}

/* clip_to_window, estimators.cpp:161-165 */
void orc_clip_to_window(int dx, int dy, int x0, int y0, int size, int w, int h, int range,
                        int32_t* out) {
    const win_t r = hp_window(x0, y0, size, w, h, range);
    out[0] = iclamp(dx, r.lo_x, r.hi_x);
    out[1] = iclamp(dy, r.lo_y, r.hi_y);
}

/* BlockMatcher, estimators.cpp:52-103: pel window (:62-65); eval() caches per
 * position and counts unique evaluations (:72-81) — here a dense table over
 * the window instead of a hash map. */
typedef struct {
    int w, h, x0, y0, size;
    const uint8_t *cur, *ref;
    int lo_x, hi_x, lo_y, hi_y;
    int64_t* val;   /* -1 = not yet evaluated */
    int64_t count;
} matcher_t;

static int matcher_init(matcher_t* m, int w, int h, const uint8_t* cur, const uint8_t* ref,
                        int x0, int y0, int size, int range) {
    m->w = w; m->h = h; m->x0 = x0; m->y0 = y0; m->size = size; m->cur = cur; m->ref = ref;
    m->lo_x = imax(-range, -x0);
    m->hi_x = imin(range, w - x0 - size);
    m->lo_y = imax(-range, -y0);
    m->hi_y = imin(range, h - y0 - size);
    const size_t n = (size_t)(m->hi_x - m->lo_x + 1) * (size_t)(m->hi_y - m->lo_y + 1);
    m->val = (int64_t*)malloc(n * sizeof(int64_t));
    if (!m->val) return -1;
    for (size_t i = 0; i < n; ++i) m->val[i] = -1;
    m->count = 0;
    return 0;
}

static int admissible(const matcher_t* m, int dx, int dy) {
    return dx >= m->lo_x && dx <= m->hi_x && dy >= m->lo_y && dy <= m->hi_y;
}

static int64_t m_eval(matcher_t* m, int dx, int dy) {
    int64_t* slot = &m->val[(size_t)(dy - m->lo_y) * (m->hi_x - m->lo_x + 1) + (dx - m->lo_x)];
    if (*slot >= 0) return *slot;
    *slot = (int64_t)orc_sad_texture(m->w, m->h, m->cur, m->ref, m->x0, m->y0, m->size, 2 * dx,
                                     2 * dy);
    ++m->count;
    return *slot;
}

/* probe_ring, estimators.cpp:85-102: strict improvement, listed order. */
static void probe_ring(matcher_t* m, const int (*offs)[2], int n, int radius, int* cx, int* cy,
                       int64_t* best) {
    int bx = *cx, by = *cy;
    for (int i = 0; i < n; ++i) {
        const int dx = *cx + offs[i][0] * radius, dy = *cy + offs[i][1] * radius;
        if (!admissible(m, dx, dy)) continue;
        const int64_t v = m_eval(m, dx, dy);
        if (v < *best) { *best = v; bx = dx; by = dy; }
    }
    *cx = bx;
    *cy = by;
}

/* full_search :167-187, tss_search :189-200, fss_search :202-216,
 * ds_search :218-236 */
int orc_block_search(int algo, int w, int h, const uint8_t* cur, const uint8_t* ref, int x0,
                     int y0, int size, int range, int32_t* mv, int64_t* cmp, uint32_t* cost_q4) {
    if (range < 1 || (size != 8 && size != 16))
        return err(ME_ERR_INVALID_ARGUMENT, "invalid search configuration");
    if (x0 < 0 || y0 < 0 || x0 + size > w || y0 + size > h)
        return err(ME_ERR_INVALID_ARGUMENT, "block rect outside the frame");
    matcher_t m;
    if (matcher_init(&m, w, h, cur, ref, x0, y0, size, range)) return err(ME_ERR_RUNTIME, "oom");
    int cx = 0, cy = 0;
    int64_t best;
    if (algo == ME_ALGO_ES) {
        int bman = 0;
        best = -1;
        for (int dy = m.lo_y; dy <= m.hi_y; ++dy)
            for (int dx = m.lo_x; dx <= m.hi_x; ++dx) {
                const int64_t v = m_eval(&m, dx, dy);
                const int man = abs(dx) + abs(dy);
                if (best < 0 || v < best || (v == best && man < bman)) {
                    best = v; cx = dx; cy = dy; bman = man;
                }
            }
    } else if (algo == ME_ALGO_TSS) {
        int step = 1;
        while (step * 2 <= range) step *= 2;
        best = m_eval(&m, 0, 0);
        for (; step >= 1; step /= 2) probe_ring(&m, OFF8, 8, step, &cx, &cy, &best);
    } else if (algo == ME_ALGO_FSS) {
        best = m_eval(&m, 0, 0);
        for (int round = 0; round < 3; ++round) {
            const int px0 = cx, py0 = cy;
            probe_ring(&m, OFF8, 8, 2, &cx, &cy, &best);
            if (cx == px0 && cy == py0) break;
        }
        probe_ring(&m, OFF8, 8, 1, &cx, &cy, &best);
    } else if (algo == ME_ALGO_DS) {
        best = m_eval(&m, 0, 0);
        for (;;) {
            const int px0 = cx, py0 = cy;
            probe_ring(&m, LDSP, 8, 1, &cx, &cy, &best);
            if (cx == px0 && cy == py0) break;
        }
        probe_ring(&m, SDSP, 4, 1, &cx, &cy, &best);
    } else {
        free(m.val);
        return err(ME_ERR_INVALID_ARGUMENT, "not a block search");
    }
    mv[0] = 2 * cx;
    mv[1] = 2 * cy;
    *cmp = m.count;
    *cost_q4 = (uint32_t)(best * 4);
    free(m.val);
    return 0;
}

/* brs_select, estimators.cpp:257-301 */
int orc_brs_select(int w, int h, const uint8_t* cur, const uint8_t* ref, const uint8_t* ca,
                   const uint8_t* ra, int x0, int y0, int size, int btype, const int32_t* cands,
                   int range, int boundary_temporal, int32_t* mv, uint8_t* kinds,
                   uint32_t* scores_q4) {
    if (range < 1 || (size != 8 && size != 16))
        return err(ME_ERR_INVALID_ARGUMENT, "invalid search configuration");
    if (x0 < 0 || y0 < 0 || x0 + size > w || y0 + size > h)
        return err(ME_ERR_INVALID_ARGUMENT, "block rect outside the frame");
    if (btype == ME_TRANSPARENT)
        return err(ME_ERR_INVALID_ARGUMENT, "candidate selection on a transparent block");
    if (btype == ME_BOUNDARY && (!ca || !ra))
        return err(ME_ERR_INVALID_ARGUMENT, "boundary block requires both alpha planes");
    double best = 0.0;
    for (int i = 0; i < 4; ++i) {
        int32_t cv[2];
        orc_clip_to_window(cands[2 * i], cands[2 * i + 1], x0, y0, size, w, h, range, cv);
        const int shape = btype == ME_BOUNDARY && (i < 3 || boundary_temporal == ME_BT_SHAPE);
        double score;
        if (shape) {
            /* llround(h/2) of a half-pel component (:284-286) */
            const int fx = (int)llround(0.5 * cv[0]), fy = (int)llround(0.5 * cv[1]);
            int64_t s;
            orc_sad_shape(w, h, ca, ra, x0, y0, size, 2 * fx, 2 * fy, &s);
            score = (double)s;
        } else {
            score = orc_sad_texture(w, h, cur, ref, x0, y0, size, cv[0], cv[1]);
        }
        if (kinds) kinds[i] = (uint8_t)shape;
        if (scores_q4) scores_q4[i] = (uint32_t)llround(score * 4.0);
        if (i == 0 || score < best) {
            best = score;
            mv[0] = cv[0];
            mv[1] = cv[1];
        }
    }
    return 0;
}

/* prs_update, estimators.cpp:303-309 */
void orc_prs_update(int w, int h, const uint8_t* cur, const uint8_t* ref, int x, int y,
                    const int32_t* d, double eps, double theta, double* out) {
    const double e = dpd(w, h, cur, ref, x, y, d[0], d[1]);
    const double ux = update_term(grad(w, h, cur, x, y, 0), theta);
    const double uy = update_term(grad(w, h, cur, x, y, 1), theta);
    out[0] = 0.5 * d[0] - eps * e * ux;
    out[1] = 0.5 * d[1] - eps * e * uy;
}

/* prs_refine, estimators.cpp:311-382.  The cost cache (:321-332) is a dense
 * table over the half-pel window. */
int orc_prs_refine(int w, int h, const uint8_t* cur, const uint8_t* ref, int x0, int y0,
                   int size, const int32_t* d0, int range, double eps, double theta, int max_iter,
                   int step, int32_t* mv, int64_t* dpd_out, uint32_t* log_q4, int* log_len) {
    if (range < 1 || (size != 8 && size != 16))
        return err(ME_ERR_INVALID_ARGUMENT, "invalid search configuration");
    if (!(eps > 0.0) || !(theta > 0.0) || max_iter < 1 || (step != 1 && step != 2))
        return err(ME_ERR_INVALID_ARGUMENT, "invalid refinement configuration");
    if (x0 < 0 || y0 < 0 || x0 + size > w || y0 + size > h)
        return err(ME_ERR_INVALID_ARGUMENT, "block rect outside the frame");
    const win_t win = hp_window(x0, y0, size, w, h, range);
    const int ww = win.hi_x - win.lo_x + 1, wh = win.hi_y - win.lo_y + 1;
    double* cache = (double*)malloc(sizeof(double) * (size_t)ww * wh);
    if (!cache) return err(ME_ERR_RUNTIME, "oom");
    for (int i = 0; i < ww * wh; ++i) cache[i] = -1.0;
    int64_t count = 0;
#define PRS_COST(VX, VY, OUT)                                                                 \
    do {                                                                                      \
        double* s_ = &cache[(size_t)((VY) - win.lo_y) * ww + ((VX) - win.lo_x)];              \
        if (*s_ < 0.0) {                                                                      \
            /* block_dpd_aggregate(-v) == sad_texture(v), metrics.cpp:90-95 */                \
            *s_ = orc_sad_texture(w, h, cur, ref, x0, y0, size, (VX), (VY));                  \
            ++count;                                                                          \
        }                                                                                     \
        (OUT) = *s_;                                                                          \
    } while (0)

    int32_t c[2];
    orc_clip_to_window(d0[0], d0[1], x0, y0, size, w, h, range, c);
    double ccost;
    PRS_COST(c[0], c[1], ccost);
    int n = 0;
    if (log_q4) log_q4[n] = (uint32_t)llround(ccost * 4.0);
    ++n;
    const double npix = (double)size * size;
    for (int iter = 0; iter < max_iter; ++iter) {
        if (ccost == 0.0) break;
        const int dmx = -c[0], dmy = -c[1];
        double sx = 0.0, sy = 0.0;
        for (int y = y0; y < y0 + size; ++y)
            for (int x = x0; x < x0 + size; ++x) {
                const int32_t dm[2] = {dmx, dmy};
                double u[2];
                orc_prs_update(w, h, cur, ref, x, y, dm, eps, theta, u);
                sx += u[0];
                sy += u[1];
            }
        const double dir_x = -(sx / npix - 0.5 * dmx);
        const double dir_y = -(sy / npix - 0.5 * dmy);
        /* stable descending sort of the 8 offsets by off . dir (:357-362) */
        int order[8];
        double key[8];
        for (int i = 0; i < 8; ++i) key[i] = OFF8[i][0] * dir_x + OFF8[i][1] * dir_y;
        for (int i = 0; i < 8; ++i) {
            int j = i;
            while (j > 0 && key[i] > key[order[j - 1]]) {
                order[j] = order[j - 1];
                --j;
            }
            order[j] = i;
        }
        int bx = c[0], by = c[1];
        double best = ccost;
        for (int k = 0; k < 8; ++k) {
            const int idx = order[k];
            const int vx = c[0] + OFF8[idx][0] * step, vy = c[1] + OFF8[idx][1] * step;
            if (vx < win.lo_x || vx > win.hi_x || vy < win.lo_y || vy > win.hi_y) continue;
            double cc;
            PRS_COST(vx, vy, cc);
            if (cc < best) { best = cc; bx = vx; by = vy; }
        }
        if (bx == c[0] && by == c[1]) break;
        c[0] = bx;
        c[1] = by;
        ccost = best;
        if (log_q4) log_q4[n] = (uint32_t)llround(ccost * 4.0);
        ++n;
    }
#undef PRS_COST
    free(cache);
    mv[0] = c[0];
    mv[1] = c[1];
    *dpd_out = count;
    if (log_len) *log_len = n;
    return 0;
}

static int validate_cfg(const me_config* c) {
    /* SearchConfig::validate / PrsConfig::validate, estimators.cpp:139-150 */
    if (c->search_range < 1) return err(ME_ERR_INVALID_ARGUMENT, "search_range must be >= 1");
    if (c->block_size != 8 && c->block_size != 16)
        return err(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if (c->ref_distance < 1) return err(ME_ERR_INVALID_ARGUMENT, "ref_distance must be >= 1");
    if (!(c->epsilon > 0.0)) return err(ME_ERR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (!(c->theta > 0.0)) return err(ME_ERR_INVALID_ARGUMENT, "theta must be > 0");
    if (c->max_iterations < 1) return err(ME_ERR_INVALID_ARGUMENT, "max_iterations must be >= 1");
    if (c->step != 1 && c->step != 2) return err(ME_ERR_INVALID_ARGUMENT, "step must be 1 or 2");
    if (c->algo < 0 || c->algo > 4) return err(ME_ERR_INVALID_ARGUMENT, "unknown algorithm");
    return 0;
}

/* estimate_field, estimators.cpp:384-440 (gather_candidates :238-255 inline) */
int orc_estimate_field(const me_config* c, int w, int h, const uint8_t* cur, const uint8_t* ref,
                       const uint8_t* ca, const uint8_t* ra, const int32_t* prev_mv,
                       int prev_cols, int prev_rows, me_block_rec* recs, me_pair_stats* st) {
    int rc = validate_cfg(c);
    if (rc) return rc;
    const int bs = c->block_size;
    if (bs <= 0 || w % bs || h % bs)
        return err(ME_ERR_INVALID_ARGUMENT, "block size does not divide the frame");
    const int cols = w / bs, rows = h / bs;
    if (prev_mv && (prev_cols != cols || prev_rows != rows))
        return err(ME_ERR_INVALID_ARGUMENT, "previous motion field grid mismatch");
    const int step = c->halfpel ? 1 : c->step;
    memset(st, 0, sizeof *st);
    uint8_t* types = (uint8_t*)malloc((size_t)cols * rows);
    orc_classify(w, h, ca, bs, types);
    for (int v = 0; v < rows; ++v)
        for (int hh = 0; hh < cols; ++hh) {
            const size_t i = (size_t)v * cols + hh;
            me_block_rec* r = &recs[i];
            memset(r, 0, sizeof *r);
            const int bt = types[i];
            r->type = (uint8_t)bt;
            if (bt == ME_OPAQUE) ++st->blocks_opaque;
            else if (bt == ME_BOUNDARY) ++st->blocks_boundary;
            else { ++st->blocks_transparent; continue; }
            const int x0 = hh * bs, y0 = v * bs;
            int32_t mv[2];
            if (c->algo != ME_ALGO_PA) {
                int64_t cmp;
                uint32_t cq;
                orc_block_search(c->algo, w, h, cur, ref, x0, y0, bs, c->search_range, mv, &cmp, &cq);
                r->comparisons = (uint16_t)(cmp > 65535 ? 65535 : cmp); /* saturated (ES at S >= 128) */
                r->cost_q4 = cq;
                st->block_comparisons += cmp;
            } else {
                int32_t cs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                if (hh - 1 >= 0) { cs[0] = recs[i - 1].dx; cs[1] = recs[i - 1].dy; }
                if (v - 1 >= 0) { cs[2] = recs[i - cols].dx; cs[3] = recs[i - cols].dy; }
                if (hh + 1 < cols && v - 1 >= 0) { cs[4] = recs[i - cols + 1].dx; cs[5] = recs[i - cols + 1].dy; }
                if (prev_mv) { cs[6] = prev_mv[2 * i]; cs[7] = prev_mv[2 * i + 1]; }
                int32_t v0[2];
                rc = orc_brs_select(w, h, cur, ref, ca, ra, x0, y0, bs, bt, cs, c->search_range,
                                    c->boundary_temporal, v0, NULL, NULL);
                if (rc) { free(types); return rc; }
                st->block_comparisons += 4;
                int64_t dpdn;
                uint32_t logq[64];
                int nlog;
                orc_prs_refine(w, h, cur, ref, x0, y0, bs, v0, c->search_range, c->epsilon,
                               c->theta, c->max_iterations, step, mv, &dpdn, logq, &nlog);
                r->comparisons = 4;
                r->dpd_steps = (uint16_t)dpdn;
                r->iterations = (uint8_t)(nlog - 1);
                r->cost_q4 = logq[nlog - 1];
                st->dpd_refinement_steps += dpdn;
            }
            r->dx = (int16_t)mv[0];
            r->dy = (int16_t)mv[1];
        }
    free(types);
    return 0;
}

/* predict_frame, compensation.cpp:30-71 (luma only) */
int orc_predict_frame(int w, int h, const uint8_t* ref, const int32_t* mv, const uint8_t* types,
                      int bs, uint8_t* pred) {
    if (bs != 8 && bs != 16) return err(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if (w % bs || h % bs) return err(ME_ERR_INVALID_ARGUMENT, "motion field grid does not cover the frame");
    const int cols = w / bs, rows = h / bs;
    for (int v = 0; v < rows; ++v)
        for (int hh = 0; hh < cols; ++hh) {
            const size_t i = (size_t)v * cols + hh;
            int dx2 = mv[2 * i], dy2 = mv[2 * i + 1];
            if (types && types[i] == ME_TRANSPARENT) dx2 = dy2 = 0;
            for (int y = v * bs; y < (v + 1) * bs; ++y)
                for (int x = hh * bs; x < (hh + 1) * bs; ++x) {
                    uint8_t o;
                    if (dx2 % 2 == 0 && dy2 % 2 == 0) {
                        o = px(ref, w, h, x + dx2 / 2, y + dy2 / 2);
                    } else {
                        const double s = halfpel(ref, w, h, 2 * x + dx2, 2 * y + dy2);
                        double r = nearbyint(s); /* ties to even */
                        r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
                        o = (uint8_t)r;
                    }
                    pred[(size_t)y * w + x] = o;
                }
        }
    return 0;
}

/* run_experiment's pair loop, bench.cpp:155-205 (no I/O): pairs tau = d..F-1,
 * PA threads the previous pair's field (bench.cpp:204). */
int orc_run_sequence(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                     const uint8_t* alpha, me_block_rec* recs, me_pair_stats* stats,
                     uint8_t* pred) {
    int rc = validate_cfg(c);
    if (rc) return rc;
    const int d = c->ref_distance, bs = c->block_size;
    const int cols = w / bs, rows = h / bs;
    const size_t nb = (size_t)cols * rows, plane = (size_t)w * h;
    int32_t* prev = NULL;
    int32_t* mv = (int32_t*)malloc(sizeof(int32_t) * 2 * nb);
    uint8_t* types = (uint8_t*)malloc(nb);
    uint8_t* pbuf = (uint8_t*)malloc(plane);
    for (int tau = d; tau < n_frames; ++tau) {
        const int p = tau - d;
        me_block_rec* r = recs + nb * p;
        const uint8_t* cur = luma + plane * tau;
        const uint8_t* ref = luma + plane * (tau - d);
        rc = orc_estimate_field(c, w, h, cur, ref, alpha ? alpha + plane * tau : NULL,
                                alpha ? alpha + plane * (tau - d) : NULL, prev, cols, rows, r,
                                stats + p);
        if (rc) break;
        for (size_t i = 0; i < nb; ++i) {
            mv[2 * i] = r[i].dx;
            mv[2 * i + 1] = r[i].dy;
            types[i] = r[i].type;
        }
        uint8_t* out = pred ? pred + plane * p : pbuf;
        orc_predict_frame(w, h, ref, mv, types, bs, out);
        stats[p].sse = orc_sse(w, h, cur, out);
        if (c->algo == ME_ALGO_PA) {
            if (!prev) prev = (int32_t*)malloc(sizeof(int32_t) * 2 * nb);
            memcpy(prev, mv, sizeof(int32_t) * 2 * nb);
        }
    }
    free(prev);
    free(mv);
    free(types);
    free(pbuf);
    return rc;
}

/* ---- threaded drivers (CPU baseline) --------------------------------------- */

typedef struct {
    const me_config* c;
    int n_units, n_frames, w, h;
    const uint8_t *luma, *alpha;
    me_block_rec* recs;
    me_pair_stats* stats;
    int first_pair;
    int mode; /* 0 sequences, 1 pairs */
    int next;
    int rc;
    pthread_mutex_t mu;
} pool_t;

static void* pool_worker(void* arg) {
    pool_t* P = (pool_t*)arg;
    const int d = P->c->ref_distance, bs = P->c->block_size;
    const size_t plane = (size_t)P->w * P->h;
    const size_t nb = (size_t)(P->w / bs) * (P->h / bs);
    const int pairs = P->n_frames - d;
    uint8_t* pbuf = (uint8_t*)malloc(plane);
    int32_t* mv = (int32_t*)malloc(sizeof(int32_t) * 2 * nb);
    uint8_t* types = (uint8_t*)malloc(nb);
    for (;;) {
        pthread_mutex_lock(&P->mu);
        const int k = P->next++;
        pthread_mutex_unlock(&P->mu);
        if (k >= P->n_units) break;
        int rc;
        if (P->mode == 0) {
            const size_t seq = plane * P->n_frames;
            rc = orc_run_sequence(P->c, P->n_frames, P->w, P->h, P->luma + seq * k,
                                  P->alpha ? P->alpha + seq * k : NULL,
                                  P->recs + nb * pairs * k, P->stats + (size_t)pairs * k, NULL);
        } else {
            const int tau = d + P->first_pair + k;
            const uint8_t* cur = P->luma + plane * tau;
            const uint8_t* ref = P->luma + plane * (tau - d);
            me_block_rec* r = P->recs + nb * k;
            rc = orc_estimate_field(P->c, P->w, P->h, cur, ref,
                                    P->alpha ? P->alpha + plane * tau : NULL,
                                    P->alpha ? P->alpha + plane * (tau - d) : NULL, NULL, 0, 0,
                                    r, P->stats + k);
            if (!rc) {
                for (size_t i = 0; i < nb; ++i) {
                    mv[2 * i] = r[i].dx;
                    mv[2 * i + 1] = r[i].dy;
                    types[i] = r[i].type;
                }
                orc_predict_frame(P->w, P->h, ref, mv, types, bs, pbuf);
                P->stats[k].sse = orc_sse(P->w, P->h, cur, pbuf);
            }
        }
        if (rc) P->rc = rc;
    }
    free(pbuf);
    free(mv);
    free(types);
    return NULL;
}

static int run_pool(pool_t* P, int threads) {
    if (threads < 1) threads = 1;
    pthread_mutex_init(&P->mu, NULL);
    P->next = 0;
    P->rc = 0;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, pool_worker, P);
    pool_worker(P);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&P->mu);
    return P->rc;
}

int orc_run_sequences_threaded(const me_config* c, int n_seq, int n_frames, int w, int h,
                               const uint8_t* luma, const uint8_t* alpha, me_block_rec* recs,
                               me_pair_stats* stats, int threads) {
    pool_t P;
    memset(&P, 0, sizeof P);
    P.c = c; P.n_units = n_seq; P.n_frames = n_frames; P.w = w; P.h = h;
    P.luma = luma; P.alpha = alpha; P.recs = recs; P.stats = stats; P.mode = 0;
    return run_pool(&P, threads);
}

int orc_run_pairs_threaded(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                           const uint8_t* alpha, int first_pair, int n_pairs, me_block_rec* recs,
                           me_pair_stats* stats, int threads) {
    pool_t P;
    memset(&P, 0, sizeof P);
    P.c = c; P.n_units = n_pairs; P.n_frames = n_frames; P.w = w; P.h = h;
    P.luma = luma; P.alpha = alpha; P.recs = recs; P.stats = stats; P.mode = 1;
    P.first_pair = first_pair;
    return run_pool(&P, threads);
}

typedef struct {
    const me_config* c;
    int w, h, n;
    const uint8_t *cur, *ref;
    const int32_t* xy;
    int32_t* mv;
    int64_t* cmp;
    int next;
    pthread_mutex_t mu;
} bpool_t;

static void* bpool_worker(void* arg) {
    bpool_t* P = (bpool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&P->mu);
        const int k = P->next++;
        pthread_mutex_unlock(&P->mu);
        if (k >= P->n) break;
        uint32_t cq;
        orc_block_search(P->c->algo, P->w, P->h, P->cur, P->ref, P->xy[2 * k], P->xy[2 * k + 1],
                         P->c->block_size, P->c->search_range, P->mv + 2 * k, P->cmp + k, &cq);
    }
    return NULL;
}

int orc_search_blocks(const me_config* c, int w, int h, const uint8_t* cur, const uint8_t* ref,
                      const int32_t* block_xy, int n_blocks, int threads, int32_t* mv_out,
                      int64_t* cmp_out) {
    bpool_t P;
    memset(&P, 0, sizeof P);
    P.c = c; P.w = w; P.h = h; P.n = n_blocks; P.cur = cur; P.ref = ref; P.xy = block_xy;
    P.mv = mv_out; P.cmp = cmp_out;
    pthread_mutex_init(&P.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, bpool_worker, &P);
    bpool_worker(&P);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&P.mu);
    return 0;
}
