// synth.cpp — deterministic synthetic sequences for BASELINE.json configs 1..5
// (SURVEY §8d).  Host code, integer arithmetic only (the blur taps are a fixed
// table), so every consumer — the CUDA path, the CPU oracle, the reference
// driver — sees byte-identical inputs for a given (preset, seed).
//
// Not part of the reference API: the reference's own generators
// (proj/src/bench.cpp:255-382, smooth_noise / synth_*) make moving squares, not
// the blurred-noise ellipse scenes BASELINE.json specifies.
//
// Frozen decisions (documented in DESIGN.md §Inputs):
//  * PRNG: SplitMix64 streams; per-pixel noise uses a counter hash so frames
//    can be generated in any order.
//  * Blur: separable Gaussian, sigma 1.5, radius 4, taps normalised to 2^12,
//    edge-replicated, round-half-up per pass.
//  * Background: (W+2M)x(H+2M) blurred noise; frame t samples it at the
//    cumulative global offset (jitter: per-frame shift in [-j,j]^2 from frame 1
//    on; drift: round(t * drift)); reads outside replicate the edge.
//  * Objects: own blurred-noise texture, ellipse (or rectangle) inside a
//    bw x bh box, integer velocity, bouncing off the frame edges so the box
//    stays inside; drawn in ascending index (later objects occlude); the alpha
//    plane is the union of all object masks (255 inside, 0 outside).
//  * Noise: Irwin-Hall sum of 12 uniform 16-bit draws (sigma 2^16), scaled to
//    sigma, rounded half to even, added, clamped to [0, 255].

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "me_b200.h"
#include "me_internal.h"
#include "synth.h"

namespace {

struct SplitMix {
    uint64_t s;
    uint64_t next() { return mes::mix64(s += mes::kGolden); }
    int range(int lo, int hi) {  // inclusive
        return lo + int(next() % uint64_t(hi - lo + 1));
    }
    // the state before an image's pixel draws; skips them (one draw per 8 pixels)
    uint64_t skip_image(int w, int h) {
        const uint64_t s0 = s;
        s += uint64_t((int64_t(w) * h + 7) / 8) * mes::kGolden;
        return s0;
    }
};

int floor_div(int64_t a, int64_t b) {  // b > 0
    int64_t q = a / b;
    if ((a % b) != 0 && a < 0) --q;
    return int(q);
}

// Position of the box at frame t with reflection off [0, W-bw] x [0, H-bh].
void object_pos(const mes::PlanObject& o, int W, int H, int t, int& x, int& y) {
    x = o.x0;
    y = o.y0;
    int vx = o.vx, vy = o.vy;
    const int mx = std::max(W - o.bw, 0), my = std::max(H - o.bh, 0);
    auto reflect = [](int& p, int& v, int hi) {
        for (int guard = 0; guard < 8 && (p < 0 || p > hi); ++guard) {
            if (p < 0) { p = -p; v = -v; }
            if (p > hi) { p = 2 * hi - p; v = -v; }
        }
        p = std::clamp(p, 0, hi);
    };
    for (int i = 0; i < t; ++i) {
        x += vx;
        y += vy;
        reflect(x, vx, mx);
        reflect(y, vy, my);
    }
}

// Separable blur, edge-replicated, round-half-up per pass.
void blur(std::vector<uint8_t>& img, int w, int h) {
    std::vector<uint8_t> tmp(img.size());
    for (int y = 0; y < h; ++y) {
        const uint8_t* r = img.data() + size_t(y) * w;
        for (int x = 0; x < w; ++x) {
            int acc = mes::blur_tap(0) * r[x];
            for (int k = 1; k <= 4; ++k)
                acc += mes::blur_tap(k) * (r[std::max(x - k, 0)] + r[std::min(x + k, w - 1)]);
            tmp[size_t(y) * w + x] = uint8_t((acc + 2048) >> 12);
        }
    }
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            int acc = mes::blur_tap(0) * tmp[size_t(y) * w + x];
            for (int k = 1; k <= 4; ++k)
                acc += mes::blur_tap(k) * (tmp[size_t(std::max(y - k, 0)) * w + x] +
                                        tmp[size_t(std::min(y + k, h - 1)) * w + x]);
            img[size_t(y) * w + x] = uint8_t((acc + 2048) >> 12);
        }
    }
}

std::vector<uint8_t> blurred_noise(int w, int h, uint64_t s0) {
    std::vector<uint8_t> img(size_t(w) * h);
    for (size_t i = 0; i < img.size(); ++i) img[i] = mes::noise_byte(s0, i);
    blur(img, w, h);
    return img;
}

}  // namespace

namespace mes {

me_status make_plan(const me_synth_params* p, Plan& P) {
    if (!p) return me_fail(ME_ERR_INVALID_ARGUMENT, "null argument");
    const int W = p->width, H = p->height, F = p->frames;
    if (W <= 0 || H <= 0 || W % 16 || H % 16 || F < 1)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "frame dimensions must be positive multiples of 16");
    if (p->n_objects < 0 || p->n_objects > kMaxObjects) return me_fail(ME_ERR_INVALID_ARGUMENT, "n_objects");
    if (p->blur_sigma_q8 != 384) return me_fail(ME_ERR_INVALID_ARGUMENT, "only sigma 1.5 blur");
    SplitMix rng{p->seed * 0x2545F4914F6CDD1DULL + 1};
    P.W = W;
    P.H = H;
    P.F = F;
    P.n_objects = p->n_objects;
    P.noise_sigma_q8 = p->noise_sigma_q8;
    // global offsets per frame
    P.ox.assign(size_t(F), 0);
    P.oy.assign(size_t(F), 0);
    for (int t = 0; t < F; ++t) {
        if (p->bg_jitter > 0) {
            if (t > 0) {
                P.ox[size_t(t)] = P.ox[size_t(t - 1)] + rng.range(-p->bg_jitter, p->bg_jitter);
                P.oy[size_t(t)] = P.oy[size_t(t - 1)] + rng.range(-p->bg_jitter, p->bg_jitter);
            }
        } else {
            P.ox[size_t(t)] = floor_div(int64_t(t) * p->bg_drift_q8[0] + 128, 256);
            P.oy[size_t(t)] = floor_div(int64_t(t) * p->bg_drift_q8[1] + 128, 256);
        }
    }
    P.M = 4;
    for (int t = 0; t < F; ++t)
        P.M = std::max(P.M, std::max(std::abs(P.ox[size_t(t)]), std::abs(P.oy[size_t(t)])) + 4);
    P.BW = W + 2 * P.M;
    P.BH = H + 2 * P.M;
    P.bg_s0 = rng.skip_image(P.BW, P.BH);
    P.objs.assign(size_t(p->n_objects), PlanObject{});
    for (int i = 0; i < p->n_objects; ++i) {
        PlanObject& o = P.objs[size_t(i)];
        if (i < 4 && p->obj_w[i] > 0) {
            o.bw = 2 * p->obj_w[i];
            o.bh = 2 * p->obj_h[i];
            o.ellipse = 1;
        } else {
            o.bw = rng.range(p->obj_min, p->obj_max);
            o.bh = rng.range(p->obj_min, p->obj_max);
            o.ellipse = p->shapes == 0 ? 1 : (rng.next() & 1) == 0;
        }
        o.bw = std::min(o.bw, W);
        o.bh = std::min(o.bh, H);
        if (p->vel_fixed && i < 4) {
            o.vx = p->obj_v[i][0];
            o.vy = p->obj_v[i][1];
        } else {
            o.vx = rng.range(-p->vmax, p->vmax);
            o.vy = rng.range(-p->vmax, p->vmax);
        }
        o.x0 = rng.range(0, W - o.bw);
        o.y0 = rng.range(0, H - o.bh);
        o.tex_s0 = rng.skip_image(o.bw, o.bh);
    }
    P.noise_key = rng.next();
    P.px.assign(size_t(F) * p->n_objects, 0);
    P.py.assign(size_t(F) * p->n_objects, 0);
    for (int t = 0; t < F; ++t)
        for (int i = 0; i < p->n_objects; ++i)
            object_pos(P.objs[size_t(i)], W, H, t, P.px[size_t(t) * p->n_objects + i], P.py[size_t(t) * p->n_objects + i]);
    return ME_OK;
}

}  // namespace mes

extern "C" me_status me_b200_synth_preset(int config_id, uint64_t seed, me_synth_params* p) {
    if (!p) return me_fail(ME_ERR_INVALID_ARGUMENT, "null params");
    std::memset(p, 0, sizeof *p);
    p->seed = seed;
    p->blur_sigma_q8 = 384;
    switch (config_id) {
        case 1:  // QCIF, 10 f, one ellipse 40x28 @ (+3,-1), bg jitter [-2,2]
            p->width = 176; p->height = 144; p->frames = 10;
            p->bg_jitter = 2;
            p->n_objects = 1;
            p->obj_w[0] = 40; p->obj_h[0] = 28;
            p->obj_v[0][0] = 3; p->obj_v[0][1] = -1;
            p->vel_fixed = 1;
            break;
        case 2:  // CIF, 30 f, ellipses 60x40 & 30x50, v in [-4,4], noise sigma 2
        case 4:  // the throughput batch uses the config-2 generator, seed = base + i
            p->width = 352; p->height = 288; p->frames = 30;
            p->bg_jitter = 2;
            p->n_objects = 2;
            p->obj_w[0] = 60; p->obj_h[0] = 40;
            p->obj_w[1] = 30; p->obj_h[1] = 50;
            p->vmax = 4;
            p->noise_sigma_q8 = 2 * 256;
            break;
        case 3:  // 1920x1088, 60 f, 8 ellipse/rect objects 64-256 px, v in [-8,8], drift
            p->width = 1920; p->height = 1088; p->frames = 60;
            p->n_objects = 8;
            p->obj_min = 64; p->obj_max = 256;
            p->vmax = 8;
            p->shapes = 1;
            p->bg_drift_q8[0] = 77;   // ~0.3 px/frame
            p->bg_drift_q8[1] = -51;  // ~-0.2 px/frame
            break;
        case 5:  // 3840x2160, 30 f, 16 objects 128-512 px, v in [-24,24], noise sigma 3
            p->width = 3840; p->height = 2160; p->frames = 30;
            p->n_objects = 16;
            p->obj_min = 128; p->obj_max = 512;
            p->vmax = 24;
            p->shapes = 1;
            p->bg_drift_q8[0] = 128;
            p->bg_drift_q8[1] = 64;
            p->noise_sigma_q8 = 3 * 256;
            break;
        default:
            return me_fail(ME_ERR_INVALID_ARGUMENT, "config id must be 1..5");
    }
    return ME_OK;
}

extern "C" me_status me_b200_synth(const me_synth_params* p, uint8_t* luma, uint8_t* alpha) {
    if (!luma) return me_fail(ME_ERR_INVALID_ARGUMENT, "null argument");
    mes::Plan P;
    const me_status st = mes::make_plan(p, P);
    if (st) return st;
    const int W = P.W, H = P.H, F = P.F, BW = P.BW, BH = P.BH, M = P.M, no = P.n_objects;
    const std::vector<uint8_t> bg = blurred_noise(BW, BH, P.bg_s0);
    std::vector<std::vector<uint8_t>> tex(static_cast<size_t>(no));
    for (int i = 0; i < no; ++i) tex[size_t(i)] = blurred_noise(P.objs[size_t(i)].bw, P.objs[size_t(i)].bh, P.objs[size_t(i)].tex_s0);
    const size_t plane = size_t(W) * H;
    for (int t = 0; t < F; ++t) {
        uint8_t* f = luma + plane * t;
        uint8_t* a = alpha ? alpha + plane * t : nullptr;
        for (int y = 0; y < H; ++y) {
            const int sy = std::clamp(y + M + P.oy[size_t(t)], 0, BH - 1);
            for (int x = 0; x < W; ++x) {
                const int sx = std::clamp(x + M + P.ox[size_t(t)], 0, BW - 1);
                f[size_t(y) * W + x] = bg[size_t(sy) * BW + sx];
            }
        }
        if (a) std::memset(a, 0, plane);
        for (int i = 0; i < no; ++i) {  // ascending index: later objects occlude
            const mes::PlanObject& o = P.objs[size_t(i)];
            const int px = P.px[size_t(t) * no + i], py = P.py[size_t(t) * no + i];
            for (int y = 0; y < o.bh; ++y) {
                const int fy = py + y;
                if (fy < 0 || fy >= H) continue;
                for (int x = 0; x < o.bw; ++x) {
                    const int fx = px + x;
                    if (fx < 0 || fx >= W || !mes::inside_box(o.ellipse, o.bw, o.bh, x, y)) continue;
                    f[size_t(fy) * W + fx] = tex[size_t(i)][size_t(y) * o.bw + x];
                    if (a) a[size_t(fy) * W + fx] = 255;
                }
            }
        }
        if (P.noise_sigma_q8 > 0)
            for (size_t i = 0; i < plane; ++i)
                f[i] = uint8_t(std::clamp(int(f[i]) + mes::noise_delta(P.noise_key, t, i, P.noise_sigma_q8), 0, 255));
    }
    return ME_OK;
}
