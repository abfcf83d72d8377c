// synth.h — the scalar plan of a synthetic sequence (csrc/synth.cpp): every
// random draw that is not a pixel (global offsets, object boxes, velocities,
// positions) resolved on the host, and the SplitMix64 counters at which the
// pixel draws (background and object textures) start.  Both renderers — the
// host one (me_b200_synth) and the device one (me_b200_synth_dev) — consume
// the same plan, so they produce identical bytes.  Not installed.
#pragma once

#include <cstdint>
#include <vector>

#include "me_b200.h"

namespace mes {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr int kMaxObjects = 64;
#ifdef __CUDACC__
#define MES_HD __host__ __device__
#else
#define MES_HD
#endif

// sigma = 1.5, radius 4: round(4096 * g_k / sum g), centre adjusted to sum 4096.
MES_HD constexpr int blur_tap(int k) { return k == 0 ? 1092 : k == 1 ? 874 : k == 2 ? 449 : k == 3 ? 148 : 31; }

MES_HD inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Byte i of a blurred-noise image whose SplitMix64 stream starts at `s0`
// (before blurring): draw j = i / 8 is mix64(s0 + (j + 1) * golden).
MES_HD inline uint8_t noise_byte(uint64_t s0, uint64_t i) {
    return uint8_t(mix64(s0 + (i / 8 + 1) * kGolden) >> (8 * (i % 8)));
}

// Additive noise of pixel i of frame t (Irwin-Hall of 12 16-bit draws scaled
// to sigma, rounded half to even).
MES_HD inline int noise_delta(uint64_t key, int t, uint64_t i, int64_t sigma_q8) {
    const uint64_t base = key ^ (uint64_t(t) << 40) ^ (i * 3);
    int64_t s = 0;
    for (int k = 0; k < 3; ++k) {
        const uint64_t r = mix64(base + uint64_t(k) * kGolden);
        s += int64_t(r & 0xFFFF) + int64_t((r >> 16) & 0xFFFF) + int64_t((r >> 32) & 0xFFFF) + int64_t(r >> 48);
    }
    s -= 6 * 65535;
    const int64_t num = s * sigma_q8;
    const int64_t den = int64_t(1) << 24;
    int64_t q = num >= 0 ? num / den : -((-num) / den);
    const int64_t r = num - q * den;
    const int64_t ar = r < 0 ? -r : r;
    if (2 * ar > den || (2 * ar == den && (q & 1))) q += num >= 0 ? 1 : -1;
    return int(q);
}

// Ellipse (or full box) membership of box pixel (x, y).
MES_HD inline bool inside_box(bool ellipse, int bw, int bh, int x, int y) {
    if (!ellipse) return true;
    const int64_t a2 = int64_t(bw) * bw, b2 = int64_t(bh) * bh;
    const int64_t ex = 2 * x + 1 - bw, ey = 2 * y + 1 - bh;
    return ex * ex * b2 + ey * ey * a2 <= a2 * b2;
}

struct PlanObject {
    int bw, bh, ellipse, vx, vy, x0, y0;
    uint64_t tex_s0;  // SplitMix state before the texture draws
};

struct Plan {
    int W, H, F, M, BW, BH, n_objects;
    int64_t noise_sigma_q8;
    uint64_t bg_s0, noise_key;
    std::vector<int> ox, oy;          // global offset per frame
    std::vector<PlanObject> objs;
    std::vector<int> px, py;          // [F][n_objects] box positions (bounce)
};

// Validates p and resolves the plan (me_b200_synth's error messages).
me_status make_plan(const me_synth_params* p, Plan& out);

}  // namespace mes
