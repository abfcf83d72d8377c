// device.cuh — device helpers shared by the kernel translation units of
// libme_b200.so (integer SAD/SSE primitives, half-pel sampling, MV words,
// record stores, work-list decoding).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "stages.h"

namespace mek {

// ---------------------------------------------------------------------------
// Small device helpers
// ---------------------------------------------------------------------------

constexpr uint32_t kSentinel = 0x80008000u;  // MV word of a block not yet estimated
constexpr uint32_t kInf = 0xFFFFFFFFu;
constexpr uint32_t kBoundaryBit = 0x80000000u;

// kOff8 (estimators.cpp:33-35): {dx, dy}, raster order of (dy, dx)
static __constant__ int c_off8[8][2] = {{-1, -1}, {0, -1}, {1, -1}, {-1, 0}, {1, 0}, {-1, 1}, {0, 1}, {1, 1}};
// kLdsp / kSdsp (estimators.cpp:222-225)
static __constant__ int c_ldsp[8][2] = {{0, -2}, {-1, -1}, {1, -1}, {-2, 0}, {2, 0}, {-1, 1}, {1, 1}, {0, 2}};
static __constant__ int c_sdsp[4][2] = {{0, -1}, {-1, 0}, {1, 0}, {0, 1}};

// d = sum over the 4 byte lanes of |a - b|, plus c  (one VABSDIFF4.U8.ACC)
__device__ __forceinline__ uint32_t vad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
}

// 8 bytes at an arbitrary address (read-only data).  The third aligned word is
// loaded only when the span crosses into it, so no byte past p+7's word is read.
__device__ __forceinline__ void ld8u(const uint8_t* p, uint32_t& r0, uint32_t& r1) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = uint32_t(a & 3) * 8;
    const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1);
    const uint32_t w2 = sh ? __ldg(w + 2) : 0u;
    r0 = __funnelshift_r(w0, w1, sh);
    r1 = __funnelshift_r(w1, w2, sh);
}

__device__ __forceinline__ void ld16u(const uint8_t* p, uint32_t r[4]) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = uint32_t(a & 3) * 8;
    uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2), w3 = __ldg(w + 3);
    const uint32_t w4 = sh ? __ldg(w + 4) : 0u;
    r[0] = __funnelshift_r(w0, w1, sh);
    r[1] = __funnelshift_r(w1, w2, sh);
    r[2] = __funnelshift_r(w2, w3, sh);
    r[3] = __funnelshift_r(w3, w4, sh);
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// sample_clamped (frame.cpp:58-62)
__device__ __forceinline__ int pxc(const uint8_t* f, int W, int H, int x, int y) {
    return f[size_t(clampi(y, 0, H - 1)) * W + clampi(x, 0, W - 1)];
}

// 4 x sample_halfpel (frame.cpp:64-79): the bilinear weights are 0 or 1/2, so
// four times the sample is an exact integer.
__device__ __forceinline__ int interp4(const uint8_t* f, int W, int H, int x2, int y2) {
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    const int p00 = pxc(f, W, H, xi, yi);
    if (!fx && !fy) return 4 * p00;
    if (fx && !fy) return 2 * (p00 + pxc(f, W, H, xi + 1, yi));
    if (!fx) return 2 * (p00 + pxc(f, W, H, xi, yi + 1));
    return p00 + pxc(f, W, H, xi + 1, yi) + pxc(f, W, H, xi, yi + 1) + pxc(f, W, H, xi + 1, yi + 1);
}

// Half-pel window (estimators.cpp:41-48), half-pel units.
struct Win {
    int lo_x, hi_x, lo_y, hi_y;
};
__device__ __forceinline__ Win hp_window(int x0, int y0, int bs, int W, int H, int S) {
    Win w;
    w.lo_x = max(-2 * S, -2 * x0);
    w.hi_x = min(2 * S, 2 * (W - x0 - bs));
    w.lo_y = max(-2 * S, -2 * y0);
    w.hi_y = min(2 * S, 2 * (H - y0 - bs));
    return w;
}

// 4 x texture SAD of one block row (sad_texture, metrics.cpp:43-63).  Full-pel
// vectors whose displaced row lies inside the frame use VABSDIFF4 on unaligned
// loads; everything else goes through the exact clamped/half-pel path.
__device__ __forceinline__ uint32_t row_sad4(const uint8_t* cur, const uint8_t* ref, int W, int H,
                                             int x0, int y, int bs, int dx2, int dy2) {
    if (((dx2 | dy2) & 1) == 0) {
        const int sx = x0 + (dx2 >> 1), sy = y + (dy2 >> 1);
        if ((bs == 8 || bs == 16) && sx >= 0 && sx + bs <= W && sy >= 0 && sy < H && ((x0 | W) & 3) == 0) {
            const uint8_t* c = cur + size_t(y) * W + x0;
            const uint8_t* r = ref + size_t(sy) * W + sx;
            uint32_t acc = 0;
            if (bs == 8) {
                uint32_t r0, r1;
                ld8u(r, r0, r1);
                acc = vad4(ldg32(c), r0, acc);
                acc = vad4(ldg32(c + 4), r1, acc);
            } else {
                uint32_t rr[4];
                ld16u(r, rr);
#pragma unroll
                for (int i = 0; i < 4; ++i) acc = vad4(ldg32(c + 4 * i), rr[i], acc);
            }
            return acc * 4u;
        }
    }
    uint32_t acc = 0;
    for (int x = x0; x < x0 + bs; ++x) {
        const int d = 4 * int(cur[size_t(y) * W + x]) - interp4(ref, W, H, 2 * x + dx2, 2 * y + dy2);
        acc += uint32_t(d < 0 ? -d : d);
    }
    return acc;
}

// Mismatching alpha samples of one block row (sad_shape, metrics.cpp:65-84),
// full-pel pel displacement (fx, fy).  __vcmpne4 marks each differing byte
// with 0xFF, so popc/8 counts mismatches exactly for any byte values.
__device__ __forceinline__ uint32_t row_shape(const uint8_t* ca, const uint8_t* ra, int W, int H,
                                              int x0, int y, int bs, int fx, int fy) {
    const int sx = x0 + fx, sy = y + fy;
    if ((bs == 8 || bs == 16) && sx >= 0 && sx + bs <= W && sy >= 0 && sy < H && ((x0 | W) & 3) == 0) {
        const uint8_t* c = ca + size_t(y) * W + x0;
        const uint8_t* r = ra + size_t(sy) * W + sx;
        uint32_t bits = 0;
        if (bs == 8) {
            uint32_t r0, r1;
            ld8u(r, r0, r1);
            bits = __popc(__vcmpne4(ldg32(c), r0)) + __popc(__vcmpne4(ldg32(c + 4), r1));
        } else {
            uint32_t rr[4];
            ld16u(r, rr);
#pragma unroll
            for (int i = 0; i < 4; ++i) bits += __popc(__vcmpne4(ldg32(c + 4 * i), rr[i]));
        }
        return bits >> 3;
    }
    uint32_t m = 0;
    const int ry = clampi(sy, 0, H - 1);
    for (int x = x0; x < x0 + bs; ++x)
        m += ca[size_t(y) * W + x] != ra[size_t(ry) * W + clampi(x + fx, 0, W - 1)];
    return m;
}

// 8 mask bits of row y of a bit-packed plane (`wb` bytes per row) from pel x
// on (bit 0 = pel x); pels x .. x+7 lie inside the row.
__device__ __forceinline__ uint32_t mask_bits8(const uint8_t* bits, uint32_t wb, int x, int y) {
    const uint8_t* r = bits + size_t(y) * wb + (x >> 3);
    const uint32_t sh = uint32_t(x & 7);
    const uint32_t lo = __ldg(r), hi = sh ? __ldg(r + 1) : 0u;
    return ((lo | (hi << 8)) >> sh) & 0xFFu;
}

// 4 mask bits -> 4 bytes 0x00 / 0xFF (bit i -> byte i)
__device__ __forceinline__ uint32_t mask_expand4(uint32_t nib) {
    return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// Rounds 4*s/4 to nearest, ties to even (std::nearbyint, compensation.cpp:64).
__device__ __forceinline__ int round_q4(int i4) {
    const int q = i4 >> 2, rem = i4 & 3;
    if (rem < 2) return q;
    if (rem > 2) return q + 1;
    return q + (q & 1);
}

// Sum of squared differences of 4 byte lanes (IDP4A on the packed |a-b|).
__device__ __forceinline__ uint32_t sq4(uint32_t a, uint32_t b, uint32_t acc) {
    const uint32_t d = __vabsdiffu4(a, b);
    return __dp4a(d, d, acc);
}

// Squared error of one block row of cur against its motion-compensated
// prediction (predict_frame, compensation.cpp:42-66): clamped full-pel copy or
// half-pel bilinear rounded half to even.
static __device__ uint32_t row_sse(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y,
                            int bs, int dx2, int dy2) {
    uint32_t s = 0;
    for (int x = x0; x < x0 + bs; ++x) {
        const int p = ((dx2 | dy2) & 1) == 0 ? pxc(ref, W, H, x + (dx2 >> 1), y + (dy2 >> 1))
                                             : round_q4(interp4(ref, W, H, 2 * x + dx2, 2 * y + dy2));
        const int d = int(cur[size_t(y) * W + x]) - p;
        s += uint32_t(d * d);
    }
    return s;
}

// Same for a full-pel vector (pels) whose displaced row lies inside the frame
// and a word-aligned current row.
__device__ __forceinline__ uint32_t row_sse_fp(const uint8_t* cur, const uint8_t* ref, int W, int x0,
                                               int y, int bs, int dx, int dy) {
    const uint8_t* c = cur + size_t(y) * W + x0;
    const uint8_t* r = ref + size_t(y + dy) * W + x0 + dx;
    uint32_t s = 0;
    if (bs == 8) {
        uint32_t r0, r1;
        ld8u(r, r0, r1);
        s = sq4(ldg32(c), r0, s);
        s = sq4(ldg32(c + 4), r1, s);
    } else {
        uint32_t rr[4];
        ld16u(r, rr);
#pragma unroll
        for (int i = 0; i < 4; ++i) s = sq4(ldg32(c + 4 * i), rr[i], s);
    }
    return s;
}

// Per-pair SearchStats + SSE accumulation (me_pair_stats field order).
__device__ __forceinline__ void add_stats(me_pair_stats* st, uint32_t sse, uint32_t cmp,
                                          uint32_t dpd, int type) {
    unsigned long long* s = reinterpret_cast<unsigned long long*>(st);
    if (sse) atomicAdd(s + 5, static_cast<unsigned long long>(sse));
    if (cmp) atomicAdd(s + 0, static_cast<unsigned long long>(cmp));
    if (dpd) atomicAdd(s + 1, static_cast<unsigned long long>(dpd));
    atomicAdd(s + (type == ME_OPAQUE ? 2 : (type == ME_BOUNDARY ? 3 : 4)), 1ull);
}

// PA blocks: the type counts and the 4 comparisons per block are added by
// classify_kernel; the search adds only the SSE and the dpd count, as
// fire-and-forget reductions.
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void add_stats_pa(me_pair_stats* st, uint32_t sse, uint32_t dpd) {
    unsigned long long* s = reinterpret_cast<unsigned long long*>(st);
    if (sse) red_add_u64(s + 5, sse);
    red_add_u64(s + 1, dpd);
}

// The MV word is the whole payload a dependent block needs, and it is a single
// 32-bit word: relaxed gpu-scope accesses suffice (no acquire fence, which
// would invalidate the SM's L1 on every poll).
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t pack_mv(int dx, int dy) {
    return (uint32_t(uint16_t(int16_t(dx)))) | (uint32_t(uint16_t(int16_t(dy))) << 16);
}
__device__ __forceinline__ int mv_dx(uint32_t w) { return int(int16_t(uint16_t(w & 0xFFFF))); }
__device__ __forceinline__ int mv_dy(uint32_t w) { return int(int16_t(uint16_t(w >> 16))); }

__device__ __forceinline__ void write_rec(me_block_rec* r, int dx, int dy, uint32_t cost_q4,
                                          uint32_t cmp, uint32_t dpd, uint32_t iters,
                                          uint32_t type, bool release) {
    uint32_t* w = reinterpret_cast<uint32_t*>(r);
    w[1] = cost_q4;
    w[2] = min(cmp, 0xFFFFu) | (dpd << 16);  // comparisons saturate (ES at S >= 128: (2S+1)^2 > 65535)
    w[3] = (iters & 0xFF) | ((type & 0xFF) << 8);
    if (release)
        st_relaxed(w, pack_mv(dx, dy));
    else
        w[0] = pack_mv(dx, dy);
}

// The whole record in one 16-byte store; its 32-bit MV word (element 0) is
// single-copy atomic, which is all a dependent block reads.
__device__ __forceinline__ void write_rec_v4(me_block_rec* r, int dx, int dy, uint32_t cost_q4,
                                             uint32_t cmp, uint32_t dpd, uint32_t iters, uint32_t type) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(r), "r"(pack_mv(dx, dy)),
                 "r"(cost_q4), "r"((cmp & 0xFFFF) | (dpd << 16)), "r"((iters & 0xFF) | ((type & 0xFF) << 8))
                 : "memory");
}

// Unpacks a work-list entry; returns the global block index g.
__device__ __forceinline__ uint32_t decode_entry(const Batch& b, uint2 e, int& h, int& v, int& p,
                                                 int& seq, bool& boundary) {
    h = int(e.x & 0xFFFF);
    v = int((e.x >> 16) & 0x7FFF);
    boundary = (e.x & kBoundaryBit) != 0;
    p = int(e.y & 0xFFFF);
    seq = int(e.y >> 16);
    return ((uint32_t(seq) * b.pairs + p) * b.rows + v) * b.cols + h;
}

// classify_block (frame.cpp:81-104) of one block of an alpha plane
__device__ __forceinline__ int classify_one(const uint8_t* a, int W, int x0, int y0, int bs) {
    if (!a) return ME_OPAQUE;
    uint32_t any = 0, nz = 1;
    for (int y = 0; y < bs; ++y) {
        const uint8_t* row = a + size_t(y0 + y) * W + x0;
        for (int i = 0; i < bs; i += 8) {
            const uint2 w = *reinterpret_cast<const uint2*>(row + i);
            any |= w.x | w.y;
            nz &= (__vcmpeq4(w.x, 0u) | __vcmpeq4(w.y, 0u)) == 0u;
        }
    }
    return !any ? ME_TRANSPARENT : (nz ? ME_OPAQUE : ME_BOUNDARY);
}

}  // namespace mek
