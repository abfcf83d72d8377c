// pa_common.cuh — pieces shared by the PA kernels (pa.cu: the global
// dataflow wavefront kernels; pa_seq.cu: the per-sequence CTA wavefront):
// parameters, the FP64 PRS direction, patch-row helpers.
#pragma once

#include "device.cuh"

namespace mek {

struct PaParams {
    int W, H, bs, S;
    int max_iter, step, bt_shape;
    double eps, theta;
    int bm_side, bm_words;  // PRS visited bitmap (lattice side, words per warp)
};

// Per-warp block context.
struct PaBlock {
    const uint8_t *cur, *ref, *ca, *ra;
    int x0, y0;
    Win w;
};


// The PRS probing direction (estimators.cpp:343-355) for field vector
// (cx, cy): sequential raster-order double sums of prs_update terms
// (estimators.cpp:303-309), each term computed by its own lane with
// round-to-nearest intrinsics, then accumulated in order through shuffles.
static __device__ void prs_direction(const PaParams& P, const PaBlock& B, int lane, int cx, int cy,
                              double& dir_x, double& dir_y) {
    const int dmx = -cx, dmy = -cy;
    const double pdx = 0.5 * dmx, pdy = 0.5 * dmy;
    const int npix = P.bs * P.bs;
    double sx = 0.0, sy = 0.0;
    for (int base = 0; base < npix; base += 32) {
        const int pix = base + lane;
        const int x = B.x0 + pix % P.bs, y = B.y0 + pix / P.bs;
        // dpd (metrics.cpp:86-88): cur(x,y) - halfpel(ref, 2x - d.dx, 2y - d.dy)
        const int i4 = interp4(B.ref, P.W, P.H, 2 * x - dmx, 2 * y - dmy);
        const double e = __dsub_rn(double(B.cur[size_t(y) * P.W + x]), double(i4) * 0.25);
        // grad_central (metrics.cpp:97-101) on cur, clamped
        const double gx = (double(pxc(B.cur, P.W, P.H, x + 1, y)) -
                           double(pxc(B.cur, P.W, P.H, x - 1, y))) / 2.0;
        const double gy = (double(pxc(B.cur, P.W, P.H, x, y + 1)) -
                           double(pxc(B.cur, P.W, P.H, x, y - 1))) / 2.0;
        // update_term (metrics.cpp:103-106)
        const double ux = fabs(gx) < P.theta ? 0.0 : __ddiv_rn(1.0, gx);
        const double uy = fabs(gy) < P.theta ? 0.0 : __ddiv_rn(1.0, gy);
        const double ee = __dmul_rn(P.eps, e);
        const double tx = __dsub_rn(pdx, __dmul_rn(ee, ux));
        const double ty = __dsub_rn(pdy, __dmul_rn(ee, uy));
        for (int j = 0; j < 32; ++j) {
            sx = __dadd_rn(sx, __shfl_sync(0xFFFFFFFFu, tx, j));
            sy = __dadd_rn(sy, __shfl_sync(0xFFFFFFFFu, ty, j));
        }
    }
    const double n = double(P.bs) * double(P.bs);
    dir_x = -__dsub_rn(__ddiv_rn(sx, n), pdx);
    dir_y = -__dsub_rn(__ddiv_rn(sy, n), pdy);
}


__device__ __forceinline__ int clip_comp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

constexpr int kFastPR = 16;        // patch rows (8 + 2R)


// kOff8 (estimators.cpp:33-35) arithmetically: offset k in raster order of
// (dy, dx) with the centre skipped.  Lane-dependent indices into c_off8 would
// serialise the constant cache.
__device__ __forceinline__ int off8x(int k) { const int i = k + (k >= 4); return i - 3 * (i / 3) - 1; }
__device__ __forceinline__ int off8y(int k) { const int i = k + (k >= 4); return i / 3 - 1; }

__device__ __forceinline__ void cp_async16(uint32_t* smem, const void* gmem, bool fill) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int n = fill ? 16 : 0;  // n = 0: zero-fill (patch columns outside the frame)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 2 words of a staged patch row: bytes [t, t + 8) of the row's 32 raw bytes.
__device__ __forceinline__ void prow8(const uint32_t* row, int t, uint32_t& r0, uint32_t& r1) {
    const int q = t >> 2;
    const uint32_t sh = uint32_t(t & 3) * 8;
    const uint32_t w0 = row[q], w1 = row[q + 1], w2 = row[q + 2];
    r0 = __funnelshift_r(w0, w1, sh);
    r1 = __funnelshift_r(w1, w2, sh);
}


__device__ __forceinline__ void cp_async8(uint32_t* smem, const void* gmem, bool fill) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int n = fill ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}

// Host: the PA parameters of a batch configuration.
inline PaParams make_pa_params(const Batch& b, const me_config& c) {
    PaParams P;
    P.W = b.W;
    P.H = b.H;
    P.bs = b.bs;
    P.S = c.search_range;
    P.max_iter = c.max_iterations;
    P.step = c.halfpel ? 1 : c.step;
    P.bt_shape = c.boundary_temporal == ME_BT_SHAPE;
    P.eps = c.epsilon;
    P.theta = c.theta;
    // lattice radius: max_iter steps, but never more than the window allows
    const int span = (4 * c.search_range) / P.step + 1;
    int side = 2 * c.max_iterations + 1;
    if (side > 2 * span + 1) side = 2 * span + 1;
    P.bm_side = side;
    P.bm_words = (side * side + 31) / 32;
    return P;
}

}  // namespace mek
