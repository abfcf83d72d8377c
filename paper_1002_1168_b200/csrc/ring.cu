// ring.cu — tss_search / fss_search / ds_search (estimators.cpp:189-236): the
// batched kernel over the work list and the single-block kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "device.cuh"

namespace mek {

// ---------------------------------------------------------------------------
// ring_kernel: tss_search / fss_search / ds_search (estimators.cpp:189-236).
// One warp per block.  Each ring's (up to 8) admissible positions are scored
// in parallel: 4 lanes per position, BS/4 rows per lane (rows rg, rg+4, ..),
// reduced by shuffles.  A lane's current-block rows are loaded once per block
// into registers; a displaced reference row (integer-pel: always inside the
// frame, the window clips it) arrives as aligned 16-byte (BS 16) or 8-byte
// (BS 8) loads funnel-shifted into place — every load instruction of the warp
// touches 32 rows, so the instruction count per row sets the L1 cost.
// A per-warp bitmap over the clipped window counts unique evaluations
// (BlockMatcher::eval's cache, estimators.cpp:72-81); revisits are recomputed,
// not recounted.
// ---------------------------------------------------------------------------

struct RingCtx {
    const uint8_t *cur, *ref;
    int W, H, x0, y0;
    int lo_x, hi_x, lo_y, hi_y;  // pel window
    uint32_t* bitmap;            // per-warp
    uint32_t* stage;             // per-warp kStageWords, 16-byte aligned
    uint32_t count;
    int scx, scy;                // centre (pel offsets) of the staged region; scx > 2^20: nothing staged
};

// BS bytes at an arbitrary address as BS/4 words, from aligned loads (two
// 16-byte loads for BS 16, two 8-byte loads for BS 8; the second is skipped
// when the address is aligned and never leaves the aligned chunk holding the
// row's last byte).
template <int BS>
__device__ __forceinline__ void ld_row_aligned(const uint8_t* p, uint32_t (&r)[BS / 4]) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t s = uint32_t(a & (BS - 1)), q = s >> 2, sh = (s & 3) * 8;
    if (BS == 16) {
        const uint4* b = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
        const uint4 lo = __ldg(b);
        const uint4 hi = s ? __ldg(b + 1) : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        uint32_t u[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) u[i] = q == 0 ? w[i] : q == 1 ? w[i + 1] : q == 2 ? w[i + 2] : w[i + 3];
#pragma unroll
        for (int i = 0; i < BS / 4; ++i) r[i] = __funnelshift_r(u[i], u[i + 1], sh);
    } else {
        const uint2* b = reinterpret_cast<const uint2*>(a & ~uintptr_t(7));
        const uint2 lo = __ldg(b);
        const uint2 hi = s ? __ldg(b + 1) : make_uint2(0u, 0u);
        const uint32_t u0 = q ? lo.y : lo.x, u1 = q ? hi.x : lo.y, u2 = q ? hi.y : hi.x;
        r[0] = __funnelshift_r(u0, u1, sh);
        r[BS / 4 - 1] = __funnelshift_r(u1, u2, sh);
    }
}

// Small rings (extent <= kStageR: TSS's last steps, every FSS / DS ring) are
// served from a per-warp shared-memory copy of the region within kStageR pels
// of a centre: (BS + 2 kStageR) rows of 16-byte chunks from the aligned
// address at or left of the region, fetched by the whole warp (each load
// instruction covers a few rows instead of 32).  The copy stays valid while
// the later rings fit in it (FSS's rounds, DS's steps and TSS's last three
// rings mostly restage never or once), then every position's rows are read
// from shared memory.
constexpr int kStageR = 8;
constexpr int kStageRowWords = 12;                                     // 48 bytes: 3 chunks (BS + 2 kStageR <= 33)
constexpr int kStageWords = (16 + 2 * kStageR) * kStageRowWords;       // 384 words per warp

// Scores the n (<= 8) positions (cx, cy) + offs[k] * radius (pel); lanes
// 4k..4k+3 own position k and return its SAD; bit 4k of adm_mask is set for
// admissible positions.  radius 0 scores the center itself.
template <int BS>
__device__ __forceinline__ uint32_t ring_eval(RingCtx& c, const uint32_t (&cw)[BS / 4][BS / 4],
                                              const int (*offs)[2], int n, int radius, int reach, int cx,
                                              int cy, int lane, uint32_t& adm_mask) {
    const int k = lane >> 2;
    const int e = reach * radius;  // the ring's extent: max |offset| x radius
    const int dx = k < n ? cx + offs[k][0] * radius : 0;
    const int dy = k < n ? cy + offs[k][1] * radius : 0;
    const bool adm = k < n && dx >= c.lo_x && dx <= c.hi_x && dy >= c.lo_y && dy <= c.hi_y;
    uint32_t s = 0;
    if (e >= 1 && e <= kStageR) {  // warp-uniform
        constexpr int E = kStageR, NCH = (BS + 2 * E + 15 + 15) / 16;
        const uintptr_t base = reinterpret_cast<uintptr_t>(c.ref);
        if (abs(cx - c.scx) + e > E || abs(cy - c.scy) + e > E) {  // the ring leaves the staged region: restage
            c.scx = cx;
            c.scy = cy;
            const int R = BS + 2 * E, rx = c.x0 + cx - E, ry = c.y0 + cy - E;
            __syncwarp();  // every lane is done reading the previous copy
            for (int it = lane; it < R * NCH; it += 32) {
                const int row = it / NCH, ch = it - NCH * row;
                const int y = ry + row;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (y >= 0 && y < c.H) {
                    const uintptr_t rowa = base + size_t(y) * c.W;
                    const uintptr_t cb = ((rowa + uintptr_t(intptr_t(rx))) & ~uintptr_t(15)) + 16u * ch;
                    // only chunks holding a byte of this row (never outside the plane)
                    if (cb + 16 > rowa && cb < rowa + c.W) v = __ldg(reinterpret_cast<const uint4*>(cb));
                }
                *reinterpret_cast<uint4*>(c.stage + row * kStageRowWords + 4 * ch) = v;
            }
            __syncwarp();
        }
        const int rx = c.x0 + c.scx - E, ry = c.y0 + c.scy - E;
        if (adm) {
            // byte offset of staged row `row`'s first chunk: the region's start
            // misalignment, advancing by W mod 16 per row (32-bit math per row)
            const uint32_t a0 = uint32_t((base + size_t(ry) * c.W + uintptr_t(intptr_t(rx))) & 15u), wm = uint32_t(c.W) & 15u;
#pragma unroll
            for (int j = 0; j < BS / 4; ++j) {
                const int row = dy - c.scy + E + (lane & 3) + 4 * j;
                const uint32_t o = ((a0 + uint32_t(row) * wm) & 15u) + uint32_t(dx - c.scx + E);
                const uint32_t* w = c.stage + row * kStageRowWords + (o >> 2);
                const uint32_t sh = (o & 3u) * 8u;
                uint32_t u[BS / 4 + 1];
#pragma unroll
                for (int i = 0; i <= BS / 4; ++i) u[i] = w[i];
#pragma unroll
                for (int i = 0; i < BS / 4; ++i) s = vad4(cw[j][i], __funnelshift_r(u[i], u[i + 1], sh), s);
            }
        }
    } else if (adm) {
        const uint8_t* rp = c.ref + size_t(c.y0 + dy + (lane & 3)) * c.W + (c.x0 + dx);
#pragma unroll
        for (int j = 0; j < BS / 4; ++j) {
            uint32_t rr[BS / 4];
            ld_row_aligned<BS>(rp + size_t(4 * j) * c.W, rr);
#pragma unroll
            for (int i = 0; i < BS / 4; ++i) s = vad4(cw[j][i], rr[i], s);
        }
    }
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    // unique-evaluation counting
    const int WX = c.hi_x - c.lo_x + 1;
    bool fresh = false;
    if (adm && (lane & 3) == 0) {
        const int bit = (dy - c.lo_y) * WX + (dx - c.lo_x);
        const uint32_t m = 1u << (bit & 31);
        fresh = (atomicOr(&c.bitmap[bit >> 5], m) & m) == 0;
    }
    c.count += __popc(__ballot_sync(0xFFFFFFFFu, fresh));
    adm_mask = __ballot_sync(0xFFFFFFFFu, adm && (lane & 3) == 0);
    return s;
}

// probe_ring (estimators.cpp:85-102): strict improvement in listed order.
template <int BS>
__device__ __forceinline__ void probe_ring(RingCtx& c, const uint32_t (&cw)[BS / 4][BS / 4],
                                           const int (*offs)[2], int n, int radius, int reach, int& cx,
                                           int& cy, uint32_t& best, int lane) {
    uint32_t adm;
    const uint32_t s = ring_eval<BS>(c, cw, offs, n, radius, reach, cx, cy, lane, adm);
    // sequential strict improvement in listed order = the first admissible
    // position holding the ring's minimum, taken if below the centre's cost:
    // one warp reduction of (SAD << 3 | k) (SAD < 2^17)
    const int k = lane >> 2;
    const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, ((adm >> (4 * k)) & 1u) ? (s << 3) | uint32_t(k) : ~0u);
    if (m != ~0u && (m >> 3) < best) {
        best = m >> 3;
        cx += offs[m & 7][0] * radius;
        cy += offs[m & 7][1] * radius;
    }
}

template <int BS>
__device__ void ring_block(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H, int x0,
                           int y0, int S, uint32_t* bitmap, int lane, int& out_dx, int& out_dy,
                           uint32_t& out_sad, uint32_t& out_cmp) {
    RingCtx c;
    c.cur = cur;
    c.ref = ref;
    c.W = W;
    c.H = H;
    c.x0 = x0;
    c.y0 = y0;
    c.lo_x = max(-S, -x0);
    c.hi_x = min(S, W - x0 - BS);
    c.lo_y = max(-S, -y0);
    c.hi_y = min(S, H - y0 - BS);
    c.bitmap = bitmap;
    c.stage = bitmap + ((((c.hi_x - c.lo_x + 1) * (c.hi_y - c.lo_y + 1) + 31) >> 5) + 3 & ~3);
    c.count = 0;
    c.scx = c.scy = 1 << 21;  // nothing staged yet
    // the lane's current-block rows (lane & 3) + 4 j, once per block
    uint32_t cw[BS / 4][BS / 4];
#pragma unroll
    for (int j = 0; j < BS / 4; ++j) {
        const uint8_t* cp = cur + size_t(y0 + (lane & 3) + 4 * j) * W + x0;
        if (BS == 16)
            ld16u(cp, cw[j]);
        else
            ld8u(cp, cw[j][0], cw[j][BS / 4 - 1]);
    }
    const int words = ((c.hi_x - c.lo_x + 1) * (c.hi_y - c.lo_y + 1) + 31) >> 5;
    for (int i = lane; i < words; i += 32) bitmap[i] = 0;
    __syncwarp();
    int cx = 0, cy = 0;
    uint32_t best;
    {
        uint32_t adm;
        const uint32_t s = ring_eval<BS>(c, cw, c_off8, 1, 0, 1, 0, 0, lane, adm);  // the center, once
        best = __shfl_sync(0xFFFFFFFFu, s, 0);
    }
    if (algo == ME_ALGO_TSS) {
        int step = 1;
        while (step * 2 <= S) step *= 2;
        for (; step >= 1; step /= 2) probe_ring<BS>(c, cw, c_off8, 8, step, 1, cx, cy, best, lane);
    } else if (algo == ME_ALGO_FSS) {
        for (int round = 0; round < 3; ++round) {
            const int px0 = cx, py0 = cy;
            probe_ring<BS>(c, cw, c_off8, 8, 2, 1, cx, cy, best, lane);
            if (cx == px0 && cy == py0) break;
        }
        probe_ring<BS>(c, cw, c_off8, 8, 1, 1, cx, cy, best, lane);
    } else {
        for (;;) {
            const int px0 = cx, py0 = cy;
            probe_ring<BS>(c, cw, c_ldsp, 8, 1, 2, cx, cy, best, lane);  // kLdsp reaches 2
            if (cx == px0 && cy == py0) break;
        }
        probe_ring<BS>(c, cw, c_sdsp, 4, 1, 1, cx, cy, best, lane);
    }
    out_dx = cx;
    out_dy = cy;
    out_sad = best;
    out_cmp = c.count;
}

__device__ __forceinline__ void ring_block_bs(int bs, int algo, const uint8_t* cur, const uint8_t* ref, int W,
                                              int H, int x0, int y0, int S, uint32_t* bitmap, int lane,
                                              int& out_dx, int& out_dy, uint32_t& out_sad, uint32_t& out_cmp) {
    if (bs == 16)
        ring_block<16>(algo, cur, ref, W, H, x0, y0, S, bitmap, lane, out_dx, out_dy, out_sad, out_cmp);
    else
        ring_block<8>(algo, cur, ref, W, H, x0, y0, S, bitmap, lane, out_dx, out_dy, out_sad, out_cmp);
}

struct RingArgs {
    Batch b;
    int algo, S;
    const uint2* list;
    const int* nlist;
    me_block_rec* recs;
    int warp_words;  // per warp: the unique-evaluation bitmap + the ring staging buffer
    me_pair_stats* stats;
};

template <int MINB>
__global__ void __launch_bounds__(256, MINB) ring_kernel(RingArgs a) {
    extern __shared__ __align__(16) uint32_t s_bits[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* bitmap = s_bits + wid * a.warp_words;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int n = *a.nlist;
    const Batch& b = a.b;
    const size_t plane = size_t(b.W) * b.H;
    for (int item = blockIdx.x * (blockDim.x >> 5) + wid; item < n; item += nwarps) {
        int h, v, p, seq;
        bool boundary;
        const uint32_t g = decode_entry(b, a.list[item], h, v, p, seq, boundary);
        const uint8_t* cur = b.luma + (size_t(seq) * b.F + p + b.d) * plane;
        const uint8_t* ref = b.luma + (size_t(seq) * b.F + p) * plane;
        int dx, dy;
        uint32_t sad, cmp;
        ring_block_bs(b.bs, a.algo, cur, ref, b.W, b.H, h * b.bs, v * b.bs, a.S, bitmap, lane, dx, dy,
                      sad, cmp);
        uint32_t sse = lane < b.bs ? row_sse_fp(cur, ref, b.W, h * b.bs, v * b.bs + lane, b.bs, dx, dy) : 0u;
        sse = __reduce_add_sync(0xFFFFFFFFu, sse);
        if (lane == 0) {
            const int ty = boundary ? ME_BOUNDARY : ME_OPAQUE;
            write_rec(a.recs + g, 2 * dx, 2 * dy, sad * 4u, cmp, 0, 0, ty, false);
            if (a.stats) add_stats(a.stats + (size_t(seq) * b.pairs + p), sse, cmp, 0, ty);
        }
        __syncwarp();
    }
}

__global__ void ring_single_kernel(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H,
                                   int x0, int y0, int bs, int S, int64_t* out) {
    extern __shared__ __align__(16) uint32_t s_bits[];
    int dx, dy;
    uint32_t sad, cmp;
    ring_block_bs(bs, algo, cur, ref, W, H, x0, y0, S, s_bits, int(threadIdx.x & 31), dx, dy, sad, cmp);
    if (threadIdx.x == 0) {
        out[0] = 2 * dx;
        out[1] = 2 * dy;
        out[2] = cmp;
        out[3] = int64_t(sad) * 4;
    }
}

// out: [0..1] mv, [2..5] scores_q4, [6..9] kinds

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------

// Per-warp shared words: the bitmap over the largest clipped window (rounded
// to 16 bytes; ring_block places the staging buffer after its own window's
// bitmap, which is never larger) + the staging buffer.
static int ring_warp_words(int WX, int WY) { return (((WX * WY + 31) / 32 + 3) & ~3) + kStageWords; }

cudaError_t launch_ring(const Batch& b, int algo, int S, const uint2* list, const int* nlist,
                        me_block_rec* recs, me_pair_stats* stats, int num_sms, cudaStream_t st, int ctas) {
    RingArgs ra;
    ra.b = b;
    ra.algo = algo;
    ra.S = S;
    ra.list = list;
    ra.nlist = nlist;
    ra.recs = recs;
    ra.stats = stats;
    const int WX = std::min(2 * S + 1, b.W - b.bs + 1);
    const int WY = std::min(2 * S + 1, b.H - b.bs + 1);
    ra.warp_words = ring_warp_words(WX, WY);
    int warps = 8;
    while (warps > 1 && size_t(warps) * ra.warp_words * 4 > 160 * 1024) warps >>= 1;
    const size_t smem = size_t(warps) * ra.warp_words * 4;
    cudaError_t e;
    // register budget: 4 CTAs per SM (64 registers) or 3 (80, no spills)
    void (*kern)(RingArgs) = ctas == 4 ? ring_kernel<4> : ctas == 2 ? ring_kernel<2> : ring_kernel<3>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)))) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
    kern<<<num_sms * (occ > 0 ? occ : 1), warps * 32, smem, st>>>(ra);
    return cudaGetLastError();
}

cudaError_t launch_ring_single(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H,
                               int x0, int y0, int size, int range, int64_t* out, cudaStream_t st) {
    const int WX = std::min(2 * range + 1, W - size + 1);
    const int WY = std::min(2 * range + 1, H - size + 1);
    const size_t smem = size_t(ring_warp_words(WX, WY)) * 4;
    cudaError_t e = cudaFuncSetAttribute(ring_single_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e) return e;
    ring_single_kernel<<<1, 32, smem, st>>>(algo, cur, ref, W, H, x0, y0, size, range, out);
    return cudaGetLastError();
}

}  // namespace mek
