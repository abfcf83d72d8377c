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
// in parallel: 4 lanes per position, BS/4 rows per lane, reduced by shuffles.
// A per-warp bitmap over the clipped window counts unique evaluations
// (BlockMatcher::eval's cache, estimators.cpp:72-81); revisits are recomputed,
// not recounted.
// ---------------------------------------------------------------------------

struct RingCtx {
    const uint8_t *cur, *ref;
    int W, H, x0, y0, bs;
    int lo_x, hi_x, lo_y, hi_y;  // pel window
    uint32_t* bitmap;            // per-warp
    uint32_t count;
};

// Scores the n (<= 8) positions (cx, cy) + offs[k] * radius (pel); lanes
// 4k..4k+3 own position k and return its SAD; bit 4k of adm_mask is set for
// admissible positions.  radius 0 scores the center itself.
__device__ __forceinline__ uint32_t ring_eval(RingCtx& c, const int (*offs)[2], int n, int radius,
                                              int cx, int cy, int lane, uint32_t& adm_mask) {
    const int k = lane >> 2;
    const int dx = k < n ? cx + offs[k][0] * radius : 0;
    const int dy = k < n ? cy + offs[k][1] * radius : 0;
    const bool adm = k < n && dx >= c.lo_x && dx <= c.hi_x && dy >= c.lo_y && dy <= c.hi_y;
    uint32_t s = 0;
    if (adm)
        for (int r = (lane & 3); r < c.bs; r += 4)
            s += row_sad4(c.cur, c.ref, c.W, c.H, c.x0, c.y0 + r, c.bs, 2 * dx, 2 * dy);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    s >>= 2;
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
__device__ __forceinline__ void probe_ring(RingCtx& c, const int (*offs)[2], int n, int radius,
                                           int& cx, int& cy, uint32_t& best, int lane) {
    uint32_t adm;
    const uint32_t s = ring_eval(c, offs, n, radius, cx, cy, lane, adm);
    int bx = cx, by = cy;
    for (int i = 0; i < n; ++i) {
        const uint32_t v = __shfl_sync(0xFFFFFFFFu, s, 4 * i);
        if (((adm >> (4 * i)) & 1u) && v < best) {
            best = v;
            bx = cx + offs[i][0] * radius;
            by = cy + offs[i][1] * radius;
        }
    }
    cx = bx;
    cy = by;
}

__device__ void ring_block(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H, int x0,
                           int y0, int bs, int S, uint32_t* bitmap, int lane, int& out_dx,
                           int& out_dy, uint32_t& out_sad, uint32_t& out_cmp) {
    RingCtx c;
    c.cur = cur;
    c.ref = ref;
    c.W = W;
    c.H = H;
    c.x0 = x0;
    c.y0 = y0;
    c.bs = bs;
    c.lo_x = max(-S, -x0);
    c.hi_x = min(S, W - x0 - bs);
    c.lo_y = max(-S, -y0);
    c.hi_y = min(S, H - y0 - bs);
    c.bitmap = bitmap;
    c.count = 0;
    const int words = ((c.hi_x - c.lo_x + 1) * (c.hi_y - c.lo_y + 1) + 31) >> 5;
    for (int i = lane; i < words; i += 32) bitmap[i] = 0;
    __syncwarp();
    int cx = 0, cy = 0;
    uint32_t best;
    {
        uint32_t adm;
        const uint32_t s = ring_eval(c, c_off8, 1, 0, 0, 0, lane, adm);  // the center, once
        best = __shfl_sync(0xFFFFFFFFu, s, 0);
    }
    if (algo == ME_ALGO_TSS) {
        int step = 1;
        while (step * 2 <= S) step *= 2;
        for (; step >= 1; step /= 2) probe_ring(c, c_off8, 8, step, cx, cy, best, lane);
    } else if (algo == ME_ALGO_FSS) {
        for (int round = 0; round < 3; ++round) {
            const int px0 = cx, py0 = cy;
            probe_ring(c, c_off8, 8, 2, cx, cy, best, lane);
            if (cx == px0 && cy == py0) break;
        }
        probe_ring(c, c_off8, 8, 1, cx, cy, best, lane);
    } else {
        for (;;) {
            const int px0 = cx, py0 = cy;
            probe_ring(c, c_ldsp, 8, 1, cx, cy, best, lane);
            if (cx == px0 && cy == py0) break;
        }
        probe_ring(c, c_sdsp, 4, 1, cx, cy, best, lane);
    }
    out_dx = cx;
    out_dy = cy;
    out_sad = best;
    out_cmp = c.count;
}

struct RingArgs {
    Batch b;
    int algo, S;
    const uint2* list;
    const int* nlist;
    me_block_rec* recs;
    int bitmap_words;  // per warp
    me_pair_stats* stats;
};

__global__ void __launch_bounds__(256) ring_kernel(RingArgs a) {
    extern __shared__ uint32_t s_bits[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* bitmap = s_bits + wid * a.bitmap_words;
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
        ring_block(a.algo, cur, ref, b.W, b.H, h * b.bs, v * b.bs, b.bs, a.S, bitmap, lane, dx, dy,
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
    extern __shared__ uint32_t s_bits[];
    int dx, dy;
    uint32_t sad, cmp;
    ring_block(algo, cur, ref, W, H, x0, y0, bs, S, s_bits, threadIdx.x & 31, dx, dy, sad, cmp);
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

cudaError_t launch_ring(const Batch& b, int algo, int S, const uint2* list, const int* nlist,
                        me_block_rec* recs, me_pair_stats* stats, int num_sms, cudaStream_t st) {
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
    ra.bitmap_words = (WX * WY + 31) / 32;
    int warps = 8;
    while (warps > 1 && size_t(warps) * ra.bitmap_words * 4 > 160 * 1024) warps >>= 1;
    const size_t smem = size_t(warps) * ra.bitmap_words * 4;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)))) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring_kernel, warps * 32, smem);
    ring_kernel<<<num_sms * (occ > 0 ? occ : 1), warps * 32, smem, st>>>(ra);
    return cudaGetLastError();
}

cudaError_t launch_ring_single(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H,
                               int x0, int y0, int size, int range, int64_t* out, cudaStream_t st) {
    const int WX = std::min(2 * range + 1, W - size + 1);
    const int WY = std::min(2 * range + 1, H - size + 1);
    const size_t smem = size_t((WX * WY + 31) / 32) * 4;
    cudaError_t e = cudaFuncSetAttribute(ring_single_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e) return e;
    ring_single_kernel<<<1, 32, smem, st>>>(algo, cur, ref, W, H, x0, y0, size, range, out);
    return cudaGetLastError();
}

}  // namespace mek
