// frame_ops.cu — frame-level kernels: predict_frame + psnr SSE (mc_kernel),
// the bit-packed mask expansion of the host path, and the single-plane entry
// points (sad_texture / sad_shape / classify / binarize / sse).
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
// unpack_kernel: the host path ships binary alpha masks bit-packed (1/8 of the
// PCIe bytes) and expands them here: one thread per 4 packed bytes -> 32 pixels.
// ---------------------------------------------------------------------------
__global__ void unpack_kernel(const uint32_t* __restrict__ bits, uint4* __restrict__ out, size_t nwords) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = __ldg(bits + i);
        uint4 v[2];
        uint32_t* o = reinterpret_cast<uint32_t*>(v);
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // 4 pixels per output word: bits 4q .. 4q+3
            const uint32_t nib = (w >> (4 * q)) & 0xFu;
            o[q] = ((nib & 1u) ? 0xFFu : 0u) | ((nib & 2u) ? 0xFF00u : 0u) | ((nib & 4u) ? 0xFF0000u : 0u) |
                   ((nib & 8u) ? 0xFF000000u : 0u);
        }
        out[2 * i] = v[0];
        out[2 * i + 1] = v[1];
    }
}

// unpack_sparse_kernel: the same masks with the all-zero 64-pixel words elided
// (object masks are mostly background): per group of 32 words a presence mask
// and the group's first literal; one warp per group, one lane per word.
__global__ void unpack_sparse_kernel(const uint32_t* __restrict__ pres, const uint32_t* __restrict__ base,
                                     const unsigned long long* __restrict__ lit, uint4* __restrict__ out,
                                     size_t nwords) {
    const int lane = threadIdx.x & 31;
    const size_t ngroups = (nwords + 31) / 32;
    for (size_t gi = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; gi < ngroups;
         gi += (size_t(gridDim.x) * blockDim.x) >> 5) {
        const size_t w = gi * 32 + lane;
        if (w >= nwords) continue;
        const uint32_t m = __ldg(pres + gi);
        unsigned long long x = 0;
        if ((m >> lane) & 1u) x = __ldg(lit + __ldg(base + gi) + __popc(m & ((1u << lane) - 1u)));
        uint4 v[4];
        uint32_t* o = reinterpret_cast<uint32_t*>(v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {  // 4 pixels per output word
            const uint32_t nib = uint32_t(x >> (4 * q)) & 0xFu;
            o[q] = ((nib & 1u) ? 0xFFu : 0u) | ((nib & 2u) ? 0xFF00u : 0u) | ((nib & 4u) ? 0xFF0000u : 0u) |
                   ((nib & 8u) ? 0xFF000000u : 0u);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) out[4 * w + q] = v[q];
    }
}

// The same sparse form expanded to the dense bit plane (one 64-bit word per 64
// pixels): the layout the classify and PA kernels read directly.
__global__ void unpack_sparse_bits_kernel(const uint32_t* __restrict__ pres, const uint32_t* __restrict__ base,
                                          const unsigned long long* __restrict__ lit, unsigned long long* __restrict__ out,
                                          size_t nwords) {
    const int lane = threadIdx.x & 31;
    const size_t ngroups = (nwords + 31) / 32;
    for (size_t gi = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; gi < ngroups;
         gi += (size_t(gridDim.x) * blockDim.x) >> 5) {
        const size_t w = gi * 32 + lane;
        if (w >= nwords) continue;
        const uint32_t m = __ldg(pres + gi);
        unsigned long long x = 0;
        if ((m >> lane) & 1u) x = __ldg(lit + __ldg(base + gi) + __popc(m & ((1u << lane) - 1u)));
        out[w] = x;
    }
}

// ---------------------------------------------------------------------------
// mc_kernel: predict_frame (compensation.cpp:30-71) fused with the psnr SSE
// (metrics.cpp:108-124) and the per-pair SearchStats reduction.  One thread
// per 8-pixel row segment; the prediction is only stored when requested.
// ---------------------------------------------------------------------------

struct McArgs {
    Batch b;
    const me_block_rec* recs;
    me_pair_stats* stats;
    uint8_t* pred;  // [n_seq*pairs][H][W] or null
    const int32_t* mv_override;  // single-frame predict: [rows*cols][2] (recs ignored)
    const uint8_t* types_override;
    const uint8_t* ref_override;
    const uint8_t* cur_override;
};

__global__ void __launch_bounds__(256) mc_kernel(McArgs a) {
    const Batch& b = a.b;
    const int gp = blockIdx.y;  // seq * pairs + p
    const int seq = gp / b.pairs, p = gp % b.pairs;
    const size_t plane = size_t(b.W) * b.H;
    const int segs = b.W >> 3;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t sse = 0;
    uint32_t cmp = 0, dpd = 0, n_o = 0, n_b = 0, n_t = 0;
    if (idx < segs * b.H) {
        const int y = idx / segs, x = (idx - y * segs) * 8;
        const int h = x / b.bs, v = y / b.bs;
        const size_t bi = size_t(gp) * b.rows * b.cols + size_t(v) * b.cols + h;
        int dx2, dy2, ty;
        if (a.mv_override) {
            const int i = v * b.cols + h;
            dx2 = a.mv_override[2 * i];
            dy2 = a.mv_override[2 * i + 1];
            ty = a.types_override ? a.types_override[i] : ME_OPAQUE;
        } else {
            const uint4 r = *reinterpret_cast<const uint4*>(a.recs + bi);
            dx2 = mv_dx(r.x);
            dy2 = mv_dy(r.x);
            ty = int((r.w >> 8) & 0xFF);
            if (x % b.bs == 0 && y % b.bs == 0) {
                cmp = r.z & 0xFFFF;
                dpd = r.z >> 16;
                n_o = ty == ME_OPAQUE;
                n_b = ty == ME_BOUNDARY;
                n_t = ty == ME_TRANSPARENT;
            }
        }
        if (ty == ME_TRANSPARENT) dx2 = dy2 = 0;
        const uint8_t* ref = a.ref_override ? a.ref_override : b.luma + (size_t(seq) * b.F + p) * plane;
        const uint8_t* cur = a.cur_override ? a.cur_override
                                            : b.luma + (size_t(seq) * b.F + p + b.d) * plane;
        uint32_t pw0, pw1;
        const int sx = x + (dx2 >> 1), sy = y + (dy2 >> 1);
        if (((dx2 | dy2) & 1) == 0 && sx >= 0 && sx + 8 <= b.W && sy >= 0 && sy < b.H) {
            ld8u(ref + size_t(sy) * b.W + sx, pw0, pw1);
        } else {
            uint32_t w[2] = {0u, 0u};
            for (int i = 0; i < 8; ++i) {
                const int xx = x + i;
                const int val = ((dx2 | dy2) & 1) == 0
                                    ? pxc(ref, b.W, b.H, xx + (dx2 >> 1), y + (dy2 >> 1))
                                    : round_q4(interp4(ref, b.W, b.H, 2 * xx + dx2, 2 * y + dy2));
                w[i >> 2] |= uint32_t(clampi(val, 0, 255)) << (8 * (i & 3));
            }
            pw0 = w[0];
            pw1 = w[1];
        }
        if (cur) {
            const uint32_t c0 = ldg32(cur + size_t(y) * b.W + x), c1 = ldg32(cur + size_t(y) * b.W + x + 4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int d0 = int((c0 >> (8 * i)) & 0xFF) - int((pw0 >> (8 * i)) & 0xFF);
                const int d1 = int((c1 >> (8 * i)) & 0xFF) - int((pw1 >> (8 * i)) & 0xFF);
                sse += uint32_t(d0 * d0 + d1 * d1);
            }
        }
        if (a.pred) {
            uint2* dst = reinterpret_cast<uint2*>(a.pred + size_t(gp) * plane + size_t(y) * b.W + x);
            *dst = make_uint2(pw0, pw1);
        }
    }
    // CTA reduction
    __shared__ uint32_t s_red[6][8];
    uint32_t vals[6] = {sse, cmp, dpd, n_o, n_b, n_t};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint32_t v = vals[k];
        v = __reduce_add_sync(0xFFFFFFFFu, v);
        if (lane == 0) s_red[k][wid] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        unsigned long long tot = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) tot += s_red[threadIdx.x][i];
        if (tot && a.stats) {
            unsigned long long* st = reinterpret_cast<unsigned long long*>(a.stats + gp);
            const int field[6] = {5, 0, 1, 2, 3, 4};  // sse, cmp, dpd, opaque, boundary, transparent
            atomicAdd(st + field[threadIdx.x], tot);
        }
    }
}

__global__ void sad_texture_single_kernel(const uint8_t* cur, const uint8_t* ref, int W, int H,
                                          int x0, int y0, int bs, int dx2, int dy2, int64_t* out) {
    const int lane = threadIdx.x & 31;
    uint32_t s = 0;
    for (int r = lane; r < bs; r += 32) s += row_sad4(cur, ref, W, H, x0, y0 + r, bs, dx2, dy2);
    s = __reduce_add_sync(0xFFFFFFFFu, s);
    if (lane == 0) out[0] = s;
}

__global__ void sad_shape_single_kernel(const uint8_t* ca, const uint8_t* ra, int W, int H, int x0,
                                        int y0, int bs, int fx, int fy, int64_t* out) {
    const int lane = threadIdx.x & 31;
    uint32_t s = 0;
    for (int r = lane; r < bs; r += 32) s += row_shape(ca, ra, W, H, x0, y0 + r, bs, fx, fy);
    s = __reduce_add_sync(0xFFFFFFFFu, s);
    if (lane == 0) out[0] = int64_t(s) * 255;
}

__global__ void classify_frame_kernel(const uint8_t* alpha, int W, int H, int bs, uint8_t* types) {
    const int cols = W / bs, rows = H / bs;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cols * rows) return;
    types[i] = uint8_t(classify_one(alpha, W, (i % cols) * bs, (i / cols) * bs, bs));
}

__global__ void binarize_kernel(const uint8_t* g, int n, int thr, uint8_t* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = g[i] >= thr ? 255 : 0;
}

__global__ void sse_kernel(const uint8_t* x, const uint8_t* y, int n, unsigned long long* out) {
    unsigned long long s = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int d = int(x[i]) - int(y[i]);
        s += uint64_t(d * d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------

cudaError_t launch_mc_pred(const Batch& b, const me_block_rec* recs, uint8_t* pred, cudaStream_t st) {
    // the SSE and stats are already fused into the classify and search
    // kernels; this pass only materialises the prediction when asked to
    McArgs ma;
    ma.b = b;
    ma.recs = recs;
    ma.stats = nullptr;
    ma.pred = pred;
    ma.mv_override = nullptr;
    ma.types_override = nullptr;
    ma.ref_override = nullptr;
    ma.cur_override = nullptr;
    const int segs = (b.W / 8) * b.H;
    dim3 grid((segs + 255) / 256, b.n_seq * b.pairs);
    mc_kernel<<<grid, 256, 0, st>>>(ma);
    return cudaGetLastError();
}

cudaError_t sad_texture_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                               int size, int dx, int dy, int64_t* out, cudaStream_t st) {
    sad_texture_single_kernel<<<1, 32, 0, st>>>(cur, ref, W, H, x0, y0, size, dx, dy, out);
    return cudaGetLastError();
}

cudaError_t sad_shape_single(const uint8_t* ca, const uint8_t* ra, int W, int H, int x0, int y0,
                             int size, int dx, int dy, int64_t* out, cudaStream_t st) {
    sad_shape_single_kernel<<<1, 32, 0, st>>>(ca, ra, W, H, x0, y0, size, dx / 2, dy / 2, out);
    return cudaGetLastError();
}

cudaError_t classify_frame(const uint8_t* alpha, int W, int H, int bs, uint8_t* types,
                           cudaStream_t st) {
    const int n = (W / bs) * (H / bs);
    classify_frame_kernel<<<(n + 255) / 256, 256, 0, st>>>(alpha, W, H, bs, types);
    return cudaGetLastError();
}

cudaError_t unpack_mask(const uint8_t* bits, uint8_t* out, size_t n, cudaStream_t st) {
    // n / 32 full words; a tail of 8..24 pixels is expanded from a padded word
    const size_t nw = n / 32;
    if (nw) {
        const int grid = int(std::min<size_t>((nw + 255) / 256, 148 * 16));
        unpack_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(bits), reinterpret_cast<uint4*>(out), nw);
    }
    if (n % 32) return cudaErrorInvalidValue;  // callers pass whole 32-pixel groups
    return cudaGetLastError();
}

cudaError_t unpack_mask_sparse(const uint8_t* packed, uint8_t* out, size_t n, cudaStream_t st) {
    if (n % 64) return cudaErrorInvalidValue;
    const size_t nwords = n / 64, ngroups = (nwords + 31) / 32;
    const uint32_t* pres = reinterpret_cast<const uint32_t*>(packed);
    const uint32_t* base = pres + ngroups;
    const auto* lit = reinterpret_cast<const unsigned long long*>(packed + sparse_mask_header_bytes(n));
    const int grid = int(std::min<size_t>((ngroups * 32 + 255) / 256, 148 * 16));
    unpack_sparse_kernel<<<grid, 256, 0, st>>>(pres, base, lit, reinterpret_cast<uint4*>(out), nwords);
    return cudaGetLastError();
}

// bytes -> bit plane (bit = byte != 0), 64 pixels per thread; *nonbinary
// counts 64-pixel words holding a byte other than 0 / 255.
__global__ void pack_mask_kernel(const uint4* __restrict__ in, unsigned long long* __restrict__ out, size_t nwords,
                                 int* nonbinary) {
    for (size_t w = size_t(blockIdx.x) * blockDim.x + threadIdx.x; w < nwords; w += size_t(gridDim.x) * blockDim.x) {
        unsigned long long x = 0;
        uint32_t odd = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = __ldg(in + 4 * w + q);
            const uint32_t vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t nz = __vcmpne4(vs[k], 0u);                     // 0xFF per nonzero byte
                odd |= nz & __vcmpne4(vs[k], 0xFFFFFFFFu);                     // neither 0 nor 255
                const uint32_t b4 = ((nz & 0x01010101u) * 0x01020408u) >> 24;  // byte k -> bit k
                x |= (unsigned long long)(b4 & 15u) << (16 * q + 4 * k);
            }
        }
        out[w] = x;
        if (odd) atomicAdd(nonbinary, 1);
    }
}

cudaError_t pack_mask_dev(const uint8_t* alpha, size_t n, uint8_t* bits, int* nonbinary, cudaStream_t st) {
    if (n % 64) return cudaErrorInvalidValue;
    const size_t nwords = n / 64;
    const int grid = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    pack_mask_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(alpha), reinterpret_cast<unsigned long long*>(bits),
                                           nwords, nonbinary);
    return cudaGetLastError();
}

cudaError_t unpack_mask_sparse_bits(const uint8_t* packed, uint8_t* out_bits, size_t n, cudaStream_t st) {
    if (n % 64) return cudaErrorInvalidValue;
    const size_t nwords = n / 64, ngroups = (nwords + 31) / 32;
    const uint32_t* pres = reinterpret_cast<const uint32_t*>(packed);
    const uint32_t* base = pres + ngroups;
    const auto* lit = reinterpret_cast<const unsigned long long*>(packed + sparse_mask_header_bytes(n));
    const int grid = int(std::min<size_t>((ngroups * 32 + 255) / 256, 148 * 16));
    unpack_sparse_bits_kernel<<<grid, 256, 0, st>>>(pres, base, lit, reinterpret_cast<unsigned long long*>(out_bits), nwords);
    return cudaGetLastError();
}

cudaError_t binarize(const uint8_t* gray, int n, int threshold, uint8_t* out, cudaStream_t st) {
    binarize_kernel<<<std::min((n + 255) / 256, 4096), 256, 0, st>>>(gray, n, threshold, out);
    return cudaGetLastError();
}

cudaError_t predict(const uint8_t* ref, const uint8_t* cur, const int32_t* mv, const uint8_t* types,
                    int W, int H, int bs, uint8_t* pred, me_pair_stats* stats_out,
                    cudaStream_t st) {
    Batch b{};
    b.W = W;
    b.H = H;
    b.bs = bs;
    b.n_seq = 1;
    b.pairs = 1;
    b.F = 1;
    b.d = 0;
    b.cols = W / bs;
    b.rows = H / bs;
    McArgs ma;
    ma.b = b;
    ma.recs = nullptr;
    ma.stats = stats_out;  // only .sse is non-zero (no records)
    ma.pred = pred;
    ma.mv_override = mv;
    ma.types_override = types;
    ma.ref_override = ref;
    ma.cur_override = cur;
    const int segs = (W / 8) * H;
    dim3 grid((segs + 255) / 256, 1);
    mc_kernel<<<grid, 256, 0, st>>>(ma);
    return cudaGetLastError();
}

cudaError_t sse(const uint8_t* a, const uint8_t* b, int n, unsigned long long* out,
                cudaStream_t st) {
    sse_kernel<<<std::min((n + 255) / 256, 1024), 256, 0, st>>>(a, b, n, out);
    return cudaGetLastError();
}

}  // namespace mek
