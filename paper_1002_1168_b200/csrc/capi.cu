// capi.cu — the C ABI (include/me_b200.h): argument validation with the
// reference's error semantics, per-thread contexts with device buffer caches,
// host<->device staging for the host-pointer entry points, and dispatch into
// the kernels (csrc/*.cu).  No CPU compute path exists: every entry point
// either runs on an sm_100 device or fails with ME_ERR_NO_DEVICE.

#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "kernels.h"
#include "me_b200.h"
#include "me_internal.h"

namespace {
thread_local std::string g_last_error;
}

me_status me_fail(me_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

namespace {

me_status ok() {
    g_last_error.clear();
    return ME_OK;
}

bool device_ok(int dev) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return false;
    return p.major == 10;  // sm_100 family (the fatbin carries sm_100a code only)
}

constexpr int kMaxSearchRange = 255;

// SearchConfig::validate + PrsConfig::validate (estimators.cpp:139-150)
me_status validate(const me_config* c) {
    if (!c) return me_fail(ME_ERR_INVALID_ARGUMENT, "null config");
    if (c->search_range < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range must be >= 1");
    // implementation limit of the B200 path (the reference takes any S >= 1):
    // the ES tie-break key holds |dx| + |dy| <= 2S in 9 bits
    if (c->search_range > kMaxSearchRange)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range above 255 is not supported by the B200 path");
    if (c->block_size != 8 && c->block_size != 16)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if (c->ref_distance < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "ref_distance must be >= 1");
    if (!(c->epsilon > 0.0)) return me_fail(ME_ERR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (!(c->theta > 0.0)) return me_fail(ME_ERR_INVALID_ARGUMENT, "theta must be > 0");
    if (c->max_iterations < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "max_iterations must be >= 1");
    if (c->step != 1 && c->step != 2)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "step must be 1 or 2 half-pels");
    if (c->algo < ME_ALGO_ES || c->algo > ME_ALGO_PA)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "unknown algorithm");
    if (c->boundary_temporal != ME_BT_TEXTURE && c->boundary_temporal != ME_BT_SHAPE)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "unknown boundary_temporal");
    return ME_OK;
}

me_status check_rect(int W, int H, int x0, int y0, int size) {
    // require_inside (estimators.cpp:105-110)
    if (x0 < 0 || y0 < 0 || size <= 0 || x0 + size > W || y0 + size > H)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "block rect outside the frame");
    return ME_OK;
}

me_status check_ctx(me_ctx* ctx) {
    if (!ctx) return me_fail(ME_ERR_INVALID_ARGUMENT, "null context");
    if (cudaSetDevice(ctx->device) != cudaSuccess)
        return me_fail(ME_ERR_NO_DEVICE, "cannot select device");
    return ME_OK;
}

// Copies a host plane into a device buffer (size rounded up; zero padded so
// word loads of the last row never leave the allocation).
me_status upload(me_ctx* ctx, DevBuf& buf, size_t off, const void* host, size_t n) {
    ME_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(buf.p) + off, host, n, cudaMemcpyHostToDevice,
                            ctx->stream));
    return ME_OK;
}

size_t pad16(size_t n) { return (n + 15) & ~size_t(15); }

constexpr int kPipelineChunks = 32;  // upper bound (events); default chunk count below

// Lazily creates the copy / d2h streams and the chunk events of the
// host-pointer pipeline.
me_status ensure_pipeline(me_ctx* ctx) {
    if (ctx->copy_stream) return ME_OK;
    ME_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    ME_CUDA(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    for (int k = 0; k < kPipelineChunks; ++k) {
        ME_CUDA(cudaEventCreateWithFlags(&ctx->ev_in[k], cudaEventDisableTiming));
        ME_CUDA(cudaEventCreateWithFlags(&ctx->ev_out[k], cudaEventDisableTiming));
    }
    for (int k = 0; k < 2; ++k) ME_CUDA(cudaEventCreateWithFlags(&ctx->ev_pack[k], cudaEventDisableTiming));
    return ME_OK;
}

// Packs a binary mask to 1 bit per pixel (bit i of byte j = pixel 8j + i) on
// all host cores.  Returns false when some byte is neither 0 nor 255: such a
// mask is not binary and is shipped as bytes (the shape SAD compares byte
// values, so packing would not be exact).
namespace {
// 8 pixels -> 1 byte (bit i = pixel i); false if a byte is neither 0 nor 255
inline bool pack8(const uint8_t* src, uint8_t* dst) {
    uint64_t x;
    std::memcpy(&x, src, 8);
    const uint64_t hi = (x >> 7) & 0x0101010101010101ull;  // bit 0 of each byte = its bit 7
    *dst = uint8_t((hi * 0x0102040810204080ull) >> 56);
    return x == hi * 0xFFu;
}

// 64 pixels per instruction group: the byte MSBs are the packed bits
// (movepi8_mask), and the mask is binary iff every byte equals 0 or 255
__attribute__((target("avx512bw"))) int pack_range_avx512(const uint8_t* src, int64_t b0, int64_t b1, uint8_t* dst) {
    const __m512i zero = _mm512_setzero_si512(), ones = _mm512_set1_epi8(char(0xFF));
    int bad = 0;
    for (int64_t b = b0; b < b1; ++b) {
        const __m512i x = _mm512_loadu_si512(src + 64 * b);
        const __mmask64 ok = _mm512_cmpeq_epi8_mask(x, zero) | _mm512_cmpeq_epi8_mask(x, ones);
        bad |= int(ok != ~__mmask64(0));
        const uint64_t m = _mm512_movepi8_mask(x);
        std::memcpy(dst + 8 * b, &m, 8);
    }
    return bad;
}

int pack_range_scalar(const uint8_t* src, int64_t w0, int64_t w1, uint8_t* dst) {
    int bad = 0;
    for (int64_t i = w0; i < w1; ++i) bad |= int(!pack8(src + 8 * i, dst + i));
    return bad;
}
}  // namespace

// Packs a binary mask to 1 bit per pixel (bit i of byte j = pixel 8j + i) on
// all host cores (AVX-512BW when the CPU has it: measured 53 -> 100+ GB/s on
// the B200 hosts, where the scalar loop was as slow as the PCIe copies it
// overlaps).  Returns false when some byte is neither 0 nor 255: such a mask
// is not binary and is shipped as bytes (the shape SAD compares byte values,
// so packing would not be exact).
bool pack_binary_mask(const uint8_t* src, size_t n, uint8_t* dst, int threads) {
    static const bool avx512 = __builtin_cpu_supports("avx512bw");
    const int64_t nw = int64_t(n / 8), nb = avx512 ? nw / 8 : 0;  // 8-byte words, 64-byte blocks
    int bad = 0;
    const int nth = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel reduction(| : bad) num_threads(nth)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        if (nb) bad |= pack_range_avx512(src, nb * t / nt, nb * (t + 1) / nt, dst);
        const int64_t w0 = 8 * nb;  // the remainder (or everything) in 8-byte words
        bad |= pack_range_scalar(src, w0 + (nw - w0) * t / nt, w0 + (nw - w0) * (t + 1) / nt, dst);
    }
    return !bad;
}

// The sparse form (kernels.h: unpack_mask_sparse) of a binary mask, n % 64 ==
// 0: packs 64 pixels per AVX-512 step (or 8 per scalar step) into tmp, then
// keeps only the nonzero 64-pixel words.  Returns the encoded size in bytes,
// or 0 when the mask is not binary.
size_t pack_sparse_mask(const uint8_t* src, size_t n, uint8_t* dst, uint64_t* tmp, int threads) {
    static const bool avx512 = __builtin_cpu_supports("avx512bw");
    const int64_t nwords = int64_t(n / 64), ngroups = (nwords + 31) / 32;
    uint32_t* pres = reinterpret_cast<uint32_t*>(dst);
    uint32_t* base = pres + ngroups;
    uint64_t* lit = reinterpret_cast<uint64_t*>(dst + mek::sparse_mask_header_bytes(n));
    int bad = 0;
    const int nth = threads > 0 ? threads : omp_get_max_threads();
    std::vector<int64_t> tcount(size_t(nth) + 1, 0);
    int nthreads = 1;
#pragma omp parallel reduction(| : bad) num_threads(nth)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
#pragma omp single
        nthreads = nt;
        const int64_t g0 = ngroups * t / nt, g1 = ngroups * (t + 1) / nt;
        const int64_t w0 = g0 * 32, w1 = std::min(nwords, g1 * 32);
        if (avx512)
            bad |= pack_range_avx512(src, w0, w1, reinterpret_cast<uint8_t*>(tmp));
        else
            bad |= pack_range_scalar(src, 8 * w0, 8 * w1, reinterpret_cast<uint8_t*>(tmp));
        int64_t cnt = 0;
        for (int64_t g = g0; g < g1; ++g) {
            uint32_t m = 0;
            for (int64_t i = 0; i < 32 && g * 32 + i < nwords; ++i) m |= uint32_t(tmp[g * 32 + i] != 0) << i;
            pres[g] = m;
            cnt += __builtin_popcount(m);
        }
        tcount[size_t(t) + 1] = cnt;
#pragma omp barrier
#pragma omp single
        for (int i = 0; i < nt; ++i) tcount[size_t(i) + 1] += tcount[size_t(i)];
        int64_t at = tcount[size_t(t)];
        for (int64_t g = g0; g < g1; ++g) {
            base[g] = uint32_t(at);
            for (uint32_t m = pres[g]; m; m &= m - 1) lit[at++] = tmp[g * 32 + __builtin_ctz(m)];
        }
    }
    if (bad) return 0;
    return mek::sparse_mask_header_bytes(n) + size_t(tcount[size_t(nthreads)]) * 8;
}

me_status sync(me_ctx* ctx) {
    ME_CUDA(cudaStreamSynchronize(ctx->stream));
    ME_CUDA(cudaGetLastError());
    return ME_OK;
}

// Stages up to 4 host planes of n bytes each into ctx->in_luma (contiguous,
// 16-byte padded slots); returns device pointers (null for null inputs).
// The planes are gathered into pinned staging memory (zero padded) and cross
// PCIe in ONE copy: separate copies from pageable memory cost ~10 us each,
// more than the per-block kernels themselves.  Every entry point synchronises
// before returning, so the staging buffer is free again on the next call.
me_status stage_planes(me_ctx* ctx, size_t n, const uint8_t* const* host, const uint8_t** dev,
                       int count) {
    const size_t slot = pad16(n) + 256;
    ME_CUDA(ctx->in_luma.reserve(slot * count));
    ME_CUDA(ctx->pin_a.reserve(slot * count));
    uint8_t* hs = static_cast<uint8_t*>(ctx->pin_a.p);
    for (int i = 0; i < count; ++i) {
        uint8_t* d = hs + slot * i;
        if (host[i]) std::memcpy(d, host[i], n);
        std::memset(d + (host[i] ? n : 0), 0, slot - (host[i] ? n : 0));
        dev[i] = host[i] ? static_cast<const uint8_t*>(ctx->in_luma.p) + slot * i : nullptr;
    }
    ME_CUDA(cudaMemcpyAsync(ctx->in_luma.p, hs, slot * count, cudaMemcpyHostToDevice, ctx->stream));
    return ME_OK;
}

}  // namespace

extern "C" {

const char* me_b200_version(void) { return "me_b200 1.0 (sm_100a)"; }

const char* me_b200_last_error(void) { return g_last_error.c_str(); }

int me_b200_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int good = 0;
    for (int i = 0; i < n; ++i) good += device_ok(i) ? 1 : 0;
    return good;
}

me_status me_b200_ctx_create(int device, me_ctx** out) {
    if (!out) return me_fail(ME_ERR_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return me_fail(ME_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
    }
    if (!device_ok(device))
        return me_fail(ME_ERR_NO_DEVICE, "device " + std::to_string(device) + " is not sm_100");
    ME_CUDA(cudaSetDevice(device));
    me_ctx* c = new me_ctx;
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return me_fail(ME_ERR_CUDA, "stream creation failed");
    }
    *out = c;
    return ok();
}

void me_b200_ctx_destroy(me_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& set : c->ev)
        for (auto& e : set)
            if (e) cudaEventDestroy(e);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamSynchronize(c->d2h_stream);
        for (auto& e : c->ev_in) cudaEventDestroy(e);
        for (auto& e : c->ev_out) cudaEventDestroy(e);
        for (auto& e : c->ev_pack) cudaEventDestroy(e);
        cudaStreamDestroy(c->copy_stream);
        cudaStreamDestroy(c->d2h_stream);
    }
    for (DevBuf* b : {&c->types, &c->worklist, &c->counters, &c->tasks, &c->in_luma, &c->in_alpha, &c->in_bits,
                      &c->out_recs, &c->out_stats, &c->out_pred, &c->aux})
        b->release();
    c->pin_a.release();
    c->pin_b.release();
    for (int i = 0; i < 2; ++i) {
        c->pack_host[i].release();
        c->pack_dev[i].release();
    }
    cudaStreamDestroy(c->stream);
    delete c;
}

void* me_b200_ctx_stream(me_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

me_status me_b200_ctx_set_tuning(me_ctx* ctx, const me_tuning* t) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (!t) return me_fail(ME_ERR_INVALID_ARGUMENT, "null tuning");
    if (t->pa_schedule < 0 || t->pa_schedule > ME_PA_SCHED_QUAD_HYBRID || t->pa_fast_ctas < 0 || t->pa_fast_ctas > 6 ||
        (t->pa_quad_ctas && (t->pa_quad_ctas < 2 || t->pa_quad_ctas > 4)) ||
        (t->pa_duo_threads && t->pa_duo_threads != 128 && t->pa_duo_threads != 256) || t->pa_poll_ns < 0 ||
        t->pa_key_a < 0 || t->pa_key_s < 0 || t->fill_rows_per_cta < 0 || t->h2d_chunks < 0 || t->h2d_chunks > 32 ||
        t->mask_pack < 0 || t->mask_pack > 3 || t->ring_ctas < 0 || t->ring_ctas == 1 || t->ring_ctas > 4 ||
        t->host_threads < 0 || t->pa_key_plain < -1 || t->pa_key_plain > 1)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "tuning field out of range");
    ctx->tuning = *t;
    // the caller's string need not outlive the call: keep a copy
    ctx->trace_path = t->pa_trace_path ? t->pa_trace_path : "";
    ctx->tuning.pa_trace_path = ctx->trace_path.empty() ? nullptr : ctx->trace_path.c_str();
    ctx->tune = mek::resolve_tuning(&ctx->tuning);
    return ok();
}

me_status me_b200_ctx_get_tuning(me_ctx* ctx, me_tuning* out) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (!out) return me_fail(ME_ERR_INVALID_ARGUMENT, "null output");
    *out = ctx->tuning;
    return ok();
}

me_status me_b200_ctx_set_profiling(me_ctx* ctx, int enable) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    ctx->profiling = enable != 0;
    ctx->ev_valid = false;
    return ok();
}

me_status me_b200_pack_mask(const uint8_t* mask, size_t n, uint8_t* out, size_t out_cap, size_t* out_bytes) {
    if (!mask || !out || !out_bytes) return me_fail(ME_ERR_INVALID_ARGUMENT, "null argument");
    if (n % 64) return me_fail(ME_ERR_INVALID_ARGUMENT, "mask size must be a multiple of 64 pixels");
    if (out_cap < mek::sparse_mask_header_bytes(n) + n / 8)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "output buffer too small");
    std::vector<uint64_t> tmp(n / 64 + 1);
    const size_t bytes = pack_sparse_mask(mask, n, out, tmp.data(), 0);
    if (!bytes) return me_fail(ME_ERR_INVALID_ARGUMENT, "mask is not binary (bytes other than 0 and 255)");
    *out_bytes = bytes;
    return ok();
}

me_status me_b200_ctx_launches(me_ctx* ctx, int64_t* out) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (out) *out = ctx->launches;
    return ok();
}

me_status me_b200_ctx_transfer_bytes(me_ctx* ctx, int64_t* h2d, int64_t* d2h) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (h2d) *h2d = ctx->h2d_bytes;
    if (d2h) *d2h = ctx->d2h_bytes;
    return ok();
}

me_status me_b200_ctx_stage_ms(me_ctx* ctx, float* out, int n) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (!ctx->profiling || !ctx->ev_valid)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "no profiled run on this context");
    for (int i = 0; i < n && i < ME_NUM_STAGES; ++i) out[i] = 0.f;
    for (int k = 0; k < ctx->ev_sets; ++k) {  // every sub-batch of the last call
        ME_CUDA(cudaEventSynchronize(ctx->ev[k][4]));
        for (int i = 0; i < n && i < ME_NUM_STAGES; ++i) {
            float ms = 0.f;
            ME_CUDA(cudaEventElapsedTime(&ms, ctx->ev[k][i], ctx->ev[k][i + 1]));
            out[i] += ms;
        }
    }
    return ok();
}

me_status me_b200_validate_config(const me_config* cfg) {
    me_status s = validate(cfg);
    return s ? s : ok();
}

static me_status check_batch(const me_config* cfg, int n_seq, int n_frames, int W, int H) {
    me_status s = validate(cfg);
    if (s) return s;
    if (n_seq < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "n_seq must be >= 1");
    if (W <= 0 || H <= 0 || W % 16 || H % 16)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "frame dimensions must be positive multiples of 16");
    if (cfg->ref_distance >= n_frames)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "ref_distance must be smaller than the frame count");
    const int64_t nb = int64_t(n_seq) * (n_frames - cfg->ref_distance) * (W / cfg->block_size) *
                       (H / cfg->block_size);
    if (nb >= (int64_t(1) << 31)) return me_fail(ME_ERR_INVALID_ARGUMENT, "batch too large (2^31 blocks)");
    if (n_seq >= 65536 || n_frames - cfg->ref_distance >= 65536 || H / cfg->block_size >= 32768 ||
        W / cfg->block_size >= 65536)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "batch geometry exceeds the work-list encoding");
    if (cfg->algo == ME_ALGO_PA && (W / cfg->block_size - 1) + 2 * (H / cfg->block_size - 1) +
                                           (n_frames - cfg->ref_distance) > 12000)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "wavefront longer than 12000 steps");
    if (int64_t(W - cfg->block_size + 1) * (H - cfg->block_size + 1) >= (int64_t(1) << 24))
        return me_fail(ME_ERR_INVALID_ARGUMENT, "frame too large for the packed ES key");
    return ME_OK;
}

static mek::Batch make_batch(const me_config* cfg, int n_seq, int n_frames, int W, int H,
                             const uint8_t* luma, const uint8_t* alpha) {
    mek::Batch b;
    b.luma = luma;
    b.alpha = alpha;
    b.n_seq = n_seq;
    b.F = n_frames;
    b.W = W;
    b.H = H;
    b.d = cfg->ref_distance;
    b.pairs = n_frames - cfg->ref_distance;
    b.bs = cfg->block_size;
    b.cols = W / cfg->block_size;
    b.rows = H / cfg->block_size;
    return b;
}

me_status me_b200_run_sequences_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                                    int W, int H, const uint8_t* luma, const uint8_t* alpha,
                                    me_block_rec* recs, me_pair_stats* stats, uint8_t* pred,
                                    void* stream) {
    mek::NvtxRange nv("me_b200_run_sequences_dev");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_batch(cfg, n_seq, n_frames, W, H))) return s;
    if (!luma || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if ((reinterpret_cast<uintptr_t>(luma) | reinterpret_cast<uintptr_t>(alpha) |
         reinterpret_cast<uintptr_t>(recs)) & 15)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "device buffers must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: the CUDA default stream
    // Sequences are independent: a batch whose frames span 4 GiB or more runs
    // as consecutive sub-batches below 4 GiB each, so every one takes the
    // kernels with 32-bit plane offsets.
    const size_t seq_bytes = size_t(n_frames) * size_t(W) * size_t(H);
    const int per = int(std::max<size_t>(1, std::min<size_t>(size_t(n_seq), ((size_t(1) << 32) - 1) / seq_bytes)));
    const int pairs = n_frames - cfg->ref_distance;
    const size_t seq_recs = size_t(pairs) * (W / cfg->block_size) * (H / cfg->block_size);
    ctx->launches = 0;
    ctx->ev_sets = 0;
    for (int s0 = 0; s0 < n_seq; s0 += per) {
        const int ns = std::min(per, n_seq - s0);
        const mek::Batch b = make_batch(cfg, ns, n_frames, W, H, luma + seq_bytes * s0,
                                        alpha ? alpha + seq_bytes * s0 : nullptr);
        ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
        int nl = 0;
        ME_CUDA(mek::run_batch(b, *cfg, nullptr, recs + seq_recs * s0, stats + size_t(pairs) * s0,
                               pred ? pred + size_t(W) * H * pairs * s0 : nullptr, ctx->tasks.p, ctx->tasks.cap,
                               ctx->num_sms, st, ctx->tune, ctx->events(s0 / per), false, &nl));
        ctx->launches += nl;
    }
    ctx->ev_valid = ctx->profiling;
    return ok();
}

me_status me_b200_run_sequences_bits_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                                         int W, int H, const uint8_t* luma, const uint8_t* alpha_bits,
                                         me_block_rec* recs, me_pair_stats* stats, uint8_t* pred,
                                         void* stream) {
    mek::NvtxRange nv("me_b200_run_sequences_bits_dev");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_batch(cfg, n_seq, n_frames, W, H))) return s;
    if (!luma || !alpha_bits || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if ((reinterpret_cast<uintptr_t>(luma) | reinterpret_cast<uintptr_t>(recs)) & 15 ||
        reinterpret_cast<uintptr_t>(alpha_bits) & 7)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "device buffers must be 16-byte (masks 8-byte) aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t seq_bytes = size_t(n_frames) * size_t(W) * size_t(H);
    const int per = int(std::max<size_t>(1, std::min<size_t>(size_t(n_seq), ((size_t(1) << 32) - 1) / seq_bytes)));
    const int pairs = n_frames - cfg->ref_distance;
    const size_t seq_recs = size_t(pairs) * (W / cfg->block_size) * (H / cfg->block_size);
    ctx->launches = 0;
    ctx->ev_sets = 0;
    for (int s0 = 0; s0 < n_seq; s0 += per) {
        const int ns = std::min(per, n_seq - s0);
        mek::Batch b = make_batch(cfg, ns, n_frames, W, H, luma + seq_bytes * s0, nullptr);
        b.alpha_bits = alpha_bits + seq_bytes / 8 * s0;
        if (cfg->algo == ME_ALGO_PA && !mek::pa_takes_bits(b, *cfg, ctx->num_sms, ctx->tune)) {
            // this PA schedule (16x16 blocks, half-pel, duo kernels) reads mask bytes
            ME_CUDA(ctx->aux.reserve(seq_bytes * ns));
            ME_CUDA(mek::unpack_mask(b.alpha_bits, static_cast<uint8_t*>(ctx->aux.p), seq_bytes * ns, st));
            b.alpha = static_cast<const uint8_t*>(ctx->aux.p);
            b.alpha_bits = nullptr;
            ctx->launches += 1;
        }
        ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
        int nl = 0;
        ME_CUDA(mek::run_batch(b, *cfg, nullptr, recs + seq_recs * s0, stats + size_t(pairs) * s0,
                               pred ? pred + size_t(W) * H * pairs * s0 : nullptr, ctx->tasks.p, ctx->tasks.cap,
                               ctx->num_sms, st, ctx->tune, ctx->events(s0 / per), false, &nl));
        ctx->launches += nl;
    }
    ctx->ev_valid = ctx->profiling;
    return ok();
}

me_status me_b200_pack_mask_dev(me_ctx* ctx, const uint8_t* alpha, size_t n, uint8_t* bits, int* binary,
                                void* stream) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (!alpha || !bits || !binary || n % 64) return me_fail(ME_ERR_INVALID_ARGUMENT, "bad mask buffers");
    ME_CUDA(ctx->aux.reserve(16));
    int* flag = static_cast<int*>(ctx->aux.p);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ME_CUDA(cudaMemsetAsync(flag, 0, 4, st));
    ME_CUDA(mek::pack_mask_dev(alpha, n, bits, flag, st));
    ME_CUDA(cudaMemcpyAsync(binary, flag, 4, cudaMemcpyDeviceToHost, st));
    ME_CUDA(cudaStreamSynchronize(st));
    *binary = !*binary;  // flag counts non-binary bytes
    return ok();
}

me_status me_b200_run_sequence_prev_dev(me_ctx* ctx, const me_config* cfg, int n_frames, int W, int H,
                                        const uint8_t* luma, const uint8_t* alpha, const int32_t* prev_mv,
                                        int prev_integer, me_block_rec* recs, me_pair_stats* stats,
                                        void* stream) {
    mek::NvtxRange nv("me_b200_run_sequence_prev_dev");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_batch(cfg, 1, n_frames, W, H))) return s;
    if (!luma || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if ((reinterpret_cast<uintptr_t>(luma) | reinterpret_cast<uintptr_t>(alpha) |
         reinterpret_cast<uintptr_t>(recs)) & 15 || reinterpret_cast<uintptr_t>(prev_mv) & 3)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "device buffers must be 16-byte aligned");
    if (size_t(n_frames) * W * H >= (size_t(1) << 32))
        return me_fail(ME_ERR_INVALID_ARGUMENT, "a streamed chunk must stay below 4 GiB");
    const mek::Batch b = make_batch(cfg, 1, n_frames, W, H, luma, alpha);
    ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
    int nl = 0;
    ME_CUDA(mek::run_batch(b, *cfg, cfg->algo == ME_ALGO_PA ? prev_mv : nullptr, recs, stats, nullptr, ctx->tasks.p,
                           ctx->tasks.cap, ctx->num_sms, static_cast<cudaStream_t>(stream), ctx->tune,
                           (ctx->ev_sets = 0, ctx->events()), prev_integer != 0, &nl));
    ctx->launches = nl;
    ctx->ev_valid = ctx->profiling;
    return ok();
}

me_status me_b200_run_band_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames, int W,
                               int H, const uint8_t* luma, const uint8_t* alpha, int row0, int row1,
                               me_block_rec* recs, me_pair_stats* stats, void* stream) {
    mek::NvtxRange nv("me_b200_run_band_dev");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_batch(cfg, n_seq, n_frames, W, H))) return s;
    if (cfg->algo == ME_ALGO_PA)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "PA blocks depend on the rows above: no row bands");
    const int rows = H / cfg->block_size;
    if (row0 < 0 || row1 > rows || row0 >= row1) return me_fail(ME_ERR_INVALID_ARGUMENT, "bad row band");
    if (!luma || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if ((reinterpret_cast<uintptr_t>(luma) | reinterpret_cast<uintptr_t>(alpha) |
         reinterpret_cast<uintptr_t>(recs)) & 15)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "device buffers must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    mek::Batch b = make_batch(cfg, n_seq, n_frames, W, H, luma, alpha);
    b.v0 = row0;
    b.v1 = row1;
    ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
    int nl = 0;
    ME_CUDA(mek::run_batch(b, *cfg, nullptr, recs, stats, nullptr, ctx->tasks.p, ctx->tasks.cap, ctx->num_sms,
                           st, ctx->tune, (ctx->ev_sets = 0, ctx->events()), false, &nl));
    ctx->launches = nl;
    ctx->ev_valid = ctx->profiling;
    return ok();
}

// Several devices from one process: units (sequences, or for a single
// sequence of a baseline, frame pairs) sharded contiguously over devices
// 0..n_gpus-1, each shard run end to end by its own host thread and context;
// the results land in the caller's host arrays, so rank 0's gather is the
// D2H itself.
// Contexts of the multi-device entry, reused across calls (device buffers and
// pinned staging are grow-only): a call checks one out per device and returns
// it, so concurrent callers never share one.
namespace {
std::mutex g_multi_mu;
std::vector<std::vector<me_ctx*>> g_multi_free;

me_status multi_ctx_get(int device, me_ctx** out) {
    {
        std::lock_guard<std::mutex> lk(g_multi_mu);
        if (int(g_multi_free.size()) > device && !g_multi_free[device].empty()) {
            *out = g_multi_free[device].back();
            g_multi_free[device].pop_back();
            return ME_OK;
        }
    }
    return me_b200_ctx_create(device, out);
}

void multi_ctx_put(int device, me_ctx* c) {
    std::lock_guard<std::mutex> lk(g_multi_mu);
    if (int(g_multi_free.size()) <= device) g_multi_free.resize(device + 1);
    g_multi_free[device].push_back(c);
}
}  // namespace

me_status me_b200_run_sequences_multi(const me_config* cfg, int n_seq, int n_frames, int W, int H,
                                      const uint8_t* luma, const uint8_t* alpha, me_block_rec* recs,
                                      me_pair_stats* stats, int n_gpus) {
    mek::NvtxRange nv("me_b200_run_sequences_multi");
    me_status s = check_batch(cfg, n_seq, n_frames, W, H);
    if (s) return s;
    if (!luma || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    if (n_gpus < 1 || n_gpus > ndev)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "n_gpus must be between 1 and the visible device count");
    const size_t plane = size_t(W) * H, seq_bytes = plane * n_frames;
    const int pairs = n_frames - cfg->ref_distance;
    const size_t pair_recs = size_t(W / cfg->block_size) * (H / cfg->block_size);
    // a lone baseline sequence shards by frame pairs (pairs are independent
    // for ES/TSS/FSS/DS; PA pairs chain through the temporal candidate)
    const bool by_pair = n_seq == 1 && cfg->algo != ME_ALGO_PA && pairs > 1;
    const int units = by_pair ? pairs : n_seq;
    const int ng = std::min(n_gpus, units);
    std::vector<me_status> rc(ng, ME_OK);
    std::vector<std::string> msg(ng);
    auto work = [&](int g) {
        const int u0 = int(int64_t(units) * g / ng), u1 = int(int64_t(units) * (g + 1) / ng);
        me_ctx* c = nullptr;
        me_status r = multi_ctx_get(g, &c);
        if (!r) {
            if (by_pair)  // pairs [u0, u1) = frames [u0, u1 + d)
                r = me_b200_run_sequences(c, cfg, 1, (u1 - u0) + cfg->ref_distance, W, H, luma + plane * u0,
                                          alpha ? alpha + plane * u0 : nullptr, recs + pair_recs * u0,
                                          stats + u0, nullptr);
            else
                r = me_b200_run_sequences(c, cfg, u1 - u0, n_frames, W, H, luma + seq_bytes * u0,
                                          alpha ? alpha + seq_bytes * u0 : nullptr,
                                          recs + pair_recs * pairs * u0, stats + size_t(pairs) * u0, nullptr);
        }
        if (r) msg[g] = g_last_error;
        rc[g] = r;
        if (c) multi_ctx_put(g, c);
    };
    std::vector<std::thread> pool;
    for (int g = 1; g < ng; ++g) pool.emplace_back(work, g);
    work(0);
    for (auto& t : pool) t.join();
    for (int g = 0; g < ng; ++g)
        if (rc[g]) return me_fail(rc[g], "device " + std::to_string(g) + ": " + msg[g]);
    return ok();
}

me_status me_b200_run_sequences(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames, int W,
                                int H, const uint8_t* luma, const uint8_t* alpha,
                                me_block_rec* recs, me_pair_stats* stats, uint8_t* pred) {
    mek::NvtxRange nv("me_b200_run_sequences");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_batch(cfg, n_seq, n_frames, W, H))) return s;
    if (!luma || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const size_t plane = size_t(W) * H;
    const size_t seq_bytes = plane * n_frames;
    const int pairs = n_frames - cfg->ref_distance;
    const size_t seq_recs = size_t(pairs) * (W / cfg->block_size) * (H / cfg->block_size);
    ME_CUDA(ctx->in_luma.reserve(seq_bytes * n_seq + 256));
    if (alpha) ME_CUDA(ctx->in_alpha.reserve(seq_bytes * n_seq + 256));
    if (alpha) ME_CUDA(ctx->in_bits.reserve(seq_bytes * n_seq / 8 + 256));
    ME_CUDA(ctx->out_recs.reserve(seq_recs * n_seq * sizeof(me_block_rec)));
    ME_CUDA(ctx->out_stats.reserve(size_t(n_seq) * pairs * sizeof(me_pair_stats)));
    if (pred) ME_CUDA(ctx->out_pred.reserve(plane * pairs * n_seq));
    if ((s = ensure_pipeline(ctx))) return s;
    // Chunked pipeline: the sequences are independent, so chunk k's H2D (copy
    // stream) overlaps chunk k-1's estimation (compute stream) and chunk
    // k-2's D2H (d2h stream).  PCIe is the bound of this path.

    const int nchunks = std::min(n_seq, std::max(1, std::min(kPipelineChunks, ctx->tune.h2d_chunks)));
    uint8_t* dl = static_cast<uint8_t*>(ctx->in_luma.p);
    uint8_t* da = static_cast<uint8_t*>(ctx->in_alpha.p);
    uint8_t* dbits = static_cast<uint8_t*>(ctx->in_bits.p);
    me_block_rec* dr = static_cast<me_block_rec*>(ctx->out_recs.p);
    me_pair_stats* ds = static_cast<me_pair_stats*>(ctx->out_stats.p);
    uint8_t* dp = static_cast<uint8_t*>(ctx->out_pred.p);
    // Binary alpha masks cross PCIe bit-packed (packed on the host cores while
    // the previous chunk's copies are in flight, expanded on the device).
    const bool pack = alpha && ctx->tune.mask_pack != 1;
    const bool sparse = ctx->tune.mask_pack != 2;
    const size_t max_chunk = seq_bytes * size_t((n_seq + nchunks - 1) / nchunks);
    if (pack)
        for (int i = 0; i < 2; ++i) {
            ME_CUDA(ctx->pack_host[i].reserve(mek::sparse_mask_header_bytes(max_chunk) + max_chunk / 8 + 64));
            ME_CUDA(ctx->pack_dev[i].reserve(mek::sparse_mask_header_bytes(max_chunk) + max_chunk / 8 + 64));
        }
    ctx->h2d_bytes = ctx->d2h_bytes = 0;
    ctx->launches = 0;
    for (int k = 0; k < nchunks; ++k) {
        const int s0 = int(int64_t(n_seq) * k / nchunks), s1 = int(int64_t(n_seq) * (k + 1) / nchunks);
        const int ns = s1 - s0;
        const size_t o = seq_bytes * s0, n = seq_bytes * ns;
        ME_CUDA(cudaMemcpyAsync(dl + o, luma + o, n, cudaMemcpyHostToDevice, ctx->copy_stream));
        ctx->h2d_bytes += int64_t(n);
        bool packed_chunk = false;  // the mask went bit-packed (binary)
        int unpack_launches = 0;    // the sparse form's expansion to the dense bit plane
        if (alpha) {
            const int slot = k & 1;
            bool packed = false;
            if (pack) {
                // the copy out of this staging slot (chunk k - 2) must be done
                if (k >= 2) ME_CUDA(cudaEventSynchronize(ctx->ev_pack[slot]));
                uint8_t* hb = static_cast<uint8_t*>(ctx->pack_host[slot].p);
                uint8_t* db = static_cast<uint8_t*>(ctx->pack_dev[slot].p);
                if (n % 64 == 0 && sparse) {
                    // zero 64-pixel words elided (object masks are mostly background)
                    if (ctx->pack_tmp.size() < n / 64) ctx->pack_tmp.resize(max_chunk / 64 + 1);
                    const size_t bytes = pack_sparse_mask(alpha + o, n, hb, ctx->pack_tmp.data(), ctx->tune.host_threads);
                    if ((packed = bytes > 0)) {
                        ME_CUDA(cudaMemcpyAsync(db, hb, bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
                        ctx->h2d_bytes += int64_t(bytes);
                        ME_CUDA(cudaEventRecord(ctx->ev_pack[slot], ctx->copy_stream));
                        // to the dense bit plane the kernels read (not to bytes)
                        ME_CUDA(mek::unpack_mask_sparse_bits(db, dbits + o / 8, n, ctx->copy_stream));
                        unpack_launches = 1;
                    }
                } else if ((packed = pack_binary_mask(alpha + o, n, hb, ctx->tune.host_threads))) {
                    // the dense bit plane itself
                    ME_CUDA(cudaMemcpyAsync(dbits + o / 8, hb, n / 8, cudaMemcpyHostToDevice, ctx->copy_stream));
                    ctx->h2d_bytes += int64_t(n / 8);
                    ME_CUDA(cudaEventRecord(ctx->ev_pack[slot], ctx->copy_stream));
                }
                packed_chunk = packed;
            }
            if (!packed) {
                ME_CUDA(cudaMemcpyAsync(da + o, alpha + o, n, cudaMemcpyHostToDevice, ctx->copy_stream));
                ctx->h2d_bytes += int64_t(n);
            }
        }
        ME_CUDA(cudaEventRecord(ctx->ev_in[k], ctx->copy_stream));
        // estimation of chunk k (compute stream) and its D2H (d2h stream)
        ME_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[k], 0));
        mek::Batch b = make_batch(cfg, ns, n_frames, W, H, dl + seq_bytes * s0,
                                  alpha ? da + seq_bytes * s0 : nullptr);
        int nl = 0;
        if (packed_chunk) {  // binary masks: the kernels read the bit plane (popc(XOR) shape SADs)
            b.alpha = nullptr;
            b.alpha_bits = dbits + seq_bytes * s0 / 8;
            if (cfg->algo == ME_ALGO_PA && !mek::pa_takes_bits(b, *cfg, ctx->num_sms, ctx->tune)) {
                ME_CUDA(mek::unpack_mask(b.alpha_bits, da + seq_bytes * s0, n, ctx->stream));  // this schedule reads bytes
                b.alpha = da + seq_bytes * s0;
                b.alpha_bits = nullptr;
                ++nl;
            }
        }
        ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
        int nb = 0;
        ME_CUDA(mek::run_batch(b, *cfg, nullptr, dr + seq_recs * s0, ds + size_t(pairs) * s0,
                               pred ? dp + plane * pairs * s0 : nullptr, ctx->tasks.p, ctx->tasks.cap,
                               ctx->num_sms, ctx->stream, ctx->tune, nullptr, false, &nb));
        ctx->launches += nl + nb + unpack_launches;
        ME_CUDA(cudaEventRecord(ctx->ev_out[k], ctx->stream));
        ME_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_out[k], 0));
        ME_CUDA(cudaMemcpyAsync(recs + seq_recs * s0, dr + seq_recs * s0, seq_recs * ns * sizeof(me_block_rec),
                                cudaMemcpyDeviceToHost, ctx->d2h_stream));
        ME_CUDA(cudaMemcpyAsync(stats + size_t(pairs) * s0, ds + size_t(pairs) * s0,
                                size_t(pairs) * ns * sizeof(me_pair_stats), cudaMemcpyDeviceToHost,
                                ctx->d2h_stream));
        if (pred)
            ME_CUDA(cudaMemcpyAsync(pred + plane * pairs * s0, dp + plane * pairs * s0, plane * pairs * ns,
                                    cudaMemcpyDeviceToHost, ctx->d2h_stream));
        ctx->d2h_bytes += int64_t(seq_recs * ns * sizeof(me_block_rec) + size_t(pairs) * ns * sizeof(me_pair_stats) +
                                  (pred ? plane * pairs * ns : 0));
    }
    ctx->ev_valid = false;
    ME_CUDA(cudaStreamSynchronize(ctx->d2h_stream));
    s = sync(ctx);
    return s ? s : ok();
}

me_status me_b200_estimate_field(me_ctx* ctx, const me_config* cfg, int W, int H,
                                 const uint8_t* cur, const uint8_t* ref, const uint8_t* cur_alpha,
                                 const uint8_t* ref_alpha, const int32_t* prev_mv, int prev_cols,
                                 int prev_rows, me_block_rec* recs, me_pair_stats* stats) {
    mek::NvtxRange nv("me_b200_estimate_field");
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = validate(cfg))) return s;  // cfg.validate(); prs.validate() (estimators.cpp:390-391)
    if (!cur || !ref || !recs || !stats) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if (W <= 0 || H <= 0) return me_fail(ME_ERR_INVALID_ARGUMENT, "frame dimensions must be positive");
    const int bs = cfg->block_size;
    if (W % bs || H % bs)  // block_grid (frame.cpp:106-110)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "block size does not divide the frame");
    const int cols = W / bs, rows = H / bs;
    if (prev_mv && (prev_cols != cols || prev_rows != rows))
        return me_fail(ME_ERR_INVALID_ARGUMENT, "previous motion field grid mismatch");
    if (W % 8) return me_fail(ME_ERR_INVALID_ARGUMENT, "frame width must be a multiple of 8");
    const size_t plane = size_t(W) * H;
    // frame 0 = ref, frame 1 = cur (one pair at ref_distance 1)
    me_config c1 = *cfg;
    c1.ref_distance = 1;
    // one pinned staging buffer -> one H2D: [ref, cur, ref alpha, cur alpha, prev]
    const size_t prev_bytes = prev_mv ? size_t(cols) * rows * 8 : 0;
    const size_t total = (cur_alpha ? 4 : 2) * plane + prev_bytes;
    const size_t out_bytes = size_t(cols) * rows * sizeof(me_block_rec) + sizeof(me_pair_stats);
    ME_CUDA(ctx->in_luma.reserve(total + 256));
    ME_CUDA(ctx->out_recs.reserve(out_bytes));
    ME_CUDA(ctx->aux.reserve(size_t(cols) * rows + 256));
    ME_CUDA(ctx->pin_a.reserve(total + 256));
    ME_CUDA(ctx->pin_b.reserve(out_bytes));
    // the batch layout expects frames back to back; pad-free when plane % 16 == 0
    if (plane % 16) return me_fail(ME_ERR_INVALID_ARGUMENT, "frame area must be a multiple of 16");
    uint8_t* hs = static_cast<uint8_t*>(ctx->pin_a.p);
    std::memcpy(hs, ref, plane);
    std::memcpy(hs + plane, cur, plane);
    if (cur_alpha) {
        if (ref_alpha)
            std::memcpy(hs + 2 * plane, ref_alpha, plane);
        else
            std::memset(hs + 2 * plane, 0, plane);
        std::memcpy(hs + 3 * plane, cur_alpha, plane);
    }
    if (prev_mv) std::memcpy(hs + total - prev_bytes, prev_mv, prev_bytes);
    ME_CUDA(cudaMemcpyAsync(ctx->in_luma.p, hs, total, cudaMemcpyHostToDevice, ctx->stream));
    uint8_t* L = static_cast<uint8_t*>(ctx->in_luma.p);
    uint8_t* A = L + 2 * plane;
    const uint8_t* alpha_dev = nullptr;
    if (cur_alpha) {
        alpha_dev = A;
        if (!ref_alpha && cfg->algo == ME_ALGO_PA) {
            // brs_select throws on a boundary block without both planes
            // (estimators.cpp:266-268): classify first, before any estimation.
            uint8_t* types = static_cast<uint8_t*>(ctx->aux.p);
            ME_CUDA(mek::classify_frame(A + plane, W, H, bs, types, ctx->stream));
            std::vector<uint8_t> ht(size_t(cols) * rows);
            ME_CUDA(cudaMemcpyAsync(ht.data(), types, ht.size(), cudaMemcpyDeviceToHost, ctx->stream));
            if ((s = sync(ctx))) return s;
            for (uint8_t t : ht)
                if (t == ME_BOUNDARY)
                    return me_fail(ME_ERR_INVALID_ARGUMENT, "boundary block requires both alpha planes");
        }
    }
    int32_t* prev_dev = prev_mv ? reinterpret_cast<int32_t*>(L + total - prev_bytes) : nullptr;
    bool prev_integer = true;  // integer-pel prev fields can take the fast PA kernels
    if (prev_mv)
        for (size_t i = 0; i < size_t(cols) * rows * 2 && prev_integer; ++i) prev_integer = (prev_mv[i] & 1) == 0;
    const mek::Batch b = make_batch(&c1, 1, 2, W, H, L, alpha_dev);
    ME_CUDA(ctx->tasks.reserve(mek::scratch_bytes(b, cfg->algo, ctx->tune)));
    // records and stats in one device buffer -> one D2H into pinned memory
    me_block_rec* dr = static_cast<me_block_rec*>(ctx->out_recs.p);
    me_pair_stats* ds = reinterpret_cast<me_pair_stats*>(dr + size_t(cols) * rows);
    int nl = 0;
    ME_CUDA(mek::run_batch(b, c1, prev_dev, dr, ds, nullptr, ctx->tasks.p, ctx->tasks.cap, ctx->num_sms,
                           ctx->stream, ctx->tune, (ctx->ev_sets = 0, ctx->events()), prev_integer, &nl));
    ctx->launches = nl;
    ctx->ev_valid = ctx->profiling;
    ME_CUDA(cudaMemcpyAsync(ctx->pin_b.p, dr, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    if (s) return s;
    std::memcpy(recs, ctx->pin_b.p, size_t(cols) * rows * sizeof(me_block_rec));
    std::memcpy(stats, static_cast<uint8_t*>(ctx->pin_b.p) + size_t(cols) * rows * sizeof(me_block_rec),
                sizeof(me_pair_stats));
    return ok();
}

me_status me_b200_block_search(me_ctx* ctx, int algo, int W, int H, const uint8_t* cur,
                               const uint8_t* ref, int x0, int y0, int size, int range,
                               int32_t out_mv[2], int64_t* out_cmp, uint32_t* out_cost_q4) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (algo < ME_ALGO_ES || algo > ME_ALGO_DS)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "not a block search");
    if (range < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range must be >= 1");
    if (range > kMaxSearchRange) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range above 255 is not supported by the B200 path");
    if (size != 8 && size != 16) return me_fail(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if ((s = check_rect(W, H, x0, y0, size))) return s;
    if (!cur || !ref || !out_mv) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const uint8_t* host[2] = {cur, ref};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    int64_t* out = static_cast<int64_t*>(ctx->aux.p);
    ME_CUDA(mek::block_search(algo, dev[0], dev[1], W, H, x0, y0, size, range, out, ctx->stream));
    int64_t h[4];
    ME_CUDA(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if ((s = sync(ctx))) return s;
    out_mv[0] = int32_t(h[0]);
    out_mv[1] = int32_t(h[1]);
    if (out_cmp) *out_cmp = h[2];
    if (out_cost_q4) *out_cost_q4 = uint32_t(h[3]);
    return ok();
}

me_status me_b200_brs_select(me_ctx* ctx, int W, int H, const uint8_t* cur, const uint8_t* ref,
                             const uint8_t* cur_alpha, const uint8_t* ref_alpha, int x0, int y0,
                             int size, int btype, const int32_t cands[8], int range,
                             int boundary_temporal, int32_t out_mv[2], uint8_t out_kinds[4],
                             uint32_t out_scores_q4[4]) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    // cfg.validate(); require_inside; type checks (estimators.cpp:261-268)
    if (range < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range must be >= 1");
    if (range > kMaxSearchRange) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range above 255 is not supported by the B200 path");
    if (size != 8 && size != 16) return me_fail(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if ((s = check_rect(W, H, x0, y0, size))) return s;
    if (btype == ME_TRANSPARENT)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "candidate selection on a transparent block");
    if (btype == ME_BOUNDARY && (!cur_alpha || !ref_alpha))
        return me_fail(ME_ERR_INVALID_ARGUMENT, "boundary block requires both alpha planes");
    if (!cur || !ref || !cands || !out_mv) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const uint8_t* host[4] = {cur, ref, btype == ME_BOUNDARY ? cur_alpha : nullptr,
                              btype == ME_BOUNDARY ? ref_alpha : nullptr};
    const uint8_t* dev[4];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 4))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    int64_t* out = static_cast<int64_t*>(ctx->aux.p);
    int32_t* cd = reinterpret_cast<int32_t*>(out + 16);
    ME_CUDA(cudaMemcpyAsync(cd, cands, 8 * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    ME_CUDA(mek::brs_single(dev[0], dev[1], dev[2], dev[3], W, H, x0, y0, size, btype, cd, range,
                            boundary_temporal, out, ctx->stream));
    int64_t h[10];
    ME_CUDA(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if ((s = sync(ctx))) return s;
    out_mv[0] = int32_t(h[0]);
    out_mv[1] = int32_t(h[1]);
    for (int i = 0; i < 4; ++i) {
        if (out_scores_q4) out_scores_q4[i] = uint32_t(h[2 + i]);
        if (out_kinds) out_kinds[i] = uint8_t(h[6 + i]);
    }
    return ok();
}

me_status me_b200_prs_refine(me_ctx* ctx, int W, int H, const uint8_t* cur, const uint8_t* ref,
                             int x0, int y0, int size, const int32_t d0[2], int range,
                             double epsilon, double theta, int max_iterations, int step,
                             int32_t out_mv[2], int64_t* out_dpd, uint32_t* log_q4, int* log_len) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (range < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range must be >= 1");
    if (range > kMaxSearchRange) return me_fail(ME_ERR_INVALID_ARGUMENT, "search_range above 255 is not supported by the B200 path");
    if (size != 8 && size != 16) return me_fail(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if (!(epsilon > 0.0)) return me_fail(ME_ERR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (!(theta > 0.0)) return me_fail(ME_ERR_INVALID_ARGUMENT, "theta must be > 0");
    if (max_iterations < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "max_iterations must be >= 1");
    if (step != 1 && step != 2) return me_fail(ME_ERR_INVALID_ARGUMENT, "step must be 1 or 2 half-pels");
    if ((s = check_rect(W, H, x0, y0, size))) return s;
    if (!cur || !ref || !d0 || !out_mv) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const uint8_t* host[2] = {cur, ref};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(128 * 8));
    int64_t* out = static_cast<int64_t*>(ctx->aux.p);
    ME_CUDA(mek::prs_single(dev[0], dev[1], W, H, x0, y0, size, d0[0], d0[1], range, epsilon, theta,
                            max_iterations, step, out, ctx->stream));
    int64_t h[69];
    ME_CUDA(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if ((s = sync(ctx))) return s;
    out_mv[0] = int32_t(h[0]);
    out_mv[1] = int32_t(h[1]);
    if (out_dpd) *out_dpd = h[2];
    const int n = int(h[3]) + 1;
    if (log_len) *log_len = n;
    if (log_q4)
        for (int i = 0; i < n && i < 64; ++i) log_q4[i] = uint32_t(h[5 + i]);
    return ok();
}

me_status me_b200_prs_update(me_ctx* ctx, int W, int H, const uint8_t* cur, const uint8_t* ref, int x,
                             int y, const int32_t d[2], double epsilon, double theta, double out[2]) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (!cur || !ref || !d || !out) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    if (W <= 0 || H <= 0 || x < 0 || y < 0 || x >= W || y >= H)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "pixel outside the frame");
    const uint8_t* host[2] = {cur, ref};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    double* o = static_cast<double*>(ctx->aux.p);
    ME_CUDA(mek::prs_update_single(dev[0], dev[1], W, H, x, y, d[0], d[1], epsilon, theta, o, ctx->stream));
    ME_CUDA(cudaMemcpyAsync(out, o, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    return s ? s : ok();
}

me_status me_b200_sad_texture(me_ctx* ctx, int W, int H, const uint8_t* cur, const uint8_t* ref,
                              int x0, int y0, int size, int dx, int dy, uint32_t* out_sad_q4) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((s = check_rect(W, H, x0, y0, size))) return s;
    if (size > 64) return me_fail(ME_ERR_INVALID_ARGUMENT, "block size above 64");
    if (!cur || !ref || !out_sad_q4) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const uint8_t* host[2] = {cur, ref};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    int64_t* out = static_cast<int64_t*>(ctx->aux.p);
    ME_CUDA(mek::sad_texture_single(dev[0], dev[1], W, H, x0, y0, size, dx, dy, out, ctx->stream));
    int64_t h;
    ME_CUDA(cudaMemcpyAsync(&h, out, 8, cudaMemcpyDeviceToHost, ctx->stream));
    if ((s = sync(ctx))) return s;
    *out_sad_q4 = uint32_t(h);
    return ok();
}

me_status me_b200_sad_shape(me_ctx* ctx, int W, int H, const uint8_t* cur_alpha,
                            const uint8_t* ref_alpha, int x0, int y0, int size, int dx, int dy,
                            int64_t* out_sad) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if ((dx & 1) || (dy & 1))  // metrics.cpp:67-68
        return me_fail(ME_ERR_INVALID_ARGUMENT, "shape SAD requires an integer-pel vector");
    if ((s = check_rect(W, H, x0, y0, size))) return s;
    if (size > 64) return me_fail(ME_ERR_INVALID_ARGUMENT, "block size above 64");
    if (!cur_alpha || !ref_alpha || !out_sad) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const uint8_t* host[2] = {cur_alpha, ref_alpha};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    int64_t* out = static_cast<int64_t*>(ctx->aux.p);
    ME_CUDA(mek::sad_shape_single(dev[0], dev[1], W, H, x0, y0, size, dx, dy, out, ctx->stream));
    ME_CUDA(cudaMemcpyAsync(out_sad, out, 8, cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    return s ? s : ok();
}

me_status me_b200_classify_blocks(me_ctx* ctx, int W, int H, const uint8_t* alpha, int bs,
                                  uint8_t* types) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (bs <= 0 || W <= 0 || H <= 0 || W % bs || H % bs)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "block size does not divide the frame");
    if (bs % 4 || W % 4) return me_fail(ME_ERR_INVALID_ARGUMENT, "block size must be a multiple of 4");
    if (!types) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const size_t n = size_t(W / bs) * (H / bs);
    if (!alpha) {
        std::memset(types, ME_OPAQUE, n);  // classify_block(nullptr) == Opaque (frame.cpp:82)
        return ok();
    }
    const uint8_t* host[1] = {alpha};
    const uint8_t* dev[1];
    if ((s = stage_planes(ctx, size_t(W) * H, host, dev, 1))) return s;
    ME_CUDA(ctx->aux.reserve(n + 256));
    ME_CUDA(mek::classify_frame(dev[0], W, H, bs, static_cast<uint8_t*>(ctx->aux.p), ctx->stream));
    ME_CUDA(cudaMemcpyAsync(types, ctx->aux.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    return s ? s : ok();
}

me_status me_b200_binarize(me_ctx* ctx, int W, int H, const uint8_t* gray, int threshold,
                           uint8_t* out) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (W < 0 || H < 0 || !gray || !out) return me_fail(ME_ERR_INVALID_ARGUMENT, "bad arguments");
    const size_t n = size_t(W) * H;
    if (n == 0) return ok();
    const uint8_t* host[1] = {gray};
    const uint8_t* dev[1];
    if ((s = stage_planes(ctx, n, host, dev, 1))) return s;
    ME_CUDA(ctx->aux.reserve(n + 256));
    ME_CUDA(mek::binarize(dev[0], int(n), threshold, static_cast<uint8_t*>(ctx->aux.p), ctx->stream));
    ME_CUDA(cudaMemcpyAsync(out, ctx->aux.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    return s ? s : ok();
}

me_status me_b200_predict_frame(me_ctx* ctx, int W, int H, const uint8_t* ref, const int32_t* mv,
                                const uint8_t* types, int bs, const uint8_t* cur, uint8_t* pred,
                                int64_t* out_sse) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (bs != 8 && bs != 16) return me_fail(ME_ERR_INVALID_ARGUMENT, "block_size must be 8 or 16");
    if (W <= 0 || H <= 0 || W % bs || H % bs)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "motion field grid does not cover the frame");
    if (!ref || !mv) return me_fail(ME_ERR_INVALID_ARGUMENT, "null buffer");
    const size_t plane = size_t(W) * H;
    const size_t nb = size_t(W / bs) * (H / bs);
    const uint8_t* host[2] = {ref, cur};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, plane, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(nb * 9 + sizeof(me_pair_stats) + 512));
    uint8_t* aux = static_cast<uint8_t*>(ctx->aux.p);
    me_pair_stats* st = reinterpret_cast<me_pair_stats*>(aux);
    int32_t* mv_dev = reinterpret_cast<int32_t*>(aux + 256);
    uint8_t* types_dev = types ? aux + 256 + nb * 8 : nullptr;
    ME_CUDA(cudaMemsetAsync(st, 0, sizeof(me_pair_stats), ctx->stream));
    ME_CUDA(cudaMemcpyAsync(mv_dev, mv, nb * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (types) ME_CUDA(cudaMemcpyAsync(types_dev, types, nb, cudaMemcpyHostToDevice, ctx->stream));
    ME_CUDA(ctx->out_pred.reserve(plane + 256));
    ME_CUDA(mek::predict(dev[0], dev[1], mv_dev, types_dev, W, H, bs,
                         static_cast<uint8_t*>(ctx->out_pred.p), st, ctx->stream));
    if (pred)
        ME_CUDA(cudaMemcpyAsync(pred, ctx->out_pred.p, plane, cudaMemcpyDeviceToHost, ctx->stream));
    me_pair_stats hs;
    ME_CUDA(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, ctx->stream));
    if ((s = sync(ctx))) return s;
    if (out_sse) *out_sse = cur ? hs.sse : 0;
    return ok();
}

me_status me_b200_sse(me_ctx* ctx, int W, int H, const uint8_t* a, const uint8_t* b,
                      int64_t* out_sse) {
    me_status s = check_ctx(ctx);
    if (s) return s;
    if (W <= 0 || H <= 0 || !a || !b || !out_sse)
        return me_fail(ME_ERR_INVALID_ARGUMENT, "bad arguments");
    const size_t n = size_t(W) * H;
    const uint8_t* host[2] = {a, b};
    const uint8_t* dev[2];
    if ((s = stage_planes(ctx, n, host, dev, 2))) return s;
    ME_CUDA(ctx->aux.reserve(256));
    unsigned long long* out = static_cast<unsigned long long*>(ctx->aux.p);
    ME_CUDA(cudaMemsetAsync(out, 0, 8, ctx->stream));
    ME_CUDA(mek::sse(dev[0], dev[1], int(n), out, ctx->stream));
    ME_CUDA(cudaMemcpyAsync(out_sse, out, 8, cudaMemcpyDeviceToHost, ctx->stream));
    s = sync(ctx);
    return s ? s : ok();
}

}  // extern "C"
