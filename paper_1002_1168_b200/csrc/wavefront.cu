// wavefront.cu — classify_block on every block (fused transparent-block SSE
// and the per-pair type counts), the per-step histogram, its scan and the
// scatter that builds the wavefront-ordered work list.
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
// classify_kernel: classify_block (frame.cpp:81-104) on every block of every
// pair's CURRENT alpha plane (estimators.cpp:411), initialise its record
// (transparent: final all-zero record; estimated: MV = sentinel) and build the
// histogram of estimated blocks over the sort key (PA: wavefront step
// t = h + 2v + p; baselines: a single bin).
// ---------------------------------------------------------------------------

// Programmatic dependent launch along classify -> scan -> fill -> PA head:
// every kernel allows its successor to launch on entry; a successor waits for
// its predecessor's completion (and memory) before reading anything.  Both
// instructions are no-ops for kernels launched in plain stream order.
__device__ __forceinline__ void pdl_allow_next() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_prev() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// SSE of a block predicted with the zero vector (transparent blocks,
// compensation.cpp:45): cur block vs the co-located ref block.
__device__ __forceinline__ uint32_t block_sse0(const uint8_t* cur, const uint8_t* ref, int W,
                                               int x0, int y0, int bs) {
    uint32_t s = 0;
    for (int y = 0; y < bs; ++y) {
        const size_t o = size_t(y0 + y) * W + x0;
        for (int i = 0; i < bs; i += 8) {
            const uint2 c = __ldg(reinterpret_cast<const uint2*>(cur + o + i));
            const uint2 r = __ldg(reinterpret_cast<const uint2*>(ref + o + i));
            s = sq4(c.x, r.x, s);
            s = sq4(c.y, r.y, s);
        }
    }
    return s;
}

// One thread classifies a 16-pixel-wide column strip of one block row (two
// 8x8 blocks or one 16x16 block): every alpha, cur and ref row of the strip is
// fetched with 16-byte loads in a single round (the luma is loaded
// speculatively — it is only needed for transparent blocks' zero-vector SSE,
// and is the compulsory read of those frames anyway).
template <int BS, bool BITS>
__global__ void __launch_bounds__(256) classify_kernel(ClassArgs a) {
    extern __shared__ int s_hist[];
    pdl_allow_next();
    constexpr int NB = 16 / BS;  // blocks per strip
    const Batch& b = a.b;
    if (!a.hist2)
        for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const int strips = b.cols / NB;  // strips per block row
    const int64_t n = int64_t(b.n_seq) * b.pairs * b.rows * strips;
    const size_t plane = size_t(b.W) * b.H;
    const int lane = threadIdx.x & 31;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // uniform trip count so whole warps reach the warp-level reductions
    for (int64_t s0 = int64_t(blockIdx.x) * blockDim.x; s0 < n; s0 += stride) {
        const int64_t si = s0 + threadIdx.x;
        uint32_t sse = 0, n_t = 0, n_o = 0, n_b = 0;
        int64_t gp = -1;
        int hkey[NB];
        uint2 dent[NB];  // direct list entries (single-bin searches)
        bool dval[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            hkey[k] = -1;
            dval[k] = false;
            dent[k] = make_uint2(0u, 0u);
        }
        if (si < n) {
            const int hs = int(si % strips);
            int64_t t = si / strips;
            const int v = int(t % b.rows);
            gp = t / b.rows;  // seq * pairs + p
            const int p = int(gp % b.pairs);
            const int seq = int(gp / b.pairs);
            if (!b.in_band(v)) {  // outside the row band: not this call's work
#pragma unroll
                for (int k = 0; k < NB; ++k) a.types[(gp * b.rows + v) * b.cols + hs * NB + k] = uint8_t(ME_TRANSPARENT);
                gp = -1;
                goto next;
            }
            {
            const size_t fcur = size_t(seq) * b.F + p + b.d, fref = size_t(seq) * b.F + p;
            const size_t off = size_t(v * BS) * b.W + size_t(hs) * 16;
            const uint8_t* ac = b.alpha ? b.alpha + fcur * plane + off : nullptr;
            // bit-packed masks: the strip's 16 pels of a row are 2 bytes
            const uint8_t* abits = BITS ? b.alpha_bits + (fcur * plane + off) / 8 : nullptr;
            const uint8_t* cc = b.luma + fcur * plane + off;
            const uint8_t* rc = b.luma + fref * plane + off;
            int ty_[NB];
            uint32_t s_[NB];
            {
            uint4 al[BS], cu[BS], re[BS];
            uint32_t ab[BS];  // bit rows (all loads of the strip are issued before any is used)
#pragma unroll
            for (int y = 0; y < BS; ++y) {
                if (BITS)
                    ab[y] = __ldg(reinterpret_cast<const uint16_t*>(abits + size_t(y) * (b.W / 8)));
                else
                    al[y] = ac ? __ldg(reinterpret_cast<const uint4*>(ac + size_t(y) * b.W)) : make_uint4(~0u, ~0u, ~0u, ~0u);
                if (a.stats) {
                    cu[y] = __ldg(reinterpret_cast<const uint4*>(cc + size_t(y) * b.W));
                    re[y] = __ldg(reinterpret_cast<const uint4*>(rc + size_t(y) * b.W));
                }
            }
            if (BITS) {
#pragma unroll
                for (int y = 0; y < BS; ++y)
                    al[y] = make_uint4(mask_expand4(ab[y] & 15u), mask_expand4((ab[y] >> 4) & 15u),
                                       mask_expand4((ab[y] >> 8) & 15u), mask_expand4(ab[y] >> 12));
            }
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                // classify_block (frame.cpp:81-104): any sample set / all set
                uint32_t any = 0, nz = 1, s = 0;
#pragma unroll
                for (int y = 0; y < BS; ++y) {
                    const uint32_t w0 = NB == 2 ? (k ? al[y].z : al[y].x) : al[y].x;
                    const uint32_t w1 = NB == 2 ? (k ? al[y].w : al[y].y) : al[y].y;
                    any |= w0 | w1;
                    nz &= (__vcmpeq4(w0, 0u) | __vcmpeq4(w1, 0u)) == 0u;
                    if (NB == 1) {
                        any |= al[y].z | al[y].w;
                        nz &= (__vcmpeq4(al[y].z, 0u) | __vcmpeq4(al[y].w, 0u)) == 0u;
                    }
                    if (a.stats) {
                        if (NB == 2) {
                            s = sq4(k ? cu[y].z : cu[y].x, k ? re[y].z : re[y].x, s);
                            s = sq4(k ? cu[y].w : cu[y].y, k ? re[y].w : re[y].y, s);
                        } else {
                            s = sq4(cu[y].x, re[y].x, s);
                            s = sq4(cu[y].y, re[y].y, s);
                            s = sq4(cu[y].z, re[y].z, s);
                            s = sq4(cu[y].w, re[y].w, s);
                        }
                    }
                }
                ty_[k] = !any ? ME_TRANSPARENT : (nz ? ME_OPAQUE : ME_BOUNDARY);
                s_[k] = s;
            }
            }
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const int ty = ty_[k];
                const uint32_t s = s_[k];
                const int h = hs * NB + k;
                const int64_t g = (gp * b.rows + v) * b.cols + h;
                a.types[g] = uint8_t(ty);
                uint4 r;
                r.x = ty == ME_TRANSPARENT ? 0u : kSentinel;
                r.y = 0u;
                r.z = 0u;
                r.w = uint32_t(ty) << 8;
                *reinterpret_cast<uint4*>(a.recs + g) = r;
                if (ty != ME_TRANSPARENT) {
                    if (a.list_direct) {  // appended below (any order: the blocks are independent)
                        dval[k] = true;
                        dent[k] = make_uint2(uint32_t(h) | (uint32_t(v) << 16) | (ty == ME_BOUNDARY ? kBoundaryBit : 0u),
                                             uint32_t(p) | (uint32_t(seq) << 16));
                    } else if (a.hist2)  // aligned keys: per (sequence, step) counts, added below
                        hkey[k] = seq * a.nbins + (h + 2 * v + p);
                    else
                        atomicAdd(&s_hist[a.pa ? a.key_a * (h + 2 * v + p) + a.key_s * seq : 0], 1);
                    n_o += ty == ME_OPAQUE;
                    n_b += ty == ME_BOUNDARY;
                } else {
                    sse += s;
                    n_t += 1;
                }
            }
            }
        }
    next:
        if (a.list_direct && a.es_runs && NB == 1) {
            // runs of 4 / 2 horizontally adjacent estimated blocks (aligned lane
            // quads / pairs of the warp's consecutive strips in one block row),
            // else single blocks: the entry's first block, count in bits 12-14
            const unsigned E = __ballot_sync(0xFFFFFFFFu, dval[0]);
            const uint32_t hx = dent[0].x & 0xFFFu;
            const unsigned long long rid = (static_cast<unsigned long long>(dent[0].y) << 16) | ((dent[0].x >> 16) & 0x7FFFu);
            const unsigned long long rid_n = __shfl_down_sync(0xFFFFFFFFu, rid, 1);
            const uint32_t hx_n = __shfl_down_sync(0xFFFFFFFFu, hx, 1);
            const unsigned N = __ballot_sync(0xFFFFFFFFu, lane < 31 && dval[0] && rid_n == rid && hx_n == hx + 1);
            const bool q4 = (lane & 3) == 0 && ((E >> lane) & 0xFu) == 0xFu && ((N >> lane) & 0x7u) == 0x7u;
            const unsigned Q = __ballot_sync(0xFFFFFFFFu, q4);
            const bool inq = (Q >> (lane & ~3)) & 1u;
            const bool p2 = !inq && (lane & 1) == 0 && ((E >> lane) & 3u) == 3u && ((N >> lane) & 1u);
            const unsigned P = __ballot_sync(0xFFFFFFFFu, p2);
            const bool inp = (P >> (lane & ~1)) & 1u;
            const uint32_t cnt = q4 ? 4u : p2 ? 2u : (dval[0] && !inq && !inp) ? 1u : 0u;
            dval[0] = cnt != 0;
            dent[0].x = hx | (cnt << 12) | (dent[0].x & 0x7FFF0000u);
        }
        if (a.list_direct) {  // one list append per warp and block slot
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const unsigned m = __ballot_sync(0xFFFFFFFFu, dval[k]);
                if (m) {
                    const int leader = __ffs(m) - 1;
                    int base = 0;
                    if (lane == leader) base = atomicAdd(a.nlist_direct, __popc(m));
                    base = __shfl_sync(0xFFFFFFFFu, base, leader);
                    if (dval[k]) a.list_direct[base + __popc(m & ((1u << lane) - 1u))] = dent[k];
                }
            }
        }
        if (a.hist2) {  // one atomic per distinct (sequence, step) of the warp, and the sequences' first steps
            int tm = 0x7FFFFFFF, sq = -1;
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const unsigned m = __match_any_sync(0xFFFFFFFFu, hkey[k]);
                if (hkey[k] >= 0 && lane == __ffs(m) - 1) atomicAdd(&a.hist2[hkey[k]], __popc(m));
                if (hkey[k] >= 0) {
                    sq = hkey[k] / a.nbins;
                    tm = min(tm, hkey[k] - sq * a.nbins);
                }
            }
            const unsigned ms = __match_any_sync(0xFFFFFFFFu, sq);
            tm = __reduce_min_sync(ms, tm);
            if (sq >= 0 && lane == __ffs(ms) - 1) atomicMin(a.tmin_g + sq, tm);
        }
        if (a.stats) {
            const int64_t gp0 = __shfl_sync(0xFFFFFFFFu, gp, 0);
            const bool uniform = __all_sync(0xFFFFFFFFu, gp == gp0 || gp < 0);
            if (!a.pa) n_o = n_b = 0;  // the other searches count their own blocks
            if (uniform) {
                const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, sse);
                const uint32_t wn = __reduce_add_sync(0xFFFFFFFFu, n_t);
                const uint32_t wo = __reduce_add_sync(0xFFFFFFFFu, n_o);
                const uint32_t wb = __reduce_add_sync(0xFFFFFFFFu, n_b);
                if (lane == 0) {
                    unsigned long long* st = reinterpret_cast<unsigned long long*>(a.stats + gp0);
                    if (ws) red_add_u64(st + 5, ws);
                    if (wn) red_add_u64(st + 4, wn);
                    if (wo) red_add_u64(st + 2, wo);
                    if (wb) red_add_u64(st + 3, wb);
                    if (wo + wb) red_add_u64(st + 0, 4ull * (wo + wb));  // brs_select: 4 per block (:290)
                }
            } else if (gp >= 0) {
                unsigned long long* st = reinterpret_cast<unsigned long long*>(a.stats + gp);
                if (sse) red_add_u64(st + 5, sse);
                if (n_t) red_add_u64(st + 4, n_t);
                if (n_o) red_add_u64(st + 2, n_o);
                if (n_b) red_add_u64(st + 3, n_b);
                if (n_o + n_b) red_add_u64(st + 0, 4ull * (n_o + n_b));
            }
        }
    }
    if (a.hist2 || a.list_direct) return;
    __syncthreads();
    for (int i = threadIdx.x; i < a.nbins; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&a.hist[i], s_hist[i]);
}

// Exclusive scan of hist into offs[0..nbins] (single CTA), cursor = offs.
// ranges (optional): the list split at the first and after the last step
// holding >= wide blocks: {0, b1}, {b1, b2}, {b2, total} (narrow, wide, narrow).
// Aligned keys (hist2 non-null): a warp per sequence finds its first step
// holding an estimated block (tmin) and adds its step counts, shifted down by
// tmin, into the key histogram (shared memory) that the scan then reads.
__global__ void scan_kernel(const int* hist, int nbins, int pad, int* offs, int* cursor,
                            uint2* list, int wide, int* ranges, const int* hist2, int n_seq, int* tmin) {
    pdl_wait_prev();
    pdl_allow_next();
    __shared__ int s_part[1024];
    __shared__ int s_lo, s_hi;  // first / last wide step
    extern __shared__ int s_keyhist[];
    const int T = blockDim.x;
    if (hist2) {
        // two passes over hist2 with every thread's loads independent (the
        // per-sequence warp loop was a chain of dependent L2 round trips)
        int* s_tmin = s_keyhist + nbins;
        for (int i = threadIdx.x; i < nbins; i += T) s_keyhist[i] = 0;
        for (int i = threadIdx.x; i < n_seq; i += T) {
            const int t0 = tmin[i];  // classify's atomicMin (0x7F7F7F7F: no estimated block)
            s_tmin[i] = t0 < nbins ? t0 : 0;
            tmin[i] = s_tmin[i];
        }
        __syncthreads();
        const int total = n_seq * nbins;
        constexpr int CH = 16;  // independent loads in flight per thread
        for (int i0 = threadIdx.x; i0 < total; i0 += T * CH) {
            int x[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) x[j] = i0 + j * T < total ? __ldcg(hist2 + i0 + j * T) : 0;
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                if (!x[j]) continue;
                const int i = i0 + j * T, sq = i / nbins;
                atomicAdd(&s_keyhist[i - sq * nbins - s_tmin[sq]], x[j]);
            }
        }
        __syncthreads();
        hist = s_keyhist;
    }
    const int per = (nbins + T - 1) / T;
    const int lo = threadIdx.x * per, hi = min(lo + per, nbins);
    auto padded = [&](int v) { return (v + pad - 1) / pad * pad; };
    if (threadIdx.x == 0) {
        s_lo = nbins;
        s_hi = -1;
    }
    __syncthreads();
    int sum = 0, my_lo = nbins, my_hi = -1;
    for (int i = lo; i < hi; ++i) {
        sum += padded(hist[i]);
        if (hist[i] >= wide) {
            my_lo = min(my_lo, i);
            my_hi = max(my_hi, i);
        }
    }
    if (ranges && my_hi >= 0) {
        atomicMin(&s_lo, my_lo);
        atomicMax(&s_hi, my_hi);
    }
    // exclusive block scan of the per-thread sums: warp scans, then a scan of
    // the warp totals (no serial loop over the 1024 partials)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = T >> 5;
        int w = lane < nw ? s_part[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= o) wi += y;
        }
        s_part[32 + lane] = wi - w;  // exclusive warp offsets
        if (lane == 31) offs[nbins] = wi;
    }
    __syncthreads();
    int acc = s_part[32 + wid] + incl - sum;
    for (int i = lo; i < hi; ++i) {
        offs[i] = acc;
        cursor[i * kCursorStride] = acc;
        for (int k = hist[i]; k < padded(hist[i]); ++k) list[acc + k] = make_uint2(kInvalidEntry, kInvalidEntry);
        acc += padded(hist[i]);
    }
    if (ranges) {
        __syncthreads();  // offs[] complete
        if (threadIdx.x == 0) {
            const int total = offs[nbins];
            const int b1 = s_hi >= 0 ? offs[s_lo] : total, b2 = s_hi >= 0 ? offs[s_hi + 1] : total;
            ranges[0] = 0;
            ranges[1] = b1;
            ranges[2] = b1;
            ranges[3] = b2;
            ranges[4] = b2;
            ranges[5] = total;
        }
    }
}

// Scatter estimated blocks into key order as decoded list entries
// {h | v << 16 | boundary << 31, p | seq << 16} (per-CTA ranges per bin keep
// the global atomics to one per (CTA, bin)).
// One CTA per rows_per_cta block rows (32-bit index math): count into a shared
// histogram, reserve each bin's range with one global atomic per (CTA, bin),
// then scatter.

__global__ void __launch_bounds__(256) fill_kernel(ClassArgs a, int* cursor, uint2* list, uint32_t rows_per_cta) {
    pdl_wait_prev();
    pdl_allow_next();
    extern __shared__ int s_cnt[];  // [nbins] counts, then [nbins] bases
    int* s_base = s_cnt + a.nbins;
    const Batch& b = a.b;
    for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const uint32_t nrows = uint32_t(b.n_seq) * uint32_t(b.pairs) * uint32_t(b.rows);
    const uint32_t r0 = blockIdx.x * rows_per_cta, r1 = min(r0 + rows_per_cta, nrows);
    const uint32_t cols = uint32_t(b.cols), items = (r1 - r0) * cols;
    const uint8_t* types = a.types + size_t(r0) * cols;
    for (int pass = 0; pass < 2; ++pass) {
        for (uint32_t i = threadIdx.x; i < items; i += blockDim.x) {
            const int ty = types[i];
            if (ty == ME_TRANSPARENT) continue;
            const uint32_t r = r0 + i / cols, h = i - (i / cols) * cols;
            const uint32_t pr = r / uint32_t(b.rows), v = r - pr * uint32_t(b.rows);
            const uint32_t seq = pr / uint32_t(b.pairs), p = pr - seq * uint32_t(b.pairs);
            {
                const int key = !a.pa ? 0 : a.tmin ? int(h + 2 * v + p) - a.tmin[seq] : a.key_a * int(h + 2 * v + p) + a.key_s * int(seq);
                if (pass == 0) {
                    atomicAdd(&s_cnt[key], 1);
                } else {
                    const int pos = s_base[key] + atomicAdd(&s_cnt[key], 1);
                    list[pos] = make_uint2(uint32_t(h) | (v << 16) | (ty == ME_BOUNDARY ? kBoundaryBit : 0u), p | (seq << 16));
                }
            }
        }
        __syncthreads();
        if (pass == 0) {
            for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) {
                s_base[i] = s_cnt[i] ? atomicAdd(&cursor[i * kCursorStride], s_cnt[i]) : 0;
                s_cnt[i] = 0;
            }
            __syncthreads();
        }
    }
}

// fill_rows_kernel: the same scatter with a thread per block row (sequence,
// pair, row decoded once per row instead of per block; a row's blocks go to
// consecutive bins, so the shared-memory counters see fewer collisions).
__global__ void __launch_bounds__(256) fill_rows_kernel(ClassArgs a, int* cursor, uint2* list) {
    pdl_wait_prev();
    pdl_allow_next();
    extern __shared__ int s_cnt[];  // [nbins] counts, then [nbins] bases
    int* s_base = s_cnt + a.nbins;
    const Batch& b = a.b;
    for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const uint32_t nrows = uint32_t(b.n_seq) * uint32_t(b.pairs) * uint32_t(b.rows);
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t cols = uint32_t(b.cols);
    const bool live = r < nrows;
    uint32_t v = 0, p = 0, seq = 0;
    if (live) {
        const uint32_t pr = r / uint32_t(b.rows);
        v = r - pr * uint32_t(b.rows);
        seq = pr / uint32_t(b.pairs);
        p = pr - seq * uint32_t(b.pairs);
    }
    const uint8_t* types = a.types + size_t(r) * cols;
    const int key0 = !a.pa ? 0 : a.tmin ? (live ? int(2 * v + p) - a.tmin[seq] : 0) : a.key_a * int(2 * v + p) + a.key_s * int(seq);
    const int kstep = a.pa ? (a.tmin ? 1 : a.key_a) : 0;
    // rows of a multiple of 4 blocks (cfg4: 44) are read as words, and a word
    // of four transparent blocks (ME_TRANSPARENT = 0: most of them) is skipped whole
    const bool words = (cols & 3u) == 0;
    for (int pass = 0; pass < 2; ++pass) {
        if (live) {
            auto visit = [&](uint32_t h, int ty) {
                const int key = key0 + int(h) * kstep;
                if (pass == 0) {
                    atomicAdd(&s_cnt[key], 1);
                } else {
                    const int pos = s_base[key] + atomicAdd(&s_cnt[key], 1);
                    list[pos] = make_uint2(h | (v << 16) | (ty == ME_BOUNDARY ? kBoundaryBit : 0u), p | (seq << 16));
                }
            };
            if (words) {
                const uint32_t* t32 = reinterpret_cast<const uint32_t*>(types);
                for (uint32_t w = 0; w < (cols >> 2); ++w) {
                    const uint32_t t4 = t32[w];
                    if (t4 == 0u) continue;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int ty = int((t4 >> (8 * j)) & 0xFFu);
                        if (ty != ME_TRANSPARENT) visit(4 * w + j, ty);
                    }
                }
            } else {
                for (uint32_t h = 0; h < cols; ++h) {
                    const int ty = types[h];
                    if (ty != ME_TRANSPARENT) visit(h, ty);
                }
            }
        }
        __syncthreads();
        if (pass == 0) {
            for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) {
                s_base[i] = s_cnt[i] ? atomicAdd(&cursor[i * kCursorStride], s_cnt[i]) : 0;
                s_cnt[i] = 0;
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------


static cudaLaunchConfig_t pdl_config(dim3 grid, dim3 block, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    return lc;
}

static void pdl_attr(cudaLaunchConfig_t& lc, cudaLaunchAttribute* at) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
}

cudaError_t launch_classify(const ClassArgs& ca, int num_sms, cudaStream_t st) {
    const Batch& b = ca.b;
    const int threads = 256;
    // a 16-pixel strip per thread: two 8x8 blocks or one 16x16 block (W % 16 == 0)
    const int64_t strips = b.nblocks() / (16 / b.bs);
    int grid = int(std::min<int64_t>((strips + threads - 1) / threads, int64_t(num_sms) * 8));
    if (grid < 1) grid = 1;
    const size_t hist_smem = ca.hist2 ? 0 : size_t(ca.nbins) * 4;
    const bool bits = b.alpha_bits != nullptr;
    if (b.bs == 8)
        (bits ? classify_kernel<8, true> : classify_kernel<8, false>)<<<grid, threads, hist_smem, st>>>(ca);
    else
        (bits ? classify_kernel<16, true> : classify_kernel<16, false>)<<<grid, threads, hist_smem, st>>>(ca);
    return cudaGetLastError();
}

cudaError_t launch_scan(const int* hist, int nbins, int pad, int* offs, int* cursor, uint2* list,
                        int wide, int* ranges, cudaStream_t st, bool pdl, const int* hist2, int n_seq,
                        int* tmin) {
    const size_t smem = hist2 ? size_t(nbins + n_seq) * 4 : 0;
    cudaError_t e;
    if (smem > 40 * 1024 &&
        (e = cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))))
        return e;
    if (pdl) {
        cudaLaunchConfig_t lc = pdl_config(dim3(1), dim3(1024), smem, st);
        cudaLaunchAttribute at[1];
        pdl_attr(lc, at);
        return cudaLaunchKernelEx(&lc, scan_kernel, hist, nbins, pad, offs, cursor, list, wide, ranges, hist2,
                                  n_seq, tmin);
    }
    scan_kernel<<<1, 1024, smem, st>>>(hist, nbins, pad, offs, cursor, list, wide, ranges, hist2, n_seq, tmin);
    return cudaGetLastError();
}

cudaError_t launch_fill(const ClassArgs& ca, int* cursor, uint2* list, int num_sms, cudaStream_t st,
                        const Tuning& t) {
    const Batch& b = ca.b;
    // <= 64 rows per CTA, >= 2 CTAs per SM
    const int64_t nrows = int64_t(b.n_seq) * b.pairs * b.rows;
    const int64_t rmax = t.fill_rows_per_cta;  // measured: 64 <= 32, 128 < 256
    const int64_t rpc = std::max<int64_t>(4, std::min<int64_t>(rmax, nrows / (2 * num_sms)));
    const int grid = int((nrows + rpc - 1) / rpc);
    const size_t smem = 2 * size_t(ca.nbins) * 4;
    cudaError_t e;
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))))
        return e;
    // large batches: a thread per block row (measured 60 -> 31 us on cfg4);
    // few rows (single sequences) keep the per-block kernel's parallelism
    if (t.fill_rows ? t.fill_rows > 0 : nrows >= int64_t(num_sms) * 64) {
        if (smem > 48 * 1024 &&
            (e = cudaFuncSetAttribute(fill_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))))
            return e;
        if (t.sort_pdl) {
            cudaLaunchConfig_t lc = pdl_config(dim3(unsigned((nrows + 255) / 256)), dim3(256), smem, st);
            cudaLaunchAttribute at[1];
            pdl_attr(lc, at);
            return cudaLaunchKernelEx(&lc, fill_rows_kernel, ca, cursor, list);
        }
        fill_rows_kernel<<<int((nrows + 255) / 256), 256, smem, st>>>(ca, cursor, list);
        return cudaGetLastError();
    }
    fill_kernel<<<grid, 256, smem, st>>>(ca, cursor, list, uint32_t(rpc));
    return cudaGetLastError();
}

}  // namespace mek
