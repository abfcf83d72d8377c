// es.cu — full_search (estimators.cpp:167-187): the batched kernel over the
// work list and the single-block kernel behind the per-block entry point.
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
// es_kernel: full_search (estimators.cpp:167-187).  One CTA per estimated
// block (persistent CTAs pull blocks from the work list).  The reference
// window (clipped, pel units, estimators.cpp:62-65) is staged in shared memory
// as 4 copies pre-shifted by 0..3 bytes so every candidate row is read as
// aligned 32-bit words; the current block lives in registers.  A thread owns
// one dx column and a run of K consecutive dy: each staged reference row is
// loaded once and reused for every accumulator whose current row it pairs
// with.  The winner is the minimum packed key (SAD, |dx|+|dy|, raster index)
// — exactly the reference's strict-< scan with the Manhattan tie-break.
// ---------------------------------------------------------------------------

struct EsArgs {
    Batch b;
    int S;
    const uint2* list;
    const int* nlist;  // device count (offs[nbins])
    int* counter;
    me_block_rec* recs;
    int band_rows_max;  // staged rows per band (multiple of K, + BS - 1 added on top)
    me_pair_stats* stats;
    int region_words;   // shared memory per block group (NB > 1)
    const uint8_t* types;  // run mode: the blocks' types (records)
};

constexpr int kEsThreads = 256;
constexpr uint32_t kEsDead = 0xF0000000u;  // key bits of rows past the window (> any real key: SAD << 12 < 2^28)

// One task: window column col (its staged copy and word offset folded into
// `base`) x K consecutive dy.  Each staged row is loaded once and feeds every
// accumulator whose current row it pairs with.  Returns the minimum over the
// K positions of the 32-bit key (SAD << 12 | (|dx| + |dy|) << 3 | k): SAD <
// 2^16, |dx| + |dy| <= 2S < 512 for S <= 255, k < 8; rows past the window
// carry kEsDead (rkey), so the key is two IMADs (FMA pipe) and a VIMNMX.
template <int BS, int K, int PWC>
__device__ __forceinline__ uint32_t es_task(const uint32_t (&c)[BS][BS / 4], const uint32_t* base, int PW_rt,
                                            const uint32_t* rk, uint32_t adx8) {
    constexpr int NW = BS / 4;
    const int PW = PWC ? PWC : PW_rt;
    uint32_t acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0;
#pragma unroll
    for (int j = 0; j < K + BS - 1; ++j) {
        uint32_t w[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = base[j * PW + i];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int r = j - k;
            if (r >= 0 && r < BS) {
#pragma unroll
                for (int i = 0; i < NW; ++i) acc[k] = vad4(c[r][i], w[i], acc[k]);
            }
        }
    }
    uint32_t m32 = ~0u;
#pragma unroll
    for (int k = 0; k < K; ++k) m32 = min(m32, acc[k] * 4096u + (rk[k] + adx8));
    return m32;
}

// PWC: the staged row stride in words when known at compile time (the
// launcher instantiates the common search ranges; every row offset in the SAD
// loop is then an immediate), 0 = computed from the clipped window.
// The CTA's threads may form several groups, each searching its own block in
// its own shared-memory region (small windows: NB blocks per CTA pass, see
// es_kernel): tid / T = this thread's index / size within its group; every
// group passes the same CTA barriers (one band per block when NB > 1).
// Runs of horizontally adjacent blocks (es_kernel's run mode) share ONE staged
// window, the union of theirs: ux0 >= 0 is its first frame column and
// urowbytes its width; it is staged by all the CTA's threads (stid of sT) and
// each group reads its block's positions at their byte offset in it.
template <int BS, int K, int PWC = 0>
__device__ void es_block(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                         int S, int band_runs_max, uint32_t* sm, unsigned long long* s_best,
                         int& out_dx, int& out_dy, uint32_t& out_sad, uint32_t& out_cmp,
                         int tid = threadIdx.x, int T = kEsThreads, int ux0 = -1, int urowbytes = 0) {
    const int lane = tid & 31, wid = tid >> 5;
    const int lo_x = max(-S, -x0), hi_x = min(S, W - x0 - BS);
    const int lo_y = max(-S, -y0), hi_y = min(S, H - y0 - BS);
    const int WX = hi_x - lo_x + 1, WY = hi_y - lo_y + 1;
    const int nruns = (WY + K - 1) / K;
    const bool uni = ux0 >= 0;
    const int rowbytes = uni ? urowbytes : WX + BS - 1;
    const int coff = uni ? x0 + lo_x - ux0 : 0;  // this block's window start in the staged rows (bytes)
    const int stid = uni ? int(threadIdx.x) : tid, sT = uni ? kEsThreads : T;  // who stages
    const int PW = PWC ? PWC : ((rowbytes - BS) >> 2) + (BS >> 2) + 1;  // words per staged row (>= the window's)
    constexpr int NW = BS / 4;

    uint32_t c[BS][NW];
    if (((x0 | W) & 3) == 0) {
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int i = 0; i < NW; ++i) c[r][i] = ldg32(cur + size_t(y0 + r) * W + x0 + 4 * i);
    } else {
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                const uint8_t* q = cur + size_t(y0 + r) * W + x0 + 4 * i;
                c[r][i] = uint32_t(q[0]) | (uint32_t(q[1]) << 8) | (uint32_t(q[2]) << 16) |
                          (uint32_t(q[3]) << 24);
            }
    }

    unsigned long long best = ~0ull;
    for (int run0 = 0; run0 < nruns; run0 += band_runs_max) {
        const int bruns = min(band_runs_max, nruns - run0);
        const int srows = bruns * K + BS - 1;
        // (run mode, one band: a window of 8n + 1 rows ends in a one-row run,
        // so only WY + BS - 1 rows are ever read)
        const bool last1 = run0 + bruns == nruns && WY - (nruns - 1) * K == 1;
        int CW = (uni && last1 ? WY + BS - 1 : srows) * PW;
        CW += ((8 - (CW & 31)) + 32) & 31;  // copy stride = 8 (mod 32) words: conflict-free lanes
        const int row_g0 = y0 + lo_y + run0 * K;  // frame row of staged row 0
        const int rows_valid = min(srows, WY + BS - 1 - run0 * K);
        // the frame's words (32-bit offsets: a frame is < 4 GB); ref is 4-byte
        // aligned when W % 4 == 0 (checked by the launcher's caller)
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(ref) & ~uintptr_t(3));
        const uint32_t ref_mis = uint32_t(reinterpret_cast<uintptr_t>(ref) & 3);
        const uint32_t seg0 = ref_mis + uint32_t(row_g0) * uint32_t(W) + uint32_t(uni ? ux0 : x0 + lo_x);  // byte offset from rw
        __syncthreads();  // previous band / block done with smem
        // staging from aligned words: copy s, word q = bytes [4q + s, 4q + s + 4)
        // of the row segment = a funnel shift of two aligned words.  Bytes past
        // the segment are never paired with the current block (only rows and
        // columns of admissible positions are summed), so the loads clamp to
        // the segment's last aligned word and rows past the window are skipped.
        // Flat index i = row * PW + q (row by a float reciprocal: exact, since
        // (i + 0.5) / PW is never within 0.5 / PW of an integer).
        {
            const int total = rows_valid * PW;
            const float inv_pw = 1.0f / float(PW);
            uint32_t* const sm1 = sm + CW;
            uint32_t* const sm2 = sm + 2 * CW;
            uint32_t* const sm3 = sm + 3 * CW;
            // U words per thread per round, every load of the round issued
            // before any store (the staging is L2-latency-bound otherwise)
            constexpr int U = 4;
            for (int i0 = stid; i0 < total; i0 += U * sT) {
                uint32_t g[U][3], offs[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = min(i0 + u * sT, total - 1);
                    const int row = __float2int_rz((float(i) + 0.5f) * inv_pw), q = i - row * PW;
                    const uint32_t b0 = seg0 + uint32_t(row) * uint32_t(W);
                    const uint32_t w0 = b0 >> 2, wl = (b0 + uint32_t(rowbytes) - 1) >> 2;
                    offs[u] = b0 & 3u;
                    g[u][0] = __ldg(rw + min(w0 + q, wl));
                    g[u][1] = __ldg(rw + min(w0 + q + 1, wl));
                    g[u][2] = __ldg(rw + min(w0 + q + 2, wl));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * sT;
                    if (i >= total) break;
                    const uint32_t off = offs[u], sh = off * 8, g0 = g[u][0], g1 = g[u][1], g2 = g[u][2];
                    // copies s = 0..3: byte offset off + s within (g0, g1, g2)
                    sm[i] = __funnelshift_r(g0, g1, sh);
                    sm1[i] = off + 1 < 4 ? __funnelshift_r(g0, g1, sh + 8) : g1;
                    sm2[i] = off + 2 < 4 ? __funnelshift_r(g0, g1, sh + 16) : __funnelshift_r(g1, g2, sh - 16);
                    sm3[i] = off == 0 ? __funnelshift_r(g0, g1, 24) : __funnelshift_r(g1, g2, sh - 8);
                }
            }
        }
        // per window row of the band: the key's low bits, (|dy| << 3 | k), or
        // kEsDead for rows past the window, so a position's 32-bit key is two
        // IMADs (FMA pipe) and the VIMNMX — the kernel is ALU-pipe-bound
        // (VABSDIFF4 issues at half rate there)
        uint32_t* const rkey = sm + 4 * CW;
        for (int i = stid; i < bruns * K; i += sT) {
            const int wy = run0 * K + i;
            rkey[i] = wy < WY ? (uint32_t(abs(lo_y + wy)) << 3) | uint32_t(i % K) : kEsDead;
        }
        __syncthreads();
        // tasks (run, col) in raster order: flat index, run by a float
        // reciprocal.  The window's last run usually holds ONE row (WY = 2S + 1
        // = 8n + 1 for interior blocks): its tasks take a K = 1 body instead of
        // summing K - 1 rows past the window.  The K-row tasks that do not fill
        // a whole round of the group's threads are split into K one-row tasks
        // each, queued with the tail run's: the last round then costs a few
        // one-row sums instead of a whole K-row task on a fraction of the threads
        // (config 5: 2064 K-row tasks = 8 rounds + 16).
        const float inv_wx = 1.0f / float(WX);
        const bool tail1 = run0 + bruns == nruns && WY - (nruns - 1) * K == 1;
        const int nfull = (tail1 ? bruns - 1 : bruns) * WX;
        const int F = nfull / T * T, R = nfull - F;  // whole rounds of K-row tasks, leftover K-row tasks
        const int ntasks = F + R * K + (tail1 ? WX : 0);
        auto take = [&](int run, int col, int k, uint32_t m32) {
            if (m32 < kEsDead) {
                const uint32_t wy = uint32_t((run0 + run) * K) + (m32 & 7u);
                const unsigned long long key = (static_cast<unsigned long long>(m32 >> 12) << 40) |
                                               (static_cast<unsigned long long>((m32 >> 3) & 0x1FFu) << 24) |
                                               static_cast<unsigned long long>(wy * uint32_t(WX) + uint32_t(col));
                best = key < best ? key : best;
            }
        };
        for (int ti = tid; ti < ntasks; ti += T) {
            if (ti < F) {
                const int run = __float2int_rz((float(ti) + 0.5f) * inv_wx), col = ti - run * WX;
                const int o = coff + col;
                const uint32_t* base = sm + (o & 3) * CW + (run * K) * PW + (o >> 2);
                take(run, col, 0, es_task<BS, K, PWC>(c, base, PW, rkey + run * K, uint32_t(abs(lo_x + col)) << 3));
            } else {
                // one row k of a leftover K-row task, or of the one-row tail run
                const int j = ti - F;
                int run, col, k;
                if (j < R * K) {
                    const int f = F + j / K;
                    run = __float2int_rz((float(f) + 0.5f) * inv_wx);
                    col = f - run * WX;
                    k = j - (j / K) * K;
                } else {
                    run = bruns - 1;
                    col = j - R * K;
                    k = 0;
                }
                const int o = coff + col;
                const uint32_t* base = sm + (o & 3) * CW + (run * K + k) * PW + (o >> 2);
                take(run, col, k, es_task<BS, 1, PWC>(c, base, PW, rkey + run * K + k, uint32_t(abs(lo_x + col)) << 3));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        best = other < best ? other : best;
    }
    if (lane == 0) s_best[wid] = best;
    __syncthreads();
    if (tid == 0) {
        unsigned long long m = s_best[0];
        for (int i = 1; i < (T >> 5); ++i) m = s_best[i] < m ? s_best[i] : m;
        const int raster = int(m & 0xFFFFFF);
        out_dx = lo_x + raster % WX;
        out_dy = lo_y + raster / WX;
        out_sad = uint32_t(m >> 40);
        out_cmp = uint32_t(WX * WY);
    }
}

// NB > 1 (windows small enough that NB of them fit): the CTA claims NB list
// entries per pass and splits into NB groups of kEsThreads / NB threads, one
// block each, so one staging round trip, barrier and reduction serve NB blocks
// (at S = 16 one block's 165 tasks left 91 of 256 threads idle and the
// per-block staging and barriers dominated).
template <int BS, int K, int PWC, int NB>
__global__ void __launch_bounds__(kEsThreads) es_kernel(EsArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ unsigned long long s_best[kEsThreads / 32];
    __shared__ int s_item;
    __shared__ int s_res[NB][4];
    constexpr int T = kEsThreads / NB;  // threads per group
    const Batch& b = a.b;
    const int n = *a.nlist;
    const size_t plane = size_t(b.W) * b.H;
    const int band_runs = a.band_rows_max / K;
    const int grp = threadIdx.x / T, gtid = threadIdx.x - grp * T;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(a.counter, NB);
        __syncthreads();
        const int item0 = s_item;
        if (item0 >= n) return;
        const int item = item0 + grp;
        const bool live = item < n;  // (an idle group still passes every barrier)
        int h, v, p, seq;
        bool boundary;
        const uint32_t g = decode_entry(b, a.list[live ? item : item0], h, v, p, seq, boundary);
        const uint8_t* cur = b.luma + (size_t(seq) * b.F + p + b.d) * plane;
        const uint8_t* ref = b.luma + (size_t(seq) * b.F + p) * plane;
        int dx, dy;
        uint32_t sad, cmp;
        es_block<BS, K, PWC>(cur, ref, b.W, b.H, h * BS, v * BS, a.S, band_runs, sm + size_t(grp) * a.region_words,
                             s_best + grp * (T / 32), dx, dy, sad, cmp, gtid, T);
        if (gtid == 0) {
            s_res[grp][0] = dx;
            s_res[grp][1] = dy;
            s_res[grp][2] = int(sad);
            s_res[grp][3] = int(cmp);
        }
        __syncthreads();
        if (live && gtid < 32) {
            // fused predict_frame + psnr SSE of this block at its vector (the group's first warp)
            const int lane = gtid;
            const int rdx = s_res[grp][0], rdy = s_res[grp][1];
            uint32_t sse = lane < BS ? row_sse_fp(cur, ref, b.W, h * BS, v * BS + lane, BS, rdx, rdy) : 0u;
            sse = __reduce_add_sync(0xFFFFFFFFu, sse);
            if (lane == 0) {
                const int ty = boundary ? ME_BOUNDARY : ME_OPAQUE;
                write_rec(a.recs + g, 2 * rdx, 2 * rdy, uint32_t(s_res[grp][2]) * 4u, uint32_t(s_res[grp][3]), 0, 0,
                          ty, false);
                if (a.stats) add_stats(a.stats + (size_t(seq) * b.pairs + p), sse, uint32_t(s_res[grp][3]), 0, ty);
            }
        }
    }
}

// Run mode (16x16 blocks, the largest ranges): the list holds runs of 1, 2 or
// 4 horizontally adjacent estimated blocks of one block row (classify emits
// them, count in entry bits 12-14).  A pass takes one run: its blocks' union
// window (the first block's window plus 16 columns per further block) is
// staged once by the whole CTA — 144 rows x 37 words for one block at S = 64,
// 144 x 49 for four — and the CTA splits into one group per block.  Staging,
// which the other CTA on the SM does not hide (config 5: 16 % of the search),
// is shared by up to four blocks.
template <int P1, int P2, int P4>
__global__ void __launch_bounds__(kEsThreads, 2) es_run_kernel(EsArgs a) {
    constexpr int BS = 16, K = 8;
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ unsigned long long s_best[kEsThreads / 32];
    __shared__ int s_item;
    __shared__ int s_res[4][4];
    const Batch& b = a.b;
    const int n = *a.nlist;
    const size_t plane = size_t(b.W) * b.H;
    const int band_runs = a.band_rows_max / K;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= n) return;
        const uint2 e = a.list[item];
        const int h0 = int(e.x & 0xFFF), cnt = int((e.x >> 12) & 7u), v = int((e.x >> 16) & 0x7FFF);
        const int p = int(e.y & 0xFFFF), seq = int(e.y >> 16);
        const int T = kEsThreads / cnt, grp = int(threadIdx.x) / T, gtid = int(threadIdx.x) - grp * T;
        const int h = h0 + grp;
        const uint8_t* cur = b.luma + (size_t(seq) * b.F + p + b.d) * plane;
        const uint8_t* ref = b.luma + (size_t(seq) * b.F + p) * plane;
        // the union of the run's windows (frame columns)
        const int xa = h0 * BS, xb = (h0 + cnt - 1) * BS;
        const int ux0 = xa + max(-a.S, -xa), ux1 = xb + min(a.S, b.W - xb - BS) + BS - 1;
        int dx, dy;
        uint32_t sad, cmp;
        unsigned long long* sb = s_best + grp * (T / 32);
        if (cnt == 4)
            es_block<BS, K, P4>(cur, ref, b.W, b.H, h * BS, v * BS, a.S, band_runs, sm, sb, dx, dy, sad, cmp, gtid, T, ux0, ux1 - ux0 + 1);
        else if (cnt == 2)
            es_block<BS, K, P2>(cur, ref, b.W, b.H, h * BS, v * BS, a.S, band_runs, sm, sb, dx, dy, sad, cmp, gtid, T, ux0, ux1 - ux0 + 1);
        else
            es_block<BS, K, P1>(cur, ref, b.W, b.H, h * BS, v * BS, a.S, band_runs, sm, sb, dx, dy, sad, cmp, gtid, T, ux0, ux1 - ux0 + 1);
        if (gtid == 0) {
            s_res[grp][0] = dx;
            s_res[grp][1] = dy;
            s_res[grp][2] = int(sad);
            s_res[grp][3] = int(cmp);
        }
        __syncthreads();
        if (gtid < 32) {
            // fused predict_frame + psnr SSE of this group's block at its vector
            const int lane = gtid;
            const int rdx = s_res[grp][0], rdy = s_res[grp][1];
            uint32_t sse = lane < BS ? row_sse_fp(cur, ref, b.W, h * BS, v * BS + lane, BS, rdx, rdy) : 0u;
            sse = __reduce_add_sync(0xFFFFFFFFu, sse);
            if (lane == 0) {
                const size_t pr = size_t(seq) * b.pairs + p;
                const uint32_t g = uint32_t((pr * b.rows + v) * b.cols + h);
                const int ty = a.types && a.types[g] == ME_BOUNDARY ? ME_BOUNDARY : ME_OPAQUE;
                write_rec(a.recs + g, 2 * rdx, 2 * rdy, uint32_t(s_res[grp][2]) * 4u, uint32_t(s_res[grp][3]), 0, 0,
                          ty, false);
                if (a.stats) add_stats(a.stats + pr, sse, uint32_t(s_res[grp][3]), 0, ty);
            }
        }
    }
}

template <int BS>
__global__ void __launch_bounds__(kEsThreads) es_single_kernel(const uint8_t* cur, const uint8_t* ref,
                                                               int W, int H, int x0, int y0, int S,
                                                               int band_rows, int64_t* out) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ unsigned long long s_best[kEsThreads / 32];
    int dx, dy;
    uint32_t sad, cmp;
    es_block<BS, 8>(cur, ref, W, H, x0, y0, S, band_rows / 8, sm, s_best, dx, dy, sad, cmp);
    if (threadIdx.x == 0) {
        out[0] = 2 * dx;
        out[1] = 2 * dy;
        out[2] = cmp;
        out[3] = int64_t(sad) * 4;
    }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------

// dy rows of candidates staged per band (a multiple of K = 8): the whole
// window when its 4 shifted copies fit in ~110 KB (one staging pass and one
// flat task list per block, no partial band), else bands of 64 rows
int es_band_rows(int bs, int S, int W, int H) {
    const int WX = min(2 * S + 1, W - bs + 1), WY = min(2 * S + 1, H - bs + 1);
    const int PW = ((WX - 1) >> 2) + (bs >> 2) + 1;
    int rows = (WY + 7) / 8 * 8;
    while (rows > 64 && size_t(4) * (size_t(rows + bs - 1) * PW + 32) * 4 > 110 * 1024) rows -= 8;
    return rows;
}

size_t es_smem_bytes(int bs, int S, int W, int H) {
    const int WX = min(2 * S + 1, W - bs + 1);
    const int PW = ((WX - 1) >> 2) + (bs >> 2) + 1;
    const int brows = es_band_rows(bs, S, W, H), srows = brows + bs - 1;
    return size_t(4) * (size_t(srows) * PW + 32) * 4 + size_t(brows) * 4;
}

// Run mode (es_run_kernel) for 16x16 blocks at the ranges whose one-block window
// is too large for several per CTA (S > 32): while a four-block union window
// still leaves two CTAs per SM and the whole window fits in one band.
bool es_use_runs(const Batch& b, int S) {
    if (b.bs != 16 || S <= 32 || S > 64) return false;
    const int WX = min(2 * S + 1, b.W - 16 + 1), WY = min(2 * S + 1, b.H - 16 + 1);
    const int PW4 = ((WX - 1 + 48) >> 2) + 5;
    const size_t rows = size_t(WY % 8 == 1 ? WY + 15 : (WY + 7) / 8 * 8 + 15);
    return size_t(4) * (rows * PW4 + 32) * 4 + size_t(WY + 8) * 4 <= 113 * 1024 && es_band_rows(16, S, b.W, b.H) >= (WY + 7) / 8 * 8;
}

cudaError_t launch_es(const Batch& b, int S, const uint2* list, const int* nlist, int* counter,
                      me_block_rec* recs, me_pair_stats* stats, int num_sms, cudaStream_t st, const uint8_t* types) {
    EsArgs ea;
    ea.types = types;
    ea.b = b;
    ea.S = S;
    ea.list = list;
    ea.nlist = nlist;
    ea.counter = counter;
    ea.recs = recs;
    ea.band_rows_max = es_band_rows(b.bs, S, b.W, b.H);
    ea.stats = stats;
    if (es_use_runs(b, S)) {
        ea.band_rows_max = es_band_rows(b.bs, S, b.W, b.H);
        const int WX = min(2 * S + 1, b.W - 16 + 1), WY = min(2 * S + 1, b.H - 16 + 1);
        const int PW4 = ((WX - 1 + 48) >> 2) + 5;
        const size_t rows = size_t(WY % 8 == 1 ? WY + 15 : (WY + 7) / 8 * 8 + 15);
        const size_t smem = size_t(4) * (rows * PW4 + 32) * 4 + size_t(ea.band_rows_max) * 4;
        void (*kern)(EsArgs) = (S == 64 && WX == 129) ? es_run_kernel<37, 41, 49> : es_run_kernel<0, 0, 0>;
        cudaError_t e;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)))) return e;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEsThreads, smem);
        kern<<<num_sms * (occ > 0 ? occ : 1), kEsThreads, smem, st>>>(ea);
        return cudaGetLastError();
    }
    const size_t smem1 = es_smem_bytes(b.bs, S, b.W, b.H);
    // the row stride of the widest (unclipped) window, fixed for every block
    const int PW = ((min(2 * S + 1, b.W - b.bs + 1) - 1) >> 2) + (b.bs >> 2) + 1;
    // blocks per CTA pass: 4 while four whole windows fit in ~64 KB (S <= 16), 2 within ~64 KB
    // (S <= 32), else 1 (bands of rows for the largest windows)
    const int WY = min(2 * S + 1, b.H - b.bs + 1);
    const bool whole = ea.band_rows_max >= (WY + 7) / 8 * 8;
    const int nb = !whole ? 1 : 4 * smem1 <= 64 * 1024 ? 4 : 2 * smem1 <= 64 * 1024 ? 2 : 1;
    ea.region_words = int((smem1 + 15) / 16 * 4);
    const size_t smem = size_t(nb) * ea.region_words * 4;
    void (*kern)(EsArgs);
    if (b.bs == 16) {
        if (nb == 4)
            kern = PW == 13 ? es_kernel<16, 8, 13, 4> : es_kernel<16, 8, 0, 4>;
        else if (nb == 2)
            kern = PW == 21 ? es_kernel<16, 8, 21, 2> : PW == 13 ? es_kernel<16, 8, 13, 2> : es_kernel<16, 8, 0, 2>;
        else
            kern = PW == 37 ? es_kernel<16, 8, 37, 1> : PW == 21 ? es_kernel<16, 8, 21, 1> : PW == 13 ? es_kernel<16, 8, 13, 1>
                                                                                                  : es_kernel<16, 8, 0, 1>;
    } else {
        if (nb == 4)
            kern = PW == 11 ? es_kernel<8, 8, 11, 4> : es_kernel<8, 8, 0, 4>;
        else if (nb == 2)
            kern = PW == 19 ? es_kernel<8, 8, 19, 2> : PW == 11 ? es_kernel<8, 8, 11, 2> : es_kernel<8, 8, 0, 2>;
        else
            kern = PW == 35 ? es_kernel<8, 8, 35, 1> : PW == 19 ? es_kernel<8, 8, 19, 1> : PW == 11 ? es_kernel<8, 8, 11, 1>
                                                                                               : es_kernel<8, 8, 0, 1>;
    }
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)))) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEsThreads, smem);
    kern<<<num_sms * (occ > 0 ? occ : 1), kEsThreads, smem, st>>>(ea);
    return cudaGetLastError();
}

cudaError_t launch_es_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                             int size, int range, int64_t* out, cudaStream_t st) {
    const size_t smem = es_smem_bytes(size, range, W, H);
    auto kern = size == 16 ? es_single_kernel<16> : es_single_kernel<8>;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)))) return e;
    kern<<<1, kEsThreads, smem, st>>>(cur, ref, W, H, x0, y0, range, es_band_rows(size, range, W, H), out);
    return cudaGetLastError();
}

}  // namespace mek
