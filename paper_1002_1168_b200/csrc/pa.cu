// pa.cu — the proposed algorithm (estimators.cpp:238-382): gather_candidates
// + brs_select + prs_refine as a dataflow wavefront over the sorted work list
// (pa_fast_kernel: a warp per block; pa_duo_kernel: two blocks per warp;
// pa_quad_kernel: four blocks per warp, the wide middle of large batches;
// pa_smem_kernel: one small pair resident in one CTA's shared memory;
// pa_kernel: the generic path for 16x16, half-pel and external prev fields),
// and the single-block BRS / PRS / prs_update kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "pa_common.cuh"

namespace mek {

// ---------------------------------------------------------------------------
// PA: gather_candidates + brs_select + prs_refine (estimators.cpp:238-382) as
// a dataflow wavefront.  Block (h, v) of pair p depends only on A = (h-1, v),
// B = (h, v-1), C = (h+1, v-1) of pair p and T = (h, v) of pair p-1
// (bench.cpp:204 threads the previous pair's field), so every block with the
// same t = h + 2v + p is independent (a plain h + v diagonal is NOT: C lies on
// it).  The work list is sorted by t; persistent warps take list entries
// round-robin and spin (acquire loads) on their four dependencies' MV words,
// which hold a sentinel until the producing warp's release store.  Every
// dependency sits earlier in the list, so the smallest unfinished entry can
// always proceed: no grid-wide barrier, no deadlock.
// ---------------------------------------------------------------------------

// Scores 4 candidate slots (lanes 8k..8k+7 own slot k): texture (4 x SAD at a
// half-pel vector) or shape (4 x 255 x mismatches at the llround-snapped pel
// vector, estimators.cpp:284-286).  Result broadcast in each 8-lane group.
__device__ __forceinline__ uint32_t score4(const PaParams& P, const PaBlock& B, int lane,
                                           int dx2, int dy2, bool shape) {
    uint32_t s = 0;
    if (shape) {
        // llround(h / 2) == (h + sign(h)) / 2 with C truncation
        const int fx = (dx2 + (dx2 > 0) - (dx2 < 0)) / 2;
        const int fy = (dy2 + (dy2 > 0) - (dy2 < 0)) / 2;
        for (int r = lane & 7; r < P.bs; r += 8)
            s += row_shape(B.ca, B.ra, P.W, P.H, B.x0, B.y0 + r, P.bs, fx, fy);
        s *= 255u * 4u;
    } else {
        for (int r = lane & 7; r < P.bs; r += 8)
            s += row_sad4(B.cur, B.ref, P.W, P.H, B.x0, B.y0 + r, P.bs, dx2, dy2);
    }
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
    return s;
}

// 8 neighbour slots (lanes 4k..4k+3 own slot k), texture only.
__device__ __forceinline__ uint32_t score8(const PaParams& P, const PaBlock& B, int lane, int dx2,
                                           int dy2, bool active) {
    uint32_t s = 0;
    if (active)
        for (int r = lane & 3; r < P.bs; r += 4)
            s += row_sad4(B.cur, B.ref, P.W, P.H, B.x0, B.y0 + r, P.bs, dx2, dy2);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    return s;
}

struct PaResult {
    int dx, dy;
    uint32_t cost_q4, dpd, iters;
};

// prs_refine (estimators.cpp:311-382) from an already clipped start (cx, cy)
// whose texture cost is `ccost` (kInf: not yet evaluated).  Warp-uniform.
__device__ PaResult prs_warp(const PaParams& P, const PaBlock& B, int lane, int cx, int cy,
                             uint32_t ccost, uint32_t* bitmap) {
    const int M = P.bm_side / 2;  // lattice radius
    for (int i = lane; i < P.bm_words; i += 32) bitmap[i] = 0;
    __syncwarp();
    const int sx0 = cx, sy0 = cy;
    auto lattice_bit = [&](int vx, int vy) {
        return ((vy - sy0) / P.step + M) * P.bm_side + ((vx - sx0) / P.step + M);
    };
    if (lane == 0) {
        const int bit = lattice_bit(cx, cy);
        bitmap[bit >> 5] |= 1u << (bit & 31);
    }
    __syncwarp();
    uint32_t dpd = 1;
    if (ccost == kInf) {
        const uint32_t s = score4(P, B, lane, cx, cy, false);
        ccost = __shfl_sync(0xFFFFFFFFu, s, 0);
    }
    uint32_t iters = 0;
    for (int it = 0; it < P.max_iter; ++it) {
        if (ccost == 0) break;
        const int k = lane >> 2;
        const int nx = cx + c_off8[k][0] * P.step, ny = cy + c_off8[k][1] * P.step;
        const bool adm = nx >= B.w.lo_x && nx <= B.w.hi_x && ny >= B.w.lo_y && ny <= B.w.hi_y;
        const uint32_t cost = score8(P, B, lane, nx, ny, adm);
        const bool leader = (lane & 3) == 0;
        bool fresh = false;
        if (adm && leader) {
            const int bit = lattice_bit(nx, ny);
            const uint32_t m = 1u << (bit & 31);
            fresh = (atomicOr(&bitmap[bit >> 5], m) & m) == 0;
        }
        dpd += __popc(__ballot_sync(0xFFFFFFFFu, fresh));
        const uint32_t mine = (adm && leader) ? cost : kInf;
        const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, mine);
        if (m >= ccost) break;  // center kept (estimators.cpp:376)
        const uint32_t ties = __ballot_sync(0xFFFFFFFFu, adm && leader && cost == m);
        int win;
        if (__popc(ties) == 1) {
            win = (__ffs(ties) - 1) >> 2;
        } else {
            // stable descending sort by off . dir (estimators.cpp:357-362): the
            // first tied neighbour in sorted order has the largest key, and the
            // smallest index among equal keys.
            double dir_x, dir_y;
            prs_direction(P, B, lane, cx, cy, dir_x, dir_y);
            win = -1;
            double bestkey = 0.0;
            for (int i = 0; i < 8; ++i) {
                if (!((ties >> (4 * i)) & 1u)) continue;
                const double key = __dadd_rn(__dmul_rn(double(c_off8[i][0]), dir_x),
                                             __dmul_rn(double(c_off8[i][1]), dir_y));
                if (win < 0 || key > bestkey) {
                    win = i;
                    bestkey = key;
                }
            }
        }
        cx += c_off8[win][0] * P.step;
        cy += c_off8[win][1] * P.step;
        ccost = m;
        ++iters;
    }
    PaResult r;
    r.dx = cx;
    r.dy = cy;
    r.cost_q4 = ccost;
    r.dpd = dpd;
    r.iters = iters;
    return r;
}


// brs_select (estimators.cpp:257-301) then prs_refine.  cand[] holds the four
// raw candidates A, B, C, T (every lane).  Returns also the BRS winner slot.
__device__ __noinline__ PaResult pa_block(const PaParams& P, const PaBlock& B, int lane, bool boundary,
                             const int cdx[4], const int cdy[4], uint32_t* bitmap,
                             uint32_t* brs_scores = nullptr, int* brs_kinds = nullptr) {
    const int k = lane >> 3;
    int rx = cdx[0], ry = cdy[0];
#pragma unroll
    for (int i = 1; i < 4; ++i)
        if (k == i) {
            rx = cdx[i];
            ry = cdy[i];
        }
    const int vx = clip_comp(rx, B.w.lo_x, B.w.hi_x);
    const int vy = clip_comp(ry, B.w.lo_y, B.w.hi_y);
    const bool shape = boundary && (k < 3 || P.bt_shape);
    const uint32_t s = score4(P, B, lane, vx, vy, shape);
    uint32_t best = 0;
    int bx = 0, by = 0, win = 0;
    for (int i = 0; i < 4; ++i) {
        const uint32_t si = __shfl_sync(0xFFFFFFFFu, s, 8 * i);
        const int ix = __shfl_sync(0xFFFFFFFFu, vx, 8 * i), iy = __shfl_sync(0xFFFFFFFFu, vy, 8 * i);
        if (brs_scores) brs_scores[i] = si;
        if (i == 0 || si < best) {
            win = i;
            best = si;
            bx = ix;
            by = iy;
        }
    }
    if (brs_kinds)
        for (int i = 0; i < 4; ++i) brs_kinds[i] = boundary && (i < 3 || P.bt_shape);
    const bool win_shape = boundary && (win < 3 || P.bt_shape);
    return prs_warp(P, B, lane, bx, by, win_shape ? kInf : best, bitmap);
}


// ---------------------------------------------------------------------------
// PA fast path (one block per warp).  With PRS on the integer grid (step 2)
// and at most R = 4 iterations, every position prs_refine can evaluate lies
// within +/-4 pels of the BRS winner.  So a block needs exactly one round of
// global loads — a (BS+8)^2 reference patch per distinct candidate, staged in
// shared memory — after which the BRS scores, all 81 lattice costs around the
// winner (computed eagerly, in parallel) and the final SSE come from shared
// memory, and the PRS walk itself is a chain of table lookups.  The wavefront's
// critical path is a chain of blocks, so per-block latency is what this
// layout minimises.
// ---------------------------------------------------------------------------

template <int BS>
struct WPatch {
    static constexpr int R = 4;
    static constexpr int L = 2 * R + 1;     // lattice side (9)
    static constexpr int NP = L * L;        // 81 lattice positions
    static constexpr int PR = BS + 2 * R;   // patch rows
    static constexpr int PB = BS + 2 * R;   // patch bytes per row
    // A patch row is staged as CH raw 16-byte aligned chunks (two lanes per row
    // share one L1 wavefront); the candidate's byte offset into the first
    // chunk is applied when reading.  The row stride is padded so the 8
    // (or 16) block rows a warp reads at once fall in distinct banks.
    static constexpr int CH = (PB + 15) / 16 + 1;
    static constexpr int PWW = BS == 8 ? 12 : 20;
    static constexpr int WORDS = PR * PWW;
    static constexpr int WARP_WORDS = 4 * WORDS + 4;  // patches + visited bitmap
};

// Loads patch row r (0..PR-1) of the candidate at pel offset (cx, cy) into
// dst.  Branch-free: the row index is clamped and every 4-byte word is loaded
// only when it lies inside the frame row (W % 4 == 0, so words never straddle
// rows); bytes outside the frame read as 0.  Only inadmissible positions —
// never evaluated — touch those bytes.
template <int BS>
__device__ __forceinline__ void stage_patch_row(const uint8_t* ref, int W, int H, int x0, int y0,
                                                int cx, int cy, int r, uint32_t* dst) {
    using F = WPatch<BS>;
    constexpr int PW = F::PB / 4;
    const int y = clampi(y0 + cy - F::R + r, 0, H - 1);
    const int xs = x0 + cx - F::R;                 // first byte (may be < 0 or run past W)
    const int wa = xs & ~3;                        // floor to a word boundary (two's complement)
    const uint32_t sh = uint32_t(xs - wa) * 8;
    const uint8_t* row = ref + size_t(y) * W;
    uint32_t w[PW + 1];
#pragma unroll
    for (int i = 0; i <= PW; ++i) {
        const int c = wa + 4 * i;
        w[i] = (c >= 0 && c + 4 <= W) ? __ldg(reinterpret_cast<const uint32_t*>(row + c)) : 0u;
    }
#pragma unroll
    for (int i = 0; i < PW; ++i) dst[i] = __funnelshift_r(w[i], w[i + 1], sh);
    dst[PW] = 0u;
}

// BS/4 words of a patch row starting at byte offset i (0..2R).
template <int BS>
__device__ __forceinline__ void patch_words(const uint32_t* row, int i, uint32_t (&o)[BS / 4]) {
    const uint32_t* p = row + (i >> 2);
    const uint32_t sh = uint32_t(i & 3) * 8;
    uint32_t w0 = p[0];
#pragma unroll
    for (int k = 0; k < BS / 4; ++k) {
        const uint32_t w1 = p[k + 1];
        o[k] = __funnelshift_r(w0, w1, sh);
        w0 = w1;
    }
}

struct PaArgs {
    Batch b;
    PaParams P;
    const uint2* list;
    const int* nlist;
    me_block_rec* recs;
    const int32_t* prev0;  // pair 0's temporal candidates or null
    me_pair_stats* stats;
    int fast;              // patch fast path allowed (step 2, max_iter <= 4)
    int warp_words;        // shared words per warp
    int win_words;         // pa_fast_kernel: row stride (words) of the staged search window, 0 = per-candidate patches
    int awin_words;        // ... and of the boundary blocks' staged reference-alpha window (byte masks), 0 = off
    int poll_ns;           // dependency poll interval
    int pdl;               // hybrid launches chained by programmatic dependent launch (see PdlScope)
    const int* range;      // [begin, end) of the list for this launch (device) or null: [0, *nlist)
    int* claim;            // zeroed claim counter of this launch (in-order dynamic claiming) or null
    unsigned long long* trace;  // debug: per entry {claimed, deps ready, done, smid} (ns)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// gather_candidates (estimators.cpp:238-255): lane i < 4 returns candidate
// i's MV word (A, B, C, T), waiting for dependencies still in flight.
__device__ __forceinline__ uint32_t fetch_candidate(const PaArgs& a, uint32_t g, int h, int v, int p,
                                                    int lane) {
    const Batch& b = a.b;
    uint32_t mvw = 0;
    if (lane < 4) {
        const uint32_t* src = nullptr;
        if (lane == 0 && h > 0) src = reinterpret_cast<const uint32_t*>(a.recs + g - 1);
        if (lane == 1 && v > 0) src = reinterpret_cast<const uint32_t*>(a.recs + g - b.cols);
        if (lane == 2 && v > 0 && h + 1 < b.cols)
            src = reinterpret_cast<const uint32_t*>(a.recs + g - b.cols + 1);
        if (lane == 3 && p > 0)
            src = reinterpret_cast<const uint32_t*>(a.recs + g - uint32_t(b.rows) * b.cols);
        if (src) {
            mvw = ld_relaxed(src);
            while (mvw == kSentinel) {
                __nanosleep(a.poll_ns);
                mvw = ld_relaxed(src);
            }
        } else if (lane == 3 && a.prev0) {
            const int i = v * b.cols + h;
            mvw = pack_mv(a.prev0[2 * i], a.prev0[2 * i + 1]);
        }
    }
    __syncwarp();
    return mvw;
}

template <int NW>
__device__ __forceinline__ void ld8u_or16(const uint8_t* p, uint32_t (&w)[NW]) {
    if (NW == 2) ld8u(p, w[0], w[1 % NW]);
    else ld16u(p, w);
}

template <int BS>
__device__ __forceinline__ void load_row(const uint8_t* p, uint32_t (&w)[BS / 4]) {
    if (BS == 8) {
        const uint2 c2 = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = c2.x;
        w[1 % (BS / 4)] = c2.y;
    } else {
        const uint4 c4 = __ldg(reinterpret_cast<const uint4*>(p));
        w[0] = c4.x;
        w[1 % (BS / 4)] = c4.y;
        w[2 % (BS / 4)] = c4.z;
        w[3 % (BS / 4)] = c4.w;
    }
}

// Fast path for one block (warp).  mvw: lane i < 4 holds candidate i's raw MV
// word.  Returns false (nothing computed) when a clipped candidate is
// half-pel, i.e. the block needs the generic path.
template <int BS>
__device__ bool pa_patch_block(const PaParams& P, const PaBlock& B, int lane, bool boundary,
                               uint32_t mvw, uint32_t* ws, PaResult& res, uint32_t& sse_out) {
    using F = WPatch<BS>;
    constexpr int NW = BS / 4;
    constexpr int L = F::L;
    const int W = P.W;
    uint32_t* patch = ws;                 // [4][PR][PWW]
    uint32_t* table = ws + 4 * F::WORDS;  // [3] visited bitmap
    // my candidate slot (lanes 8c..8c+7 serve candidate c) and its duplicate map
    const int c = lane >> 3, sub = lane & 7;
    const uint32_t mine = __shfl_sync(0xFFFFFFFFu, mvw, c);
    const int myx = clip_comp(mv_dx(mine), B.w.lo_x, B.w.hi_x);  // clip_to_window (:275-276)
    const int myy = clip_comp(mv_dy(mine), B.w.lo_y, B.w.hi_y);
    if (__any_sync(0xFFFFFFFFu, ((myx | myy) & 1) != 0)) return false;
    int md = c;  // first candidate with the same clipped vector
#pragma unroll
    for (int j = 2; j >= 0; --j) {
        const int jx = __shfl_sync(0xFFFFFFFFu, myx, 8 * j), jy = __shfl_sync(0xFFFFFFFFu, myy, 8 * j);
        if (j < c && jx == myx && jy == myy) md = j;
    }
    // --- the single round of reference loads: distinct candidate patches -------
    // 16-byte aligned chunks, consecutive lanes on the same row (one L1
    // wavefront per row); chunks outside the frame row read as zero (only
    // inadmissible positions touch them), rows are clamped.
    int po = 0;  // byte offset of my candidate's patch start in its first chunk
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int ccx = __shfl_sync(0xFFFFFFFFu, myx, 8 * cc) >> 1;
        const int ccy = __shfl_sync(0xFFFFFFFFu, myy, 8 * cc) >> 1;
        const int cdup = __shfl_sync(0xFFFFFFFFu, md, 8 * cc);
        const int xs = B.x0 + ccx - F::R;
        const int a0 = xs & ~15;
        if (c == cc) po = xs - a0;
        if (cdup != cc) continue;  // warp-uniform
        for (int idx = lane; idx < F::PR * F::CH; idx += 32) {
            const int r = idx / F::CH, ch = idx - r * F::CH;
            const int y = clampi(B.y0 + ccy - F::R + r, 0, P.H - 1);
            const int cs = a0 + 16 * ch;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (cs >= 0 && cs + 16 <= W) v = __ldg(reinterpret_cast<const uint4*>(B.ref + size_t(y) * W + cs));
            *reinterpret_cast<uint4*>(patch + cc * F::WORDS + r * F::PWW + 4 * ch) = v;
        }
    }
    // the patch my candidate's BRS score reads (duplicates share one)
    const int mpo = __shfl_sync(0xFFFFFFFFu, po, 8 * md);
    // current block: every lane holds all of it (broadcast loads)
    uint32_t cb[BS][NW];
#pragma unroll
    for (int r = 0; r < BS; ++r) load_row<BS>(B.cur + size_t(B.y0 + r) * W + B.x0, cb[r]);
    // shape scores (boundary blocks): alpha rows of my candidate
    const bool shape = boundary && (c < 3 || P.bt_shape);
    uint32_t s = 0;
    if (shape)
        for (int r = sub; r < BS; r += 8)
            s += row_shape(B.ca, B.ra, W, P.H, B.x0, B.y0 + r, BS, myx >> 1, myy >> 1) * (255u * 4u);
    __syncwarp();
    // --- brs_select (estimators.cpp:257-301) ------------------------------------
    if (!shape) {
        const uint32_t* pc = patch + md * F::WORDS;
#pragma unroll
        for (int r = 0; r < BS; ++r) {
            if ((r & 7) != sub) continue;
            uint32_t w[NW];
            patch_words<BS>(pc + (F::R + r) * F::PWW, F::R + mpo, w);
            uint32_t acc = 0;
#pragma unroll
            for (int k = 0; k < NW; ++k) acc = vad4(cb[r][k], w[k], acc);
            s += acc * 4u;
        }
    }
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
    uint32_t best = __shfl_sync(0xFFFFFFFFu, s, 0);
    int win = 0;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
        const uint32_t si = __shfl_sync(0xFFFFFFFFu, s, 8 * i);
        if (si < best) {  // strict <: A, B, C, T tie order (:295)
            best = si;
            win = i;
        }
    }
    const bool win_shape = boundary && (win < 3 || P.bt_shape);
    const int wx = __shfl_sync(0xFFFFFFFFu, myx, 8 * win), wy = __shfl_sync(0xFFFFFFFFu, myy, 8 * win);
    const int wp = __shfl_sync(0xFFFFFFFFu, md, 8 * win);
    const int wo = __shfl_sync(0xFFFFFFFFu, mpo, 8 * win);  // its byte offset
    const uint32_t* pw = patch + wp * F::WORDS;  // the winner's patch
    // --- prs_refine (estimators.cpp:311-382), lazily from the staged patch ----
    // Each iteration scores the centre's 8 neighbours: lanes 4k..4k+3 own
    // neighbour k, BS/4 block rows each; all reads hit shared memory.
    uint32_t* vis = table;  // [3] visited lattice bits (9 x 9 around the start)
    if (lane < 3) vis[lane] = lane == 1 ? (1u << (F::R * L + F::R - 32)) : 0u;
    __syncwarp();
    uint32_t ccost = best;
    if (win_shape) {  // the centre's texture cost was not computed by BRS
        uint32_t t = 0;
#pragma unroll
        for (int r = 0; r < BS; ++r)
            if ((r & 7) == sub) {
                uint32_t w[NW];
                patch_words<BS>(pw + (F::R + r) * F::PWW, F::R + wo, w);
#pragma unroll
                for (int kk = 0; kk < NW; ++kk) t = vad4(cb[r][kk], w[kk], t);
            }
        t = (c == 0) ? t : 0u;
        ccost = 4u * __reduce_add_sync(0xFFFFFFFFu, t);
    }
    int ci = 0, cj = 0;  // centre, pels relative to the BRS winner
    uint32_t dpd = 1, iters = 0;
    const int k = lane >> 2, q = lane & 3;
    const int kx = c_off8[k][0], ky = c_off8[k][1];
    for (int it = 0; it < P.max_iter; ++it) {
        if (ccost == 0) break;  // already a global minimum (:341)
        const int px = ci + kx, py = cj + ky;
        const bool adm = wx + 2 * px >= B.w.lo_x && wx + 2 * px <= B.w.hi_x &&
                         wy + 2 * py >= B.w.lo_y && wy + 2 * py <= B.w.hi_y;
        uint32_t part = 0;
#pragma unroll
        for (int r = 0; r < BS; ++r)
            if ((r & 3) == q) {
                uint32_t w[NW];
                patch_words<BS>(pw + (F::R + py + r) * F::PWW, F::R + px + wo, w);
#pragma unroll
                for (int kk = 0; kk < NW; ++kk) part = vad4(cb[r][kk], w[kk], part);
            }
        part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
        part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
        const uint32_t cost = 4u * part;
        const bool lead = adm && q == 0;
        bool fresh = false;
        if (lead) {  // unique aggregate evaluations (:321-332)
            const int bit = (F::R + py) * L + F::R + px;
            const uint32_t m = 1u << (bit & 31);
            fresh = (atomicOr(&vis[bit >> 5], m) & m) == 0;
        }
        dpd += __popc(__ballot_sync(0xFFFFFFFFu, fresh));
        const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, lead ? cost : kInf);
        if (m >= ccost) break;  // centre kept (:376)
        const uint32_t ties = __ballot_sync(0xFFFFFFFFu, lead && cost == m);
        int w;
        if (__popc(ties) == 1) {
            w = (__ffs(ties) - 1) >> 2;
        } else {
            // stable descending sort by off . dir (:357-362): the first tied
            // neighbour in sorted order = largest key, lowest index on equal keys
            double dir_x, dir_y;
            prs_direction(P, B, lane, wx + 2 * ci, wy + 2 * cj, dir_x, dir_y);
            w = -1;
            double bestkey = 0.0;
            for (int o = 0; o < 8; ++o) {
                if (!((ties >> (4 * o)) & 1u)) continue;
                const double key = __dadd_rn(__dmul_rn(double(c_off8[o][0]), dir_x),
                                             __dmul_rn(double(c_off8[o][1]), dir_y));
                if (w < 0 || key > bestkey) {
                    w = o;
                    bestkey = key;
                }
            }
        }
        ci += c_off8[w][0];
        cj += c_off8[w][1];
        ccost = m;
        ++iters;
    }
    // --- fused predict_frame + psnr SSE at the final vector ---------------------
    uint32_t se = 0;
#pragma unroll
    for (int r = 0; r < BS; ++r) {
        if (r != lane) continue;
        uint32_t w[NW];
        patch_words<BS>(pw + (F::R + cj + r) * F::PWW, F::R + ci + wo, w);
#pragma unroll
        for (int kk = 0; kk < NW; ++kk) se = sq4(cb[r][kk], w[kk], se);
    }
    sse_out = __reduce_add_sync(0xFFFFFFFFu, se);
    res.dx = wx + 2 * ci;
    res.dy = wy + 2 * cj;
    res.cost_q4 = ccost;
    res.dpd = dpd;
    res.iters = iters;
    return true;
}

// In-order work claiming, CTA by CTA.  With `claim` (a zeroed counter per
// launch), a CTA takes BATCHES of nwarps x STEP consecutive list entries with
// one global atomicAdd, and warp w of the CTA works on entries w*STEP ..
// w*STEP+STEP-1 of each batch, batch after batch — the same locality as the
// static round-robin (a CTA's warps hold consecutive entries, which share
// reference rows in L1), but batches are handed out in list order to
// whichever CTAs are running.  Every dependency of an entry lies earlier in
// the list, so the smallest unfinished entry is always held by a running warp
// (its warp finished every earlier batch of its CTA): the grid makes progress
// whatever subset of its CTAs is resident — a concurrent kernel may hold part
// of the device.  Without `claim`: static round-robin over the whole grid,
// which needs every CTA resident.
constexpr int kClaimRing = 4;  // batch bases in flight per CTA
struct CtaClaim {
    int* sh;  // [0] batches published, [1] claims started, [2, 2+R) bases, [2+R, 2+2R) reads
    int* gctr;
    int k;    // this warp's next batch
    __device__ static void init(int* sh) {
        if (threadIdx.x < 2 + 2 * kClaimRing) sh[threadIdx.x] = 0;
        __syncthreads();
    }
    template <int STEP>
    __device__ int next(int lane, int wid, int nw) {
        const int slot = k % kClaimRing;
        int base = 0;
        if (lane == 0) {
            volatile int* v = sh;
            while (v[0] <= k) {
                if (atomicCAS(&sh[1], k, k + 1) == k) {  // this warp claims batch k for the CTA
                    if (k >= kClaimRing)                 // every warp has read batch k - R's base
                        while (v[2 + kClaimRing + slot] < nw) __nanosleep(20);
                    v[2 + kClaimRing + slot] = 0;
                    v[2 + slot] = atomicAdd(gctr, STEP * nw);
                    __threadfence_block();
                    v[0] = k + 1;
                } else {
                    __nanosleep(20);
                }
            }
            base = v[2 + slot];
            atomicAdd(&sh[2 + kClaimRing + slot], 1);
        }
        ++k;
        return __shfl_sync(0xFFFFFFFFu, base, 0) + STEP * wid;
    }
};

template <int BS>
__global__ void __launch_bounds__(256, BS == 8 ? 3 : 2) pa_kernel(PaArgs a) {
    extern __shared__ uint32_t s_pa[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* ws = s_pa + wid * a.warp_words;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int n = *a.nlist;
    const Batch& b = a.b;
    const PaParams& P = a.P;
    const size_t plane = size_t(b.W) * b.H;
    // Static round-robin over the wavefront-sorted list: every dependency of
    // entry e sits at a smaller index, each warp handles its entries in
    // increasing order and the grid is sized so every warp is resident, so
    // the smallest unfinished entry is always being worked on (no deadlock,
    // no grid-wide barrier).
    __shared__ int s_claim[2 + 2 * kClaimRing];
    CtaClaim cc{s_claim, a.claim, 0};
    CtaClaim::init(s_claim);
    int nxt = 0;
    for (int rel = a.claim ? cc.next<1>(lane, wid, blockDim.x >> 5) : blockIdx.x * (blockDim.x >> 5) + wid; rel < n;
         rel = a.claim ? cc.next<1>(lane, wid, blockDim.x >> 5) : nxt) {
        nxt = a.claim ? 0 : rel + nwarps;
        const int item = rel;
        const uint2 e = a.list[item];
        if (e.x == kInvalidEntry) continue;
        int h, v, p, seq;
        bool boundary;
        const uint32_t g = decode_entry(b, e, h, v, p, seq, boundary);
        PaBlock B;
        const size_t fc = size_t(seq) * b.F + p + b.d, fr = size_t(seq) * b.F + p;
        B.cur = b.luma + fc * plane;
        B.ref = b.luma + fr * plane;
        B.ca = b.alpha ? b.alpha + fc * plane : nullptr;
        B.ra = b.alpha ? b.alpha + fr * plane : nullptr;
        B.x0 = h * BS;
        B.y0 = v * BS;
        B.w = hp_window(B.x0, B.y0, BS, P.W, P.H, P.S);
        unsigned long long t0 = 0;
        if (a.trace) t0 = gtimer();
        const uint32_t mvw = fetch_candidate(a, g, h, v, p, lane);
        unsigned long long t1 = 0;
        if (a.trace) t1 = gtimer();
        PaResult r;
        uint32_t sse = 0;
        if (!(a.fast && pa_patch_block<BS>(P, B, lane, boundary, mvw, ws, r, sse))) {
            int rdx[4], rdy[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t w = __shfl_sync(0xFFFFFFFFu, mvw, i);
                rdx[i] = mv_dx(w);
                rdy[i] = mv_dy(w);
            }
            r = pa_block(P, B, lane, boundary, rdx, rdy, ws);
            uint32_t s = lane < BS ? row_sse(B.cur, B.ref, P.W, P.H, B.x0, B.y0 + lane, BS, r.dx, r.dy) : 0u;
            sse = __reduce_add_sync(0xFFFFFFFFu, s);
        }
        if (lane == 0) {
            const int ty = boundary ? ME_BOUNDARY : ME_OPAQUE;
            write_rec(a.recs + g, r.dx, r.dy, r.cost_q4, 4, r.dpd, r.iters, ty, true);
            if (a.stats) add_stats_pa(a.stats + (size_t(seq) * b.pairs + p), sse, r.dpd);
            if (a.trace) {
                unsigned smid;
                asm("mov.u32 %0, %%smid;" : "=r"(smid));
                a.trace[4 * item + 0] = t0;
                a.trace[4 * item + 1] = t1;
                a.trace[4 * item + 2] = gtimer();
                a.trace[4 * item + 3] = smid;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// pa_fast_kernel: the 8x8, integer-pel PA path of the benchmark (config 4),
// written for a short instruction stream per block: kernel arguments by
// value, no address-taken structs, decoded work-list entries, the current
// block staged once in shared memory, 16-byte-chunk patch staging (two lanes
// per patch row), lazy PRS on the staged patch.  Same algorithm and
// dependency protocol as pa_kernel.  All candidates are integer-pel: A, B, C
// and T come from this integer-pel search or from an external prev field the
// host checked to be integer-pel (a half-pel one is routed to pa_kernel).
// ---------------------------------------------------------------------------

constexpr int kFastPWW = 12;       // patch row stride in words (8 used: two 16-byte chunks)
constexpr int kFastPatch = kFastPR * kFastPWW;
constexpr int kFastWarpWords = 4 * kFastPatch + 16 + 4;  // patches, current block, visited

// Programmatic dependent launch between the hybrid's three persistent grids
// (head -> middle -> tail).  Their items already synchronise through the
// record polls, so a dependent grid may start as soon as every CTA of its
// predecessor is resident: each CTA allows it on entry
// (griddepcontrol.launch_dependents) and, on exit, waits for the predecessor
// grid to complete (griddepcontrol.wait), so a grid never completes before
// the one it was chained to (stream order after the tail stays intact).
struct PdlScope {
    bool on;
    __device__ explicit PdlScope(int mode) : on(mode != 0) {
        // mode 2: also chained to the sort (reads its list): wait for it first
        if (mode == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    __device__ ~PdlScope() {
        if (on) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
};

template <int MINB, bool TRACE = false>
__global__ void __launch_bounds__(256, MINB) pa_fast_kernel(const PaArgs a) {
    const PdlScope pdl_scope(a.pdl);
    extern __shared__ uint32_t s_pa[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // window mode (a.win_words): the block's whole clipped search window
    // (+4 rows / columns for the walk's neighbours) is staged at claim time,
    // while the dependencies are awaited, so no load is left between the
    // dependencies' arrival and the search; else per-candidate patches
    const int wsw = a.win_words;
    const int area = a.warp_words - 20;      // patches or window, then cw and visited
    uint32_t* ws = s_pa + wid * a.warp_words;
    uint32_t* patch = ws;                    // [4][16][12] or [rows][wsw]
    uint32_t* cw = ws + area;                // [8][2] current block
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int beg = a.range ? a.range[0] : 0, n = a.range ? a.range[1] : *a.nlist;
    const int W = a.b.W, H = a.b.H, S = a.P.S;
    const uint32_t cols = a.b.cols, rows = a.b.rows, pairs = a.b.pairs;
    const int c = lane >> 3, sub = lane & 7;
    const int k = lane >> 2, q = lane & 3;   // PRS: neighbour k, rows q and q + 4
    const int kx = off8x(k), ky = off8y(k);
    // static round-robin over the wavefront-sorted list (see pa_kernel)
    __shared__ int s_claim[2 + 2 * kClaimRing];
    CtaClaim cc{s_claim, a.claim, 0};
    CtaClaim::init(s_claim);
    int nxt = 0;
    for (int rel = a.claim ? cc.next<1>(lane, wid, blockDim.x >> 5) : blockIdx.x * (blockDim.x >> 5) + wid; beg + rel < n;
         rel = a.claim ? cc.next<1>(lane, wid, blockDim.x >> 5) : nxt) {
        nxt = a.claim ? 0 : rel + nwarps;
        const int item = beg + rel;
        const uint2 e = __ldg(a.list + item);
        if (e.x == kInvalidEntry) continue;
        unsigned long long t_claim = 0, t_ready = 0;
        long long c_ready = 0, c_patch = 0, c_brs = 0, c_walk = 0;
        if (TRACE) t_claim = gtimer();
        const int h = int(e.x & 0xFFFF), v = int((e.x >> 16) & 0x7FFF), p = int(e.y & 0xFFFF);
        const uint32_t seq = e.y >> 16;
        const bool boundary = (e.x & kBoundaryBit) != 0;
        const uint32_t pair = seq * pairs + uint32_t(p);
        const uint32_t g = (pair * rows + uint32_t(v)) * cols + uint32_t(h);
        // plane offsets in 32 bits: the launcher routes batches of >= 4 GiB elsewhere
        const uint32_t plane = uint32_t(W) * uint32_t(H);
        const uint32_t fref = seq * uint32_t(a.b.F) + uint32_t(p);
        const uint32_t oref = fref * plane, ocur = oref + uint32_t(a.b.d) * plane;
        const int x0 = h * 8, y0 = v * 8;
        const int lo_x = max(-2 * S, -2 * x0), hi_x = min(2 * S, 2 * (W - x0 - 8));
        const int lo_y = max(-2 * S, -2 * y0), hi_y = min(2 * S, 2 * (H - y0 - 8));
        // --- round A: current block rows (lanes 0..7) and the candidates' MV
        // words (lanes 0..3) in flight together
        uint2 crow = make_uint2(0u, 0u);
        if (lane < 8)
            crow = __ldg(reinterpret_cast<const uint2*>(a.b.luma + (ocur + uint32_t(y0 + lane) * W + uint32_t(x0))));
        // a candidate's 16 x 32-byte reference patch into slot `slot` (cp.async:
        // lane = patch row x 16-byte chunk; zero-fill outside the frame)
        auto stage = [&](int slot, int cpx, int cpy) {
            const int r = lane >> 1, ch = lane & 1;
            const int cs = ((x0 + cpx - 4) & ~15) + 16 * ch;
            const int y = clampi(y0 + cpy - 4 + r, 0, H - 1);
            const uint8_t* rowp = a.b.luma + (oref + uint32_t(y) * W);
            const bool in = cs >= 0 && cs + 16 <= W;
            cp_async16(patch + slot * kFastPatch + r * kFastPWW + 4 * ch, in ? rowp + cs : rowp, in);
        };
        // window mode: frame row wy0 / 16-aligned column cs0 are the window's origin
        int wy0 = 0, cs0 = 0;
        if (wsw) {
            wy0 = y0 + (lo_y >> 1) - 4;
            cs0 = (x0 + (lo_x >> 1) - 4) & ~15;
            const int nch = ((((x0 + (hi_x >> 1) - 4) & ~15) + 32) - cs0) >> 4, nr = ((hi_y - lo_y) >> 1) + 16;
            const float inv_nch = 1.0f / float(nch);
            for (int i = lane; i < nr * nch; i += 32) {
                // row by a float reciprocal: exact, (i + 0.5) / nch is never within 0.5 / nch of an integer
                const int r = __float2int_rz((float(i) + 0.5f) * inv_nch), ch = i - r * nch;
                const int y = clampi(wy0 + r, 0, H - 1), col = cs0 + 16 * ch;
                const uint8_t* rowp = a.b.luma + (oref + uint32_t(y) * W);
                const bool in = col >= 0 && col + 16 <= W;
                cp_async16(patch + r * wsw + 4 * ch, in ? rowp + col : rowp, in);
            }
        }
        // boundary blocks (byte masks, window mode): the reference alpha over
        // the candidates' reach (rows y0 + lo_y/2 .. y0 + hi_y/2 + 7, the same
        // for columns) and this lane's current alpha row, also before the wait
        const int awsw = a.awin_words;
        uint32_t* awin = patch + (2 * S + 16) * wsw;
        int wya0 = 0, csa0 = 0;
        uint2 cal_pre = make_uint2(0u, 0u);
        if (awsw && boundary) {
            wya0 = y0 + (lo_y >> 1);
            csa0 = (x0 + (lo_x >> 1)) & ~15;
            const int nch = (((x0 + (hi_x >> 1) + 8 + 15) & ~15) - csa0) >> 4, nr = ((hi_y - lo_y) >> 1) + 8;
            const float inv_nch = 1.0f / float(nch);
            for (int i = lane; i < nr * nch; i += 32) {
                const int r = __float2int_rz((float(i) + 0.5f) * inv_nch), ch = i - r * nch;
                const int col = csa0 + 16 * ch;
                const uint8_t* rowp = a.b.alpha + (oref + uint32_t(wya0 + r) * W);
                const bool in = col >= 0 && col + 16 <= W;
                cp_async16(awin + r * awsw + 4 * ch, in ? rowp + col : rowp, in);
            }
            cal_pre = __ldg(reinterpret_cast<const uint2*>(a.b.alpha + (ocur + uint32_t(y0 + sub) * W + uint32_t(x0))));
        }
        const int PWW = wsw ? wsw : kFastPWW;
        // a candidate's patch view: row 0 = frame row y0 + cpy - 4, word 0 = the
        // 16-aligned column at or left of x0 + cpx - 4
        auto pbase = [&](int slot, int cpx, int cpy) -> const uint32_t* {
            return wsw ? patch + (y0 + cpy - 4 - wy0) * wsw + ((((x0 + cpx - 4) & ~15) - cs0) >> 2) : patch + slot * kFastPatch;
        };
        uint32_t mvw = 0;
        bool b_early;
        {
            int back = -1;  // records back from g: A 1, B cols, C cols - 1, T rows * cols
            if (lane == 0 && h > 0) back = 1;
            if (lane == 1 && v > 0) back = int(cols);
            if (lane == 2 && v > 0 && uint32_t(h) + 1 < cols) back = int(cols) - 1;
            if (lane == 3 && p > 0) back = int(rows * cols);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(a.recs + (g - uint32_t(back)));
            if (back >= 0) mvw = ld_relaxed(src);
            if (lane == 3 && p == 0 && a.prev0) {  // pair 0: T from the external (integer-pel) field
                const int i = v * int(cols) + h;
                mvw = pack_mv(a.prev0[2 * i], a.prev0[2 * i + 1]);
            }
            // B lies two wavefront steps back and is usually final already: its
            // patch (slot 1) goes out before the wait for A, C and T
            const uint32_t mb = __shfl_sync(0xFFFFFFFFu, mvw, 1);
            b_early = mb != kSentinel && !wsw;
            if (b_early) stage(1, clip_comp(mv_dx(mb), lo_x, hi_x) >> 1, clip_comp(mv_dy(mb), lo_y, hi_y) >> 1);
            // warp-uniform wait (a vote per poll keeps the warp converged)
            while (__any_sync(0xFFFFFFFFu, back >= 0 && mvw == kSentinel)) {
                __nanosleep(a.poll_ns);
                if (back >= 0 && mvw == kSentinel) mvw = ld_relaxed(src);
            }
        }
        if (TRACE) {
            t_ready = gtimer();
            c_ready = clock64();
        }
        if (lane < 8) {
            cw[2 * lane] = crow.x;
            cw[2 * lane + 1] = crow.y;
        }
        __syncwarp();  // reconverge after the polls (else the shuffles below take the divergent path)
        // my candidate (lanes 8c..8c+7 serve candidate c), clip_to_window (:275-276)
        const uint32_t mine = __shfl_sync(0xFFFFFFFFu, mvw, c);
        const int myx = clip_comp(mv_dx(mine), lo_x, hi_x), myy = clip_comp(mv_dy(mine), lo_y, hi_y);
        // duplicate candidates share a patch: B's slot first (it may be staged
        // already), else the first equal candidate's.  Window mode needs no
        // patch slots (and skips these dependent shuffles: the per-block
        // latency is a chain of ~30-cycle shuffle / shared-memory steps)
        int md = c;
        if (!wsw) {
            const int bx = __shfl_sync(0xFFFFFFFFu, myx, 8), by = __shfl_sync(0xFFFFFFFFu, myy, 8);
#pragma unroll
            for (int j = 2; j >= 0; --j) {
                const int jx = __shfl_sync(0xFFFFFFFFu, myx, 8 * j), jy = __shfl_sync(0xFFFFFFFFu, myy, 8 * j);
                if (j < c && jx == myx && jy == myy) md = j;
            }
            if (bx == myx && by == myy) md = 1;
            // --- round B: the remaining distinct patches and the shape rows in flight
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int ccx = __shfl_sync(0xFFFFFFFFu, myx, 8 * cc) >> 1;
                const int ccy = __shfl_sync(0xFFFFFFFFu, myy, 8 * cc) >> 1;
                const bool own = __shfl_sync(0xFFFFFFFFu, md, 8 * cc) == cc;  // warp-uniform
                if (own && !(cc == 1 && b_early)) stage(cc, ccx, ccy);
            }
        }
        const bool shape = boundary && (c < 3 || a.P.bt_shape);
        uint2 cal = make_uint2(0u, 0u);
        uint32_t ral0 = 0, ral1 = 0, xbits = 0;
        if (shape) {
            if (a.b.alpha_bits) {  // popc(XOR) of the 8 mask bits of my row
                const uint32_t wb = uint32_t(W) >> 3;
                const uint8_t* cb = a.b.alpha_bits + (ocur >> 3);
                const uint8_t* rb = a.b.alpha_bits + (oref >> 3);
                xbits = mask_bits8(cb, wb, x0, y0 + sub) ^ mask_bits8(rb, wb, x0 + (myx >> 1), y0 + sub + (myy >> 1));
            } else if (!awsw) {
                const uint32_t ao = uint32_t(y0 + sub) * W + uint32_t(x0);
                cal = __ldg(reinterpret_cast<const uint2*>(a.b.alpha + (ocur + ao)));
                ld8u(a.b.alpha + (oref + ao + uint32_t((myy >> 1) * W + (myx >> 1))), ral0, ral1);
            }
        }
        cp_async_wait_all();
        if (shape && awsw) {  // from the staged alpha window
            cal = cal_pre;
            prow8(awin + (y0 + sub + (myy >> 1) - wya0) * awsw, x0 + (myx >> 1) - csa0, ral0, ral1);
        }
        // shape scores (boundary blocks): my candidate, my row
        uint32_t s = 0;
        if (shape)
            s = (a.b.alpha_bits ? __popc(xbits) : (__popc(__vcmpne4(cal.x, ral0)) + __popc(__vcmpne4(cal.y, ral1))) >> 3) *
                (255u * 4u);
        __syncwarp();
        if (TRACE) c_patch = clock64();
        // --- brs_select (estimators.cpp:257-301) --------------------------------
        const uint32_t c0 = cw[2 * sub], c1 = cw[2 * sub + 1];  // my BRS row of the block
        if (!shape) {
            const int po = (x0 + (myx >> 1) - 4) & 15;
            uint32_t w0, w1;
            prow8(pbase(md, myx >> 1, myy >> 1) + (4 + sub) * PWW, 4 + po, w0, w1);
            s = vad4(c1, w1, vad4(c0, w0, 0u)) * 4u;
        }
        s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
        s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
        s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
        // strict <: A, B, C, T tie order (:295) = the minimum of (score, candidate)
        // (scores < 2^20), one warp reduction
        const uint32_t bk = __reduce_min_sync(0xFFFFFFFFu, (s << 2) | uint32_t(c));
        const uint32_t best = bk >> 2;
        const int win = int(bk & 3u);
        const bool win_shape = boundary && (win < 3 || a.P.bt_shape);
        const int wx = __shfl_sync(0xFFFFFFFFu, myx, 8 * win), wy = __shfl_sync(0xFFFFFFFFu, myy, 8 * win);
        const int wp = __shfl_sync(0xFFFFFFFFu, md, 8 * win);
        const uint32_t* pw = pbase(wp, wx >> 1, wy >> 1);
        const int wo = (x0 + (wx >> 1) - 4) & 15;  // the winner patch's byte offset
        // my two PRS rows of the block
        const uint32_t ra0 = cw[2 * q], ra1 = cw[2 * q + 1], rb0 = cw[2 * q + 8], rb1 = cw[2 * q + 9];
        uint32_t ccost = best;
        if (win_shape) {  // the centre's texture cost was not computed by BRS
            uint32_t w0, w1;
            prow8(pw + (4 + sub) * PWW, 4 + wo, w0, w1);
            uint32_t t = c == 0 ? vad4(c1, w1, vad4(c0, w0, 0u)) : 0u;
            ccost = 4u * __reduce_add_sync(0xFFFFFFFFu, t);
        }
        if (TRACE) c_brs = clock64();
        // --- prs_refine (estimators.cpp:311-382), lazily from the patch ---------
        int ci = 0, cj = 0, pc0 = 0, pc1 = 0, pc2 = 0;  // earlier centres (see pa_duo_kernel)
        uint32_t dpd = 1, iters = 0;
        for (int it = 0; it < a.P.max_iter; ++it) {
            if (ccost == 0) break;  // already a global minimum (:341)
            const int px = ci + kx, py = cj + ky;
            const bool adm = wx + 2 * px >= lo_x && wx + 2 * px <= hi_x && wy + 2 * py >= lo_y && wy + 2 * py <= hi_y;
            uint32_t w0, w1, w2, w3;
            prow8(pw + (4 + py + q) * PWW, 4 + px + wo, w0, w1);
            prow8(pw + (8 + py + q) * PWW, 4 + px + wo, w2, w3);
            uint32_t part = vad4(rb1, w3, vad4(rb0, w2, vad4(ra1, w1, vad4(ra0, w0, 0u))));
            part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
            part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
            const uint32_t cost = 4u * part;
            const bool lead = adm && q == 0;
            // unique aggregate evaluations (:321-332): new iff at Chebyshev
            // distance >= 2 from every earlier centre
            auto far = [&](int pc) { return max(abs(px + 8 - (pc & 15)), abs(py + 8 - (pc >> 4))) >= 2; };
            bool fresh = lead;
            if (it >= 1) fresh = fresh && far(pc0);
            if (it >= 2) fresh = fresh && far(pc1);
            if (it >= 3) fresh = fresh && far(pc2);
            dpd += __popc(__ballot_sync(0xFFFFFFFFu, fresh));
            const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, lead ? cost : kInf);
            if (m >= ccost) break;  // centre kept (:376)
            const uint32_t ties = __ballot_sync(0xFFFFFFFFu, lead && cost == m);
            int w;
            if (__popc(ties) == 1) {
                w = (__ffs(ties) - 1) >> 2;
            } else {
                // stable descending sort by off . dir (:357-362): the first tied
                // neighbour in sorted order = largest key, lowest index on equal keys
                PaBlock B;
                B.cur = a.b.luma + ocur;
                B.ref = a.b.luma + oref;
                B.ca = B.ra = nullptr;
                B.x0 = x0;
                B.y0 = y0;
                double dir_x, dir_y;
                prs_direction(a.P, B, lane, wx + 2 * ci, wy + 2 * cj, dir_x, dir_y);
                w = -1;
                double bestkey = 0.0;
                for (int o = 0; o < 8; ++o) {
                    if (!((ties >> (4 * o)) & 1u)) continue;
                    const double key = __dadd_rn(__dmul_rn(double(c_off8[o][0]), dir_x), __dmul_rn(double(c_off8[o][1]), dir_y));
                    if (w < 0 || key > bestkey) {
                        w = o;
                        bestkey = key;
                    }
                }
            }
            const int pc = (ci + 8) | ((cj + 8) << 4);
            if (it == 0) pc0 = pc;
            if (it == 1) pc1 = pc;
            if (it == 2) pc2 = pc;
            ci += off8x(w);
            cj += off8y(w);
            ccost = m;
            ++iters;
        }
        if (TRACE) c_walk = clock64();
        // publish first (the dependents wait on the record, not on the SSE)
        if (lane == 0) write_rec_v4(a.recs + g, wx + 2 * ci, wy + 2 * cj, ccost, 4, dpd, iters, boundary ? ME_BOUNDARY : ME_OPAQUE);
        // --- fused predict_frame + psnr SSE at the final vector -----------------
        uint32_t se = 0;
        if (lane < 8) {
            uint32_t w0, w1;
            prow8(pw + (4 + cj + lane) * PWW, 4 + ci + wo, w0, w1);
            se = sq4(cw[2 * lane + 1], w1, sq4(cw[2 * lane], w0, 0u));
        }
        se = __reduce_add_sync(0xFFFFFFFFu, se);
        if (lane == 0) {
            if (a.stats) add_stats_pa(a.stats + pair, se, dpd);
            if (TRACE) {  // as pa_duo_kernel
                unsigned long long* tr = a.trace + size_t(item) * 4;
                const long long c_end = clock64();
                auto c16 = [](long long d) { return (unsigned long long)min(max(d, 0ll), 65535ll); };
                tr[0] = t_claim;
                tr[1] = t_ready;
                tr[2] = gtimer();
                tr[3] = c16(c_patch - c_ready) | (c16(c_brs - c_patch) << 16) | (c16(c_walk - c_brs) << 32) |
                        (c16(c_end - c_walk) << 48);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// pa_duo_kernel: pa_fast_kernel's algorithm with TWO blocks per warp, one per
// half-warp, so the per-block scalar work (decode, window, candidate
// bookkeeping, reductions, loop control) is issued once for two blocks.  The
// two blocks are consecutive list entries of the same wavefront step (the
// sort pads every step to an even count), hence independent.  Patches are
// staged with cp.async (no register staging).  Lanes of a half: BRS =
// candidate x rows {q, q+4}; PRS = neighbour x rows {q, q+2, q+4, q+6}.
// ---------------------------------------------------------------------------

#ifndef ME_DUO_PWW
#define ME_DUO_PWW 8
#endif
constexpr int kDuoPWW = ME_DUO_PWW;            // patch row stride in words (8 used)
constexpr int kDuoPatch = kFastPR * kDuoPWW;
constexpr int kDuoTaskWords = 4 * kDuoPatch + 16 + 4;  // patches, current block, visited
constexpr int kDuoWarpWords = 2 * kDuoTaskWords;


template <int THREADS, int MINB, bool TRACE = false>
__global__ void __launch_bounds__(THREADS, MINB) pa_duo_kernel(const PaArgs a) {
    extern __shared__ uint32_t s_pa[];
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int hf = lane >> 4, hl = lane & 15, hb = hf << 4;
    const uint32_t hmask = hf ? 0xFFFF0000u : 0x0000FFFFu;
    uint32_t* ws = s_pa + wid * kDuoWarpWords;
    uint32_t* patch = ws + hf * kDuoTaskWords;  // [4][16][12]
    uint32_t* cw = patch + 4 * kDuoPatch;      // [8][2] current block
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int beg = a.range ? a.range[0] : 0, n = a.range ? a.range[1] : *a.nlist;  // beg, n even
    const int W = a.b.W, H = a.b.H, S = a.P.S;
    const uint32_t cols = a.b.cols, rows = a.b.rows, pairs = a.b.pairs;
    const uint32_t plane = uint32_t(W) * uint32_t(H);
    const int c = hl >> 2, q4 = hl & 3;  // BRS: candidate c, block rows q4 and q4 + 4
    const int k = hl >> 1, q2 = hl & 1;  // PRS: neighbour k, block rows q2 + {0, 2, 4, 6}
    const int kx = off8x(k), ky = off8y(k);
    __shared__ int s_claim[2 + 2 * kClaimRing];
    CtaClaim cc{s_claim, a.claim, 0};
    CtaClaim::init(s_claim);
    int nxt = 0;
    for (int rel = a.claim ? cc.next<2>(lane, wid, blockDim.x >> 5) : 2 * (blockIdx.x * (blockDim.x >> 5) + wid); beg + rel < n;
         rel = a.claim ? cc.next<2>(lane, wid, blockDim.x >> 5) : nxt) {
        nxt = a.claim ? 0 : rel + 2 * nwarps;
        const int item = beg + rel;
        const uint2 e = __ldg(a.list + item + hf);
        const bool act = e.x != kInvalidEntry;  // uniform per half
        unsigned long long t_claim = 0, t_ready = 0;
        if (TRACE) t_claim = gtimer();
        if (!__any_sync(FULL, act)) continue;
        const int h = int(e.x & 0xFFFF), v = int((e.x >> 16) & 0x7FFF), p = int(e.y & 0xFFFF);
        const uint32_t seq = e.y >> 16;
        const bool boundary = (e.x & kBoundaryBit) != 0;
        const uint32_t pair = seq * pairs + uint32_t(p);
        const uint32_t g = (pair * rows + uint32_t(v)) * cols + uint32_t(h);
        const uint32_t fref = seq * uint32_t(a.b.F) + uint32_t(p);
        const uint32_t oref = fref * plane, ocur = oref + uint32_t(a.b.d) * plane;
        const int x0 = h * 8, y0 = v * 8;
        const int lo_x = max(-2 * S, -2 * x0), hi_x = min(2 * S, 2 * (W - x0 - 8));
        const int lo_y = max(-2 * S, -2 * y0), hi_y = min(2 * S, 2 * (H - y0 - 8));
        // --- round A: current rows (lanes 0..7 of a half) + MV words (0..3) ----
        uint2 crow = make_uint2(0u, 0u);
        if (act && hl < 8)
            crow = __ldg(reinterpret_cast<const uint2*>(a.b.luma + (ocur + uint32_t(y0 + hl) * W + uint32_t(x0))));
        // a candidate's 16 x 32-byte reference patch into slot `slot` (cp.async,
        // lane = patch row, two 16-byte chunks; zero-fill outside the frame)
        auto stage = [&](int slot, int cpx, int cpy) {
            const int cs = (x0 + cpx - 4) & ~15;
            const int y = clampi(y0 + cpy - 4 + hl, 0, H - 1);
            const uint8_t* rowp = a.b.luma + (oref + uint32_t(y) * W);
            uint32_t* dst = patch + slot * kDuoPatch + hl * kDuoPWW;
            const bool in0 = cs >= 0 && cs + 16 <= W, in1 = cs + 16 >= 0 && cs + 32 <= W;
            cp_async16(dst, in0 ? rowp + cs : rowp, in0);
            cp_async16(dst + 4, in1 ? rowp + cs + 16 : rowp, in1);
        };
        uint32_t mvw = 0;
        {
            int back = -1;  // records back from g: A 1, B cols, C cols - 1, T rows * cols
            if (act && hl == 0 && h > 0) back = 1;
            if (act && hl == 1 && v > 0) back = int(cols);
            if (act && hl == 2 && v > 0 && uint32_t(h) + 1 < cols) back = int(cols) - 1;
            if (act && hl == 3 && p > 0) back = int(rows * cols);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(a.recs + (g - uint32_t(back)));
            if (back >= 0) mvw = ld_relaxed(src);
            // warp-uniform wait (a vote per poll keeps the warp converged)
            while (__any_sync(FULL, back >= 0 && mvw == kSentinel)) {
                __nanosleep(a.poll_ns);
                if (back >= 0 && mvw == kSentinel) mvw = ld_relaxed(src);
            }
        }
        long long c_ready = 0;
        if (TRACE) {
            t_ready = gtimer();
            c_ready = clock64();
        }
        if (hl < 8) {
            cw[2 * hl] = crow.x;
            cw[2 * hl + 1] = crow.y;
        }
        __syncwarp();
        // my candidate, clip_to_window (:275-276)
        const uint32_t mine = __shfl_sync(FULL, mvw, hb + c);
        const int myx = clip_comp(mv_dx(mine), lo_x, hi_x), myy = clip_comp(mv_dy(mine), lo_y, hi_y);
        // duplicate candidates share a patch: B's slot first, else the first
        // equal candidate's (B is staged early in pa_fast_kernel; this
        // throughput-bound kernel stages all candidates in one round — measured
        // 0.7 % faster)
        int md = c;
        {
            const int bx = __shfl_sync(FULL, myx, hb + 4), by = __shfl_sync(FULL, myy, hb + 4);
#pragma unroll
            for (int j = 2; j >= 0; --j) {
                const int jx = __shfl_sync(FULL, myx, hb + 4 * j), jy = __shfl_sync(FULL, myy, hb + 4 * j);
                if (j < c && jx == myx && jy == myy) md = j;
            }
            if (bx == myx && by == myy) md = 1;
        }
        // --- round B: patches of the distinct candidates and the shape rows,
        // all in flight together ---------------------------------------------
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int ccx = __shfl_sync(FULL, myx, hb + 4 * cc) >> 1;
            const int ccy = __shfl_sync(FULL, myy, hb + 4 * cc) >> 1;
            const bool own = __shfl_sync(FULL, md, hb + 4 * cc) == cc;  // uniform per half
            if (act && own) stage(cc, ccx, ccy);
        }
        const bool shape = act && boundary && (c < 3 || a.P.bt_shape);
        uint2 ca0 = make_uint2(0u, 0u), ca1 = ca0;
        uint32_t r00 = 0, r01 = 0, r10 = 0, r11 = 0;
        if (shape) {
            const uint32_t ao = uint32_t(y0 + q4) * W + uint32_t(x0);
            const uint8_t* cap = a.b.alpha + (ocur + ao);
            const uint8_t* rap = a.b.alpha + (oref + ao + uint32_t((myy >> 1) * W + (myx >> 1)));
            ca0 = __ldg(reinterpret_cast<const uint2*>(cap));
            ca1 = __ldg(reinterpret_cast<const uint2*>(cap + 4 * W));
            ld8u(rap, r00, r01);
            ld8u(rap + 4 * W, r10, r11);
        }
        cp_async_wait_all();
        __syncwarp();
        long long c_patch = 0;
        if (TRACE) c_patch = clock64();
        // --- brs_select (estimators.cpp:257-301) ------------------------------
        uint32_t s;
        if (shape) {
            s = ((__popc(__vcmpne4(ca0.x, r00)) + __popc(__vcmpne4(ca0.y, r01)) + __popc(__vcmpne4(ca1.x, r10)) +
                  __popc(__vcmpne4(ca1.y, r11))) >> 3) * (255u * 4u);
        } else {
            const int po = (x0 + (myx >> 1) - 4) & 15;
            const uint32_t* pr = patch + md * kDuoPatch + (4 + q4) * kDuoPWW;
            uint32_t w0, w1, w2, w3;
            prow8(pr, 4 + po, w0, w1);
            prow8(pr + 4 * kDuoPWW, 4 + po, w2, w3);
            s = vad4(cw[2 * q4 + 9], w3, vad4(cw[2 * q4 + 8], w2, vad4(cw[2 * q4 + 1], w1, vad4(cw[2 * q4], w0, 0u)))) * 4u;
        }
        s += __shfl_xor_sync(FULL, s, 1);  // the candidate's 4 lanes
        s += __shfl_xor_sync(FULL, s, 2);
        uint32_t best = __shfl_sync(FULL, s, hb);
        int win = 0;
#pragma unroll
        for (int i = 1; i < 4; ++i) {
            const uint32_t si = __shfl_sync(FULL, s, hb + 4 * i);
            if (si < best) {  // strict <: A, B, C, T tie order (:295)
                best = si;
                win = i;
            }
        }
        const bool win_shape = boundary && (win < 3 || a.P.bt_shape);
        const int wx = __shfl_sync(FULL, myx, hb + 4 * win), wy = __shfl_sync(FULL, myy, hb + 4 * win);
        const int wp = __shfl_sync(FULL, md, hb + 4 * win);
        const uint32_t* pw = patch + wp * kDuoPatch;
        const int wo = (x0 + (wx >> 1) - 4) & 15;  // the winner patch's byte offset
        uint32_t ccost = best;
        if (__any_sync(FULL, act && win_shape)) {  // the centre's texture cost was not computed by BRS
            uint32_t w0, w1, w2, w3;
            prow8(pw + (4 + q4) * kDuoPWW, 4 + wo, w0, w1);
            prow8(pw + (8 + q4) * kDuoPWW, 4 + wo, w2, w3);
            uint32_t t = c == 0 ? vad4(cw[2 * q4 + 9], w3, vad4(cw[2 * q4 + 8], w2, vad4(cw[2 * q4 + 1], w1, vad4(cw[2 * q4], w0, 0u)))) : 0u;
            t += __shfl_xor_sync(FULL, t, 1);
            t += __shfl_xor_sync(FULL, t, 2);
            t = __shfl_sync(FULL, t, hb);
            if (win_shape) ccost = 4u * t;
        }
        long long c_brs = 0;
        if (TRACE) c_brs = clock64();
        // --- prs_refine (estimators.cpp:311-382), lazily from the patch -------
        int ci = 0, cj = 0;
        uint32_t dpd = 1, iters = 0;
        bool alive = act;
        // earlier centres (relative to the start; at most 3 before the 4th
        // iteration): a neighbour q is a fresh evaluation (:321-332) iff it is
        // at Chebyshev distance >= 2 from every earlier centre (every position
        // within distance 1 of one was evaluated then, the start included)
        int pc0 = 0, pc1 = 0, pc2 = 0;  // packed (x + 8) | (y + 8) << 4
        for (int it = 0; it < a.P.max_iter; ++it) {
            alive = alive && ccost != 0;  // already a global minimum (:341)
            if (!__any_sync(FULL, alive)) break;
            const int px = ci + kx, py = cj + ky;
            const bool adm = wx + 2 * px >= lo_x && wx + 2 * px <= hi_x && wy + 2 * py >= lo_y && wy + 2 * py <= hi_y;
            const uint32_t* pr = pw + (4 + py + q2) * kDuoPWW;
            const int tt = 4 + px + wo;
            uint32_t w0, w1, part = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // block rows q2 + 2i (current rows re-read from smem: registers)
                const uint2 cr = *reinterpret_cast<const uint2*>(cw + 2 * q2 + 4 * i);
                prow8(pr + 2 * i * kDuoPWW, tt, w0, w1);
                part = vad4(cr.y, w1, vad4(cr.x, w0, part));
            }
            part += __shfl_xor_sync(FULL, part, 1);
            const uint32_t cost = 4u * part;
            const bool lead = alive && adm && q2 == 0;
            bool fresh = lead;
            auto far = [&](int pc) { return max(abs(px + 8 - (pc & 15)), abs(py + 8 - (pc >> 4))) >= 2; };
            if (it >= 1) fresh = fresh && far(pc0);
            if (it >= 2) fresh = fresh && far(pc1);
            if (it >= 3) fresh = fresh && far(pc2);
            dpd += __popc(__ballot_sync(FULL, fresh) & hmask);
            // per-half minimum: two independent full-warp reductions (a
            // half-mask reduction would serialise the halves)
            const uint32_t mine_c = lead ? cost : kInf;
            const uint32_t m0 = __reduce_min_sync(FULL, hf ? kInf : mine_c);
            const uint32_t m1 = __reduce_min_sync(FULL, hf ? mine_c : kInf);
            const uint32_t m = hf ? m1 : m0;
            const bool move = alive && m < ccost;  // else the centre is kept (:376)
            const uint32_t ties = (__ballot_sync(FULL, lead && cost == m) & hmask) >> hb;
            int w = (__ffs(ties) - 1) >> 1;
            const bool tie = move && __popc(ties) > 1;
            if (__any_sync(FULL, tie)) {
                // stable descending sort by off . dir (:357-362), computed with the
                // full warp for each half that needs it
#pragma unroll 1
                for (int t = 0; t < 2; ++t) {
                    if (!__shfl_sync(FULL, tie, 16 * t)) continue;  // warp-uniform
                    PaBlock B;
                    B.cur = a.b.luma + __shfl_sync(FULL, ocur, 16 * t);
                    B.ref = a.b.luma + __shfl_sync(FULL, oref, 16 * t);
                    B.ca = B.ra = nullptr;
                    B.x0 = __shfl_sync(FULL, x0, 16 * t);
                    B.y0 = __shfl_sync(FULL, y0, 16 * t);
                    const int cx = __shfl_sync(FULL, wx + 2 * ci, 16 * t), cy = __shfl_sync(FULL, wy + 2 * cj, 16 * t);
                    double dir_x, dir_y;
                    prs_direction(a.P, B, lane, cx, cy, dir_x, dir_y);
                    if (hf == t) {
                        int wb = -1;
                        double bestkey = 0.0;
                        for (int o = 0; o < 8; ++o) {
                            if (!((ties >> (2 * o)) & 1u)) continue;
                            const double key = __dadd_rn(__dmul_rn(double(c_off8[o][0]), dir_x), __dmul_rn(double(c_off8[o][1]), dir_y));
                            if (wb < 0 || key > bestkey) {
                                wb = o;
                                bestkey = key;
                            }
                        }
                        w = wb;
                    }
                }
            }
            const int pc = (ci + 8) | ((cj + 8) << 4);
            if (it == 0) pc0 = pc;
            if (it == 1) pc1 = pc;
            if (it == 2) pc2 = pc;
            if (move) {
                ci += off8x(w);
                cj += off8y(w);
                ccost = m;
                ++iters;
            }
            alive = move;
        }
        long long c_walk = 0;
        if (TRACE) c_walk = clock64();
        // publish first (the dependents wait on the record, not on the SSE)
        if (act && hl == 0)
            write_rec_v4(a.recs + g, wx + 2 * ci, wy + 2 * cj, ccost, 4, dpd, iters, boundary ? ME_BOUNDARY : ME_OPAQUE);
        // --- fused predict_frame + psnr SSE at the final vector ---------------
        uint32_t se = 0;
        if (hl < 8) {
            uint32_t w0, w1;
            prow8(pw + (4 + cj + hl) * kDuoPWW, 4 + ci + wo, w0, w1);
            se = sq4(cw[2 * hl + 1], w1, sq4(cw[2 * hl], w0, 0u));
        }
        {
            const uint32_t s0 = __reduce_add_sync(FULL, hf ? 0u : se), s1 = __reduce_add_sync(FULL, hf ? se : 0u);
            se = hf ? s1 : s0;
        }
        if (act && hl == 0) {
            if (a.stats) add_stats_pa(a.stats + pair, se, dpd);
            if (TRACE) {  // {claimed, dependencies ready, published (globaltimer ns), phase cycles}
                unsigned long long* tr = a.trace + size_t(item + hf) * 4;
                const long long c_end = clock64();
                auto c16 = [](long long d) { return (unsigned long long)min(max(d, 0ll), 65535ll); };
                tr[0] = t_claim;
                tr[1] = t_ready;
                tr[2] = gtimer();
                // SM cycles: ready -> patches staged, -> BRS done, -> walk done, -> published
                tr[3] = c16(c_patch - c_ready) | (c16(c_brs - c_patch) << 16) | (c16(c_walk - c_brs) << 32) |
                        (c16(c_end - c_walk) << 48);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// pa_quad_kernel: pa_duo_kernel's algorithm with FOUR blocks per warp, one per
// 8-lane group.  The per-block bookkeeping is issued once for four blocks and
// every lane of a group evaluates one PRS neighbour over all 8 block rows, so
// the walk needs no cross-lane SAD reduction.  Patches are 16 rows x 24 bytes
// (three 8-byte cp.async chunks): the block's 8 columns plus the walk's +-4.
// Lanes of a group: BRS = candidate (gl >> 1) x rows 4 (gl & 1) .. +3; PRS =
// neighbour gl x all rows.  The sort pads every wide step to a multiple of 4.
// ---------------------------------------------------------------------------

constexpr int kQuadPWW = 6;                               // patch row stride in words (24 bytes)
constexpr int kQuadPatch = kFastPR * kQuadPWW;            // 96 words
constexpr int kQuadTaskWords = 4 * kQuadPatch + 16 + 8;   // patches, current block, bank skew
constexpr int kQuadWarpWords = 4 * kQuadTaskWords;


template <int MINB, bool TRACE = false>
__global__ void __launch_bounds__(256, MINB) pa_quad_kernel(const PaArgs a) {
    const PdlScope pdl_scope(a.pdl);
    extern __shared__ uint32_t s_pa[];
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int grp = lane >> 3, gl = lane & 7, gb = grp << 3;
    const uint32_t gmask = 0xFFu << gb;
    uint32_t* patch = s_pa + wid * kQuadWarpWords + grp * kQuadTaskWords;  // [4][16][6]
    uint32_t* cw = patch + 4 * kQuadPatch;                                 // [8][2] current block
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int beg = a.range ? a.range[0] : 0, n = a.range ? a.range[1] : *a.nlist;  // multiples of 4
    const int W = a.b.W, H = a.b.H, S = a.P.S;
    const uint32_t cols = a.b.cols, rows = a.b.rows, pairs = a.b.pairs;
    const uint32_t plane = uint32_t(W) * uint32_t(H);
    const int c = gl >> 1, hh = gl & 1;      // BRS: candidate c, block rows 4 hh .. 4 hh + 3
    const int kx = off8x(gl), ky = off8y(gl);  // PRS: neighbour gl
    __shared__ int s_claim[2 + 2 * kClaimRing];
    CtaClaim cc{s_claim, a.claim, 0};
    CtaClaim::init(s_claim);
    int nxt = 0;
    for (int rel = a.claim ? cc.next<4>(lane, wid, blockDim.x >> 5) : 4 * (blockIdx.x * (blockDim.x >> 5) + wid); beg + rel < n;
         rel = a.claim ? cc.next<4>(lane, wid, blockDim.x >> 5) : nxt) {
        nxt = a.claim ? 0 : rel + 4 * nwarps;
        const int item = beg + rel;
        const uint2 e = __ldg(a.list + item + grp);
        const bool act = e.x != kInvalidEntry;  // uniform per group
        unsigned long long t_claim = 0, t_ready = 0;
        long long c_ready = 0, c_patch = 0, c_brs = 0, c_walk = 0;
        if (TRACE) t_claim = gtimer();
        if (!__any_sync(FULL, act)) continue;
        const int h = int(e.x & 0xFFFF), v = int((e.x >> 16) & 0x7FFF), p = int(e.y & 0xFFFF);
        const uint32_t seq = e.y >> 16;
        const bool boundary = (e.x & kBoundaryBit) != 0;
        const uint32_t pair = seq * pairs + uint32_t(p);
        const uint32_t g = (pair * rows + uint32_t(v)) * cols + uint32_t(h);
        const uint32_t oref = (seq * uint32_t(a.b.F) + uint32_t(p)) * plane, ocur = oref + uint32_t(a.b.d) * plane;
        const int x0 = h * 8, y0 = v * 8;
        const int lo_x = max(-2 * S, -2 * x0), hi_x = min(2 * S, 2 * (W - x0 - 8));
        const int lo_y = max(-2 * S, -2 * y0), hi_y = min(2 * S, 2 * (H - y0 - 8));
        // --- round A: current row gl + MV words (gl 0..3) ---------------------
        uint2 crow = make_uint2(0u, 0u);
        if (act) crow = __ldg(reinterpret_cast<const uint2*>(a.b.luma + (ocur + uint32_t(y0 + gl) * W + uint32_t(x0))));
        uint32_t mvw = 0;
        {
            int back = -1;  // records back from g: A 1, B cols, C cols - 1, T rows * cols
            if (act && gl == 0 && h > 0) back = 1;
            if (act && gl == 1 && v > 0) back = int(cols);
            if (act && gl == 2 && v > 0 && uint32_t(h) + 1 < cols) back = int(cols) - 1;
            if (act && gl == 3 && p > 0) back = int(rows * cols);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(a.recs + (g - uint32_t(back)));
            if (back >= 0) mvw = ld_relaxed(src);
            while (__any_sync(FULL, back >= 0 && mvw == kSentinel)) {
                __nanosleep(a.poll_ns);
                if (back >= 0 && mvw == kSentinel) mvw = ld_relaxed(src);
            }
        }
        if (TRACE) {
            t_ready = gtimer();
            c_ready = clock64();
        }
        cw[2 * gl] = crow.x;
        cw[2 * gl + 1] = crow.y;
        // my candidate, clip_to_window (:275-276); duplicates share a patch
        const uint32_t mine = __shfl_sync(FULL, mvw, gb + c);
        const int myx = clip_comp(mv_dx(mine), lo_x, hi_x), myy = clip_comp(mv_dy(mine), lo_y, hi_y);
        int md = c;
        {
            const int bx = __shfl_sync(FULL, myx, gb + 2), by = __shfl_sync(FULL, myy, gb + 2);
#pragma unroll
            for (int j = 2; j >= 0; --j) {
                const int jx = __shfl_sync(FULL, myx, gb + 2 * j), jy = __shfl_sync(FULL, myy, gb + 2 * j);
                if (j < c && jx == myx && jy == myy) md = j;
            }
            if (bx == myx && by == myy) md = 1;
        }
        // --- round B: the distinct candidates' patches + the shape rows --------
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int ccx = __shfl_sync(FULL, myx, gb + 2 * cc) >> 1;
            const int ccy = __shfl_sync(FULL, myy, gb + 2 * cc) >> 1;
            const bool own = __shfl_sync(FULL, md, gb + 2 * cc) == cc;  // uniform per group
            if (act && own) {
                // 16 rows x 3 chunks; consecutive lanes take consecutive chunks
                const int cs = (x0 + ccx - 4) & ~7, ry0 = y0 + ccy - 4;
                uint32_t* dst = patch + cc * kQuadPatch;
                if (ry0 >= 0 && ry0 + kFastPR <= H && cs >= 0 && cs + 24 <= W) {
                    // the whole patch inside the frame (the common case): one base
                    const uint8_t* base = a.b.luma + (oref + uint32_t(ry0) * W + uint32_t(cs));
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        const int ci8 = gl + 8 * k, r = ci8 / 3, ch = ci8 - 3 * r;
                        cp_async8(dst + r * kQuadPWW + 2 * ch, base + (r * W + 8 * ch), true);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        const int ci8 = gl + 8 * k, r = ci8 / 3, ch = ci8 - 3 * r;
                        const int y = clampi(ry0 + r, 0, H - 1);
                        const int col = cs + 8 * ch;
                        const bool in = col >= 0 && col + 8 <= W;
                        const uint8_t* rowp = a.b.luma + (oref + uint32_t(y) * W);
                        cp_async8(dst + r * kQuadPWW + 2 * ch, in ? rowp + col : rowp, in);
                    }
                }
            }
        }
        const bool shape = act && boundary && (c < 3 || a.P.bt_shape);
        uint32_t sh_cnt = 0;  // mismatching mask samples x 8
        if (shape && a.b.alpha_bits) {  // bit-packed masks: popc(XOR) of 8-pel rows
            const uint32_t wb = uint32_t(W) >> 3;
            const uint8_t* cb = a.b.alpha_bits + (ocur >> 3);
            const uint8_t* rb = a.b.alpha_bits + (oref >> 3);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int y = y0 + 4 * hh + r;
                sh_cnt += __popc(mask_bits8(cb, wb, x0, y) ^ mask_bits8(rb, wb, x0 + (myx >> 1), y + (myy >> 1)));
            }
            sh_cnt <<= 3;
        } else if (shape) {
            const uint32_t ao = uint32_t(y0 + 4 * hh) * W + uint32_t(x0);
            const uint8_t* cap = a.b.alpha + (ocur + ao);
            const uint8_t* rap = a.b.alpha + (oref + ao + uint32_t((myy >> 1) * W + (myx >> 1)));
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint2 ca = __ldg(reinterpret_cast<const uint2*>(cap + r * W));
                uint32_t r0, r1;
                ld8u(rap + r * W, r0, r1);
                sh_cnt += __popc(__vcmpne4(ca.x, r0)) + __popc(__vcmpne4(ca.y, r1));
            }
        }
        cp_async_wait_all();
        __syncwarp();
        if (TRACE) c_patch = clock64();
        // --- brs_select (estimators.cpp:257-301) ------------------------------
        uint32_t s;
        if (shape) {
            s = (sh_cnt >> 3) * (255u * 4u);
        } else {
            const int po = (x0 + (myx >> 1) - 4) & 7;
            const uint32_t* pr = patch + md * kQuadPatch + (4 + 4 * hh) * kQuadPWW;
            uint32_t acc0 = 0, acc1 = 0;
#pragma unroll
            for (int r = 0; r < 4; r += 2) {
                const uint4 cr = *reinterpret_cast<const uint4*>(cw + 8 * hh + 2 * r);
                uint32_t w0, w1, w2, w3;
                prow8(pr + r * kQuadPWW, 4 + po, w0, w1);
                prow8(pr + (r + 1) * kQuadPWW, 4 + po, w2, w3);
                acc0 = vad4(cr.y, w1, vad4(cr.x, w0, acc0));
                acc1 = vad4(cr.w, w3, vad4(cr.z, w2, acc1));
            }
            s = (acc0 + acc1) * 4u;
        }
        s += __shfl_xor_sync(FULL, s, 1);  // the candidate's 2 lanes
        uint32_t best = __shfl_sync(FULL, s, gb);
        int win = 0;
#pragma unroll
        for (int i = 1; i < 4; ++i) {
            const uint32_t si = __shfl_sync(FULL, s, gb + 2 * i);
            if (si < best) {  // strict <: A, B, C, T tie order (:295)
                best = si;
                win = i;
            }
        }
        const bool win_shape = boundary && (win < 3 || a.P.bt_shape);
        const int wx = __shfl_sync(FULL, myx, gb + 2 * win), wy = __shfl_sync(FULL, myy, gb + 2 * win);
        const int wp = __shfl_sync(FULL, md, gb + 2 * win);
        const uint32_t* pw = patch + wp * kQuadPatch;
        const int wo = (x0 + (wx >> 1) - 4) & 7;  // the winner patch's byte offset
        uint32_t ccost = best;
        if (__any_sync(FULL, act && win_shape)) {  // the centre's texture cost was not computed by BRS
            uint32_t t = 0;
            if (c == 0) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint2 cr = *reinterpret_cast<const uint2*>(cw + 8 * hh + 2 * r);
                    uint32_t w0, w1;
                    prow8(pw + (4 + 4 * hh + r) * kQuadPWW, 4 + wo, w0, w1);
                    t = vad4(cr.y, w1, vad4(cr.x, w0, t));
                }
            }
            t += __shfl_xor_sync(FULL, t, 1);
            t = __shfl_sync(FULL, t, gb);
            if (win_shape) ccost = 4u * t;
        }
        if (TRACE) c_brs = clock64();
        // --- prs_refine (estimators.cpp:311-382), lazily from the patch -------
        int ci = 0, cj = 0;
        uint32_t dpd = 1, iters = 0;
        bool alive = act;
        int pc0 = 0, pc1 = 0, pc2 = 0;  // earlier centres, packed (x + 8) | (y + 8) << 4 (see pa_duo_kernel)
        for (int it = 0; it < a.P.max_iter; ++it) {
            alive = alive && ccost != 0;  // already a global minimum (:341)
            if (!__any_sync(FULL, alive)) break;
            const int px = ci + kx, py = cj + ky;
            const bool adm = wx + 2 * px >= lo_x && wx + 2 * px <= hi_x && wy + 2 * py >= lo_y && wy + 2 * py <= hi_y;
            const uint32_t* pr = pw + (4 + py) * kQuadPWW;
            const int tt = 4 + px + wo;
            uint32_t part0 = 0, part1 = 0;  // two accumulation chains
#pragma unroll
            for (int r = 0; r < 8; r += 2) {
                const uint4 cr = *reinterpret_cast<const uint4*>(cw + 2 * r);
                uint32_t w0, w1, w2, w3;
                prow8(pr + r * kQuadPWW, tt, w0, w1);
                prow8(pr + (r + 1) * kQuadPWW, tt, w2, w3);
                part0 = vad4(cr.y, w1, vad4(cr.x, w0, part0));
                part1 = vad4(cr.w, w3, vad4(cr.z, w2, part1));
            }
            const uint32_t cost = 4u * (part0 + part1);
            const bool lead = alive && adm;
            bool fresh = lead;
            auto far = [&](int pc) { return max(abs(px + 8 - (pc & 15)), abs(py + 8 - (pc >> 4))) >= 2; };
            if (it >= 1) fresh = fresh && far(pc0);
            if (it >= 2) fresh = fresh && far(pc1);
            if (it >= 3) fresh = fresh && far(pc2);
            dpd += __popc(__ballot_sync(FULL, fresh) & gmask);
            uint32_t m = lead ? cost : kInf;  // the group's minimum
            m = min(m, __shfl_xor_sync(FULL, m, 1));
            m = min(m, __shfl_xor_sync(FULL, m, 2));
            m = min(m, __shfl_xor_sync(FULL, m, 4));
            const bool move = alive && m < ccost;  // else the centre is kept (:376)
            const uint32_t ties = (__ballot_sync(FULL, lead && cost == m) & gmask) >> gb;
            int w = __ffs(ties) - 1;
            const bool tie = move && __popc(ties) > 1;
            if (__any_sync(FULL, tie)) {
                // stable descending sort by off . dir (:357-362), the full warp
                // for each group that needs it
#pragma unroll 1
                for (int t = 0; t < 4; ++t) {
                    if (!__shfl_sync(FULL, tie, 8 * t)) continue;  // warp-uniform
                    PaBlock B;
                    B.cur = a.b.luma + __shfl_sync(FULL, ocur, 8 * t);
                    B.ref = a.b.luma + __shfl_sync(FULL, oref, 8 * t);
                    B.ca = B.ra = nullptr;
                    B.x0 = __shfl_sync(FULL, x0, 8 * t);
                    B.y0 = __shfl_sync(FULL, y0, 8 * t);
                    const int cx = __shfl_sync(FULL, wx + 2 * ci, 8 * t), cy = __shfl_sync(FULL, wy + 2 * cj, 8 * t);
                    double dir_x, dir_y;
                    prs_direction(a.P, B, lane, cx, cy, dir_x, dir_y);
                    if (grp == t) {
                        int wb = -1;
                        double bestkey = 0.0;
                        for (int o = 0; o < 8; ++o) {
                            if (!((ties >> o) & 1u)) continue;
                            const double key = __dadd_rn(__dmul_rn(double(c_off8[o][0]), dir_x), __dmul_rn(double(c_off8[o][1]), dir_y));
                            if (wb < 0 || key > bestkey) {
                                wb = o;
                                bestkey = key;
                            }
                        }
                        w = wb;
                    }
                }
            }
            const int pc = (ci + 8) | ((cj + 8) << 4);
            if (it == 0) pc0 = pc;
            if (it == 1) pc1 = pc;
            if (it == 2) pc2 = pc;
            if (move) {
                ci += off8x(w);
                cj += off8y(w);
                ccost = m;
                ++iters;
            }
            alive = move;
        }
        if (TRACE) c_walk = clock64();
        // publish first (the dependents wait on the record, not on the SSE)
        if (act && gl == 0)
            write_rec_v4(a.recs + g, wx + 2 * ci, wy + 2 * cj, ccost, 4, dpd, iters, boundary ? ME_BOUNDARY : ME_OPAQUE);
        // --- fused predict_frame + psnr SSE at the final vector ---------------
        uint32_t se;
        {
            uint32_t w0, w1;
            prow8(pw + (4 + cj + gl) * kQuadPWW, 4 + ci + wo, w0, w1);
            se = sq4(cw[2 * gl + 1], w1, sq4(cw[2 * gl], w0, 0u));
            se += __shfl_xor_sync(FULL, se, 1);
            se += __shfl_xor_sync(FULL, se, 2);
            se += __shfl_xor_sync(FULL, se, 4);
        }
        if (act && gl == 0) {
            if (a.stats) add_stats_pa(a.stats + pair, se, dpd);
            if (TRACE) {  // as pa_duo_kernel
                unsigned long long* tr = a.trace + size_t(item + grp) * 4;
                const long long c_end = clock64();
                auto c16 = [](long long d) { return (unsigned long long)min(max(d, 0ll), 65535ll); };
                tr[0] = t_claim;
                tr[1] = t_ready;
                tr[2] = gtimer();
                tr[3] = c16(c_patch - c_ready) | (c16(c_brs - c_patch) << 16) | (c16(c_walk - c_brs) << 32) |
                        (c16(c_end - c_walk) << 48);
            }
        }
        __syncwarp();
    }
}

__global__ void brs_single_kernel(PaParams P, PaBlock B, int boundary, const int32_t* cands,
                                  int64_t* out) {
    extern __shared__ uint32_t s_bits[];
    const int lane = threadIdx.x & 31;
    int cdx[4], cdy[4];
    for (int i = 0; i < 4; ++i) {
        cdx[i] = cands[2 * i];
        cdy[i] = cands[2 * i + 1];
    }
    const int k = lane >> 3;
    const int vx = clip_comp(cdx[k], B.w.lo_x, B.w.hi_x);
    const int vy = clip_comp(cdy[k], B.w.lo_y, B.w.hi_y);
    const bool shape = boundary && (k < 3 || P.bt_shape);
    const uint32_t s = score4(P, B, lane, vx, vy, shape);
    uint32_t sc[4];
    int bx = 0, by = 0, win = 0;
    for (int i = 0; i < 4; ++i) {
        sc[i] = __shfl_sync(0xFFFFFFFFu, s, 8 * i);
        const int ix = __shfl_sync(0xFFFFFFFFu, vx, 8 * i), iy = __shfl_sync(0xFFFFFFFFu, vy, 8 * i);
        if (i == 0 || sc[i] < sc[win]) {
            win = i;
            bx = ix;
            by = iy;
        }
    }
    if (lane == 0) {
        out[0] = bx;
        out[1] = by;
        for (int i = 0; i < 4; ++i) {
            out[2 + i] = sc[i];
            out[6 + i] = boundary && (i < 3 || P.bt_shape);
        }
    }
}

// out: [0..1] mv, [2] dpd, [3] iterations, [4] final cost_q4, [5..] descent log
__global__ void prs_single_kernel(PaParams P, PaBlock B, int d0x, int d0y, int64_t* out) {
    extern __shared__ uint32_t s_bits[];
    const int lane = threadIdx.x & 31;
    const int cx = clip_comp(d0x, B.w.lo_x, B.w.hi_x), cy = clip_comp(d0y, B.w.lo_y, B.w.hi_y);
    // replay the descent to produce the log: run prs with max_iter = 0.. is
    // wasteful; instead record accepted centers inline by re-running per step.
    PaParams Q = P;
    uint32_t logv[64];
    int nlog = 0;
    PaResult r{};
    const int cap = P.max_iter < 63 ? P.max_iter : 63;
    for (int m = 0; m <= cap; ++m) {
        Q.max_iter = m;
        if (m == 0) {
            // center cost only
            const uint32_t s = score4(P, B, lane, cx, cy, false);
            logv[nlog++] = __shfl_sync(0xFFFFFFFFu, s, 0);
            continue;
        }
        r = prs_warp(Q, B, lane, cx, cy, kInf, s_bits);
        if (int(r.iters) < m) break;  // stopped before using the m-th iteration
        logv[nlog++] = r.cost_q4;
    }
    r = prs_warp(P, B, lane, cx, cy, kInf, s_bits);
    if (lane == 0) {
        out[0] = r.dx;
        out[1] = r.dy;
        out[2] = r.dpd;
        out[3] = r.iters;
        out[4] = r.cost_q4;
        for (int i = 0; i < nlog && i < 64; ++i) out[5 + i] = logv[i];
    }
}

// prs_update (estimators.cpp:303-309) at one pixel, round-to-nearest intrinsics.
__global__ void prs_update_kernel(const uint8_t* cur, const uint8_t* ref, int W, int H, int x, int y,
                                  int dx, int dy, double eps, double theta, double* out) {
    const int i4 = interp4(ref, W, H, 2 * x - dx, 2 * y - dy);
    const double e = __dsub_rn(double(cur[size_t(y) * W + x]), double(i4) * 0.25);
    const double gx = (double(pxc(cur, W, H, x + 1, y)) - double(pxc(cur, W, H, x - 1, y))) / 2.0;
    const double gy = (double(pxc(cur, W, H, x, y + 1)) - double(pxc(cur, W, H, x, y - 1))) / 2.0;
    const double ux = fabs(gx) < theta ? 0.0 : __ddiv_rn(1.0, gx);
    const double uy = fabs(gy) < theta ? 0.0 : __ddiv_rn(1.0, gy);
    const double ee = __dmul_rn(eps, e);
    out[0] = __dsub_rn(0.5 * dx, __dmul_rn(ee, ux));
    out[1] = __dsub_rn(0.5 * dy, __dmul_rn(ee, uy));
}

// ---------------------------------------------------------------------------
// pa_smem_kernel: one small frame pair (estimate_field on e.g. QCIF) in ONE
// CTA with both frames (and alpha planes) resident in shared memory.  The
// wavefront runs as dataflow on a shared MV array (dependency waits cost a
// shared-memory load instead of a global round trip) and every pixel read is
// a shared-memory load; SSE and records are produced after the wavefront.  Same algorithm and
// results as the batched kernels (classify + BRS + PRS + fused SSE); the
// per-pair API's latency path.
// ---------------------------------------------------------------------------

// 8 bytes at byte offset x of a shared-memory row (4-byte aligned row start)
__device__ __forceinline__ void srow8(const uint8_t* row, int x, uint32_t& r0, uint32_t& r1) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (x >> 2);
    const uint32_t sh = uint32_t(x & 3) * 8;
    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
    r0 = __funnelshift_r(w0, w1, sh);
    r1 = __funnelshift_r(w1, w2, sh);
}

struct PaSmemArgs {
    Batch b;  // n_seq = 1, one pair (frame 0 = ref, frame 1 = cur)
    PaParams P;
    const int32_t* prev0;  // integer-pel T candidates or null
    me_block_rec* recs;
    me_pair_stats* stats;
    int plane_pad;  // bytes per staged plane (plane + 16)
    long long* trace;  // debug (tuning pa_trace_path): per block {wait start, ready, BRS done, walk done, published} SM clocks
};

__global__ void __launch_bounds__(1024, 1) pa_smem_kernel(const PaSmemArgs a) {
    extern __shared__ __align__(16) uint8_t s_frames[];
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    __shared__ unsigned long long s_sse, s_dpd;
    __shared__ unsigned s_cnt[3];  // opaque, boundary, transparent
    const Batch& b = a.b;
    const int W = b.W, H = b.H, S = a.P.S, cols = b.cols, rows = b.rows;
    const int plane = W * H, pp = a.plane_pad;
    const bool has_alpha = b.alpha != nullptr;
    uint8_t* s_ref = s_frames;
    uint8_t* s_cur = s_ref + pp;
    uint8_t* s_ra = s_cur + pp;  // alpha planes only when present
    uint8_t* s_ca = s_ra + pp;
    uint32_t* s_mv = reinterpret_cast<uint32_t*>(s_frames + (has_alpha ? 4 : 2) * size_t(pp));
    uint32_t* s_cost = s_mv + cols * rows;  // final cost_q4 of estimated blocks
    uint32_t* s_meta = s_cost + cols * rows;  // dpd << 8 | iterations
    uint32_t* s_prev = s_meta + cols * rows;  // pair 0's temporal candidates, packed (when given)
    uint8_t* s_type = reinterpret_cast<uint8_t*>(s_prev + (a.prev0 ? cols * rows : 0));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    // stage the planes (16-byte copies) and clear the MV words: the pair's ref
    // is frame 0 and its cur frame d (ref_distance), which need not be adjacent
    {
        const int pw = plane / 16;
        for (int i = tid; i < 2 * pw; i += blockDim.x) {
            const int f = i / pw, o = i - f * pw;
            const uint4* g = reinterpret_cast<const uint4*>(b.luma + size_t(f ? b.d : 0) * plane);
            reinterpret_cast<uint4*>(s_frames + f * size_t(pp))[o] = __ldg(g + o);
        }
        if (has_alpha) {
            for (int i = tid; i < 2 * pw; i += blockDim.x) {
                const int f = i / pw, o = i - f * pw;
                const uint4* ga = reinterpret_cast<const uint4*>(b.alpha + size_t(f ? b.d : 0) * plane);
                reinterpret_cast<uint4*>(s_ra + f * size_t(pp))[o] = __ldg(ga + o);
            }
        }
        for (int i = tid; i < cols * rows; i += blockDim.x) {
            s_mv[i] = 0u;
            if (a.prev0) s_prev[i] = pack_mv(a.prev0[2 * i], a.prev0[2 * i + 1]);
        }
        if (tid == 0) {
            s_sse = s_dpd = 0ull;
            s_cnt[0] = s_cnt[1] = s_cnt[2] = 0u;
        }
    }
    __syncthreads();
    unsigned long long my_sse = 0, my_dpd = 0;
    unsigned n_opaque = 0, n_boundary = 0, n_transparent = 0;
    // phase 1: classify every block (cur alpha, frame.cpp:81-104); transparent
    // blocks are final here (MV 0, SSE at the zero vector)
    for (int g = wid; g < cols * rows; g += nw) {
        const int h = g % cols, v = g / cols, x0 = h * 8, y0 = v * 8;
        int ty = ME_OPAQUE;
        if (has_alpha) {
            uint32_t r0 = 0, r1 = 0;
            if (lane < 8) {
                const uint2 w = *reinterpret_cast<const uint2*>(s_ca + (y0 + lane) * W + x0);
                r0 = w.x;
                r1 = w.y;
            }
            const bool any = __any_sync(FULL, (r0 | r1) != 0u);
            const bool allnz = __all_sync(FULL, lane >= 8 || (__vcmpeq4(r0, 0u) | __vcmpeq4(r1, 0u)) == 0u);
            ty = !any ? ME_TRANSPARENT : (allnz ? ME_OPAQUE : ME_BOUNDARY);
        }
        if (lane == 0) {
            s_type[g] = uint8_t(ty);
            if (ty != ME_TRANSPARENT) s_mv[g] = kSentinel;  // published by phase 2
        }
        if (ty == ME_TRANSPARENT) {
            uint32_t se = 0;
            if (lane < 8) {
                const uint2 c = *reinterpret_cast<const uint2*>(s_cur + (y0 + lane) * W + x0);
                const uint2 r = *reinterpret_cast<const uint2*>(s_ref + (y0 + lane) * W + x0);
                se = sq4(c.y, r.y, sq4(c.x, r.x, 0u));
            }
            se = __reduce_add_sync(FULL, se);
            if (lane == 0) {
                write_rec(a.recs + g, 0, 0, 0u, 0u, 0u, 0u, ME_TRANSPARENT, false);
                my_sse += se;
                ++n_transparent;
            }
        }
    }
    __syncthreads();
    // phase 2: the wavefront as shared-memory dataflow.  Warps take the blocks
    // in wavefront order (t = h + 2v, then v) round robin and wait on their
    // dependencies' MV words (sentinel until published); every dependency
    // lies earlier in that order, so the least unfinished block can always
    // proceed.  A block starts as soon as ITS dependencies are done, not when
    // the slowest block of the previous step is.
    const int c = lane >> 3, sub = lane & 7;  // BRS: candidate c, row sub
    const int k = lane >> 2, q = lane & 3;    // PRS: neighbour k, rows q and q + 4
    const int kx = off8x(k), ky = off8y(k);
    volatile uint32_t* vmv = s_mv;
    for (int idx = wid, t = 0, first = 0; idx < cols * rows; idx += nw) {
        int vmin = 0, vmax = 0;
        for (;; ++t) {  // the step holding block number idx (monotonic per warp)
            vmin = max(0, (t - (cols - 1) + 1) / 2);
            vmax = min(rows - 1, t / 2);
            if (idx < first + vmax - vmin + 1) break;
            first += vmax - vmin + 1;
        }
        {
            const int v = vmin + (idx - first), h = t - 2 * v, g = v * cols + h;
            const int ty = s_type[g];
            if (ty == ME_TRANSPARENT) continue;  // warp-uniform
            const bool boundary = ty == ME_BOUNDARY;
            const int x0 = h * 8, y0 = v * 8;
            const int lo_x = max(-2 * S, -2 * x0), hi_x = min(2 * S, 2 * (W - x0 - 8));
            const int lo_y = max(-2 * S, -2 * y0), hi_y = min(2 * S, 2 * (H - y0 - 8));
            // gather_candidates (estimators.cpp:238-255): A, B, C, T
            long long tr0 = 0;
            if (a.trace) tr0 = clock64();
            int dep = -1;
            if (c == 0 && h > 0) dep = g - 1;
            if (c == 1 && v > 0) dep = g - cols;
            if (c == 2 && v > 0 && h + 1 < cols) dep = g - cols + 1;
            // (the T candidate and this block's current rows do not depend on the wait)
            const uint32_t tw = c == 3 && a.prev0 ? s_prev[g] : 0u;
            const uint2 cr = *reinterpret_cast<const uint2*>(s_cur + (y0 + sub) * W + x0);
            const uint2 ca_ = *reinterpret_cast<const uint2*>(s_cur + (y0 + q) * W + x0);
            const uint2 cb_ = *reinterpret_cast<const uint2*>(s_cur + (y0 + q + 4) * W + x0);
            uint32_t mw = dep >= 0 ? vmv[dep] : 0u;
            while (__any_sync(FULL, mw == kSentinel)) mw = dep >= 0 ? vmv[dep] : 0u;
            if (c == 3) mw = tw;
            long long tr1 = 0, tr2 = 0, tr3 = 0;
            if (a.trace) tr1 = clock64();
            const int myx = clip_comp(mv_dx(mw), lo_x, hi_x), myy = clip_comp(mv_dy(mw), lo_y, hi_y);
            // brs_select (estimators.cpp:257-301): row `sub` of candidate c
            uint32_t s;
            const int ry = y0 + sub + (myy >> 1), rx = x0 + (myx >> 1);
            if (boundary && (c < 3 || a.P.bt_shape)) {
                const uint2 ca = *reinterpret_cast<const uint2*>(s_ca + (y0 + sub) * W + x0);
                uint32_t r0, r1;
                srow8(s_ra + ry * W, rx, r0, r1);
                s = ((__popc(__vcmpne4(ca.x, r0)) + __popc(__vcmpne4(ca.y, r1))) >> 3) * (255u * 4u);
            } else {
                uint32_t r0, r1;
                srow8(s_ref + ry * W, rx, r0, r1);
                s = vad4(cr.y, r1, vad4(cr.x, r0, 0u)) * 4u;
            }
            s += __shfl_xor_sync(FULL, s, 1);
            s += __shfl_xor_sync(FULL, s, 2);
            s += __shfl_xor_sync(FULL, s, 4);
            // strict <: A, B, C, T tie order (:295) = the minimum of (score, candidate)
            // (scores < 2^17), one warp reduction
            const uint32_t bk = __reduce_min_sync(FULL, (s << 2) | uint32_t(c));
            const uint32_t best = bk >> 2;
            const int win = int(bk & 3u);
            const uint32_t wxy = __shfl_sync(FULL, pack_mv(myx, myy), 8 * win);
            const int wx = mv_dx(wxy), wy = mv_dy(wxy);
            uint32_t ccost = best;
            if (boundary && (win < 3 || a.P.bt_shape)) {  // the centre's texture cost
                uint32_t tsum = 0;
                if (lane < 8) {
                    const uint2 cr = *reinterpret_cast<const uint2*>(s_cur + (y0 + lane) * W + x0);
                    uint32_t r0, r1;
                    srow8(s_ref + (y0 + lane + (wy >> 1)) * W, x0 + (wx >> 1), r0, r1);
                    tsum = vad4(cr.y, r1, vad4(cr.x, r0, 0u));
                }
                ccost = 4u * __reduce_add_sync(FULL, tsum);
            }
            if (a.trace) tr2 = clock64();
            // prs_refine (estimators.cpp:311-382); unique evaluations: a neighbour
            // is new iff it is at Chebyshev distance >= 2 from every earlier centre
            int ci = 0, cj = 0, pc0 = 0, pc1 = 0, pc2 = 0;
            uint32_t dpd = 1, iters = 0;
            for (int it = 0; it < a.P.max_iter; ++it) {
                if (ccost == 0) break;  // already a global minimum (:341)
                const int px = ci + kx, py = cj + ky;
                const bool adm = wx + 2 * px >= lo_x && wx + 2 * px <= hi_x && wy + 2 * py >= lo_y && wy + 2 * py <= hi_y;
                uint32_t part = 0;
                if (adm) {
                    const int bx = x0 + (wx >> 1) + px, by = y0 + (wy >> 1) + py;
                    uint32_t r0, r1, r2, r3;
                    srow8(s_ref + (by + q) * W, bx, r0, r1);
                    srow8(s_ref + (by + q + 4) * W, bx, r2, r3);
                    part = vad4(cb_.y, r3, vad4(cb_.x, r2, vad4(ca_.y, r1, vad4(ca_.x, r0, 0u))));
                }
                part += __shfl_xor_sync(FULL, part, 1);
                part += __shfl_xor_sync(FULL, part, 2);
                const uint32_t cost = 4u * part;
                const bool lead = adm && q == 0;
                auto far = [&](int pc) { return max(abs(px + 8 - (pc & 15)), abs(py + 8 - (pc >> 4))) >= 2; };
                bool fresh = lead;
                if (it >= 1) fresh = fresh && far(pc0);
                if (it >= 2) fresh = fresh && far(pc1);
                if (it >= 3) fresh = fresh && far(pc2);
                dpd += __popc(__ballot_sync(FULL, fresh));
                const uint32_t m = __reduce_min_sync(FULL, lead ? cost : kInf);
                if (m >= ccost) break;  // centre kept (:376)
                const uint32_t ties = __ballot_sync(FULL, lead && cost == m);
                int w;
                if (__popc(ties) == 1) {
                    w = (__ffs(ties) - 1) >> 2;
                } else {
                    // stable descending sort by off . dir (:357-362)
                    PaBlock B;
                    B.cur = b.luma + plane;
                    B.ref = b.luma;
                    B.ca = B.ra = nullptr;
                    B.x0 = x0;
                    B.y0 = y0;
                    double dir_x, dir_y;
                    prs_direction(a.P, B, lane, wx + 2 * ci, wy + 2 * cj, dir_x, dir_y);
                    w = -1;
                    double bestkey = 0.0;
                    for (int o = 0; o < 8; ++o) {
                        if (!((ties >> (4 * o)) & 1u)) continue;
                        const double key = __dadd_rn(__dmul_rn(double(c_off8[o][0]), dir_x), __dmul_rn(double(c_off8[o][1]), dir_y));
                        if (w < 0 || key > bestkey) {
                            w = o;
                            bestkey = key;
                        }
                    }
                }
                const int pc = (ci + 8) | ((cj + 8) << 4);
                if (it == 0) pc0 = pc;
                if (it == 1) pc1 = pc;
                if (it == 2) pc2 = pc;
                ci += off8x(w);
                cj += off8y(w);
                ccost = m;
                ++iters;
            }
            // only the vector is on the wavefront's critical path: the SSE and
            // the record are produced after the last step (phase 3)
            if (a.trace) tr3 = clock64();
            if (lane == 0) {
                // publish first: the dependents read only the MV word (cost and
                // counters are read by phase 3, after the barrier)
                vmv[g] = pack_mv(wx + 2 * ci, wy + 2 * cj);
                s_cost[g] = ccost;
                s_meta[g] = (dpd << 8) | iters;
                if (a.trace) {
                    long long* tr = a.trace + size_t(g) * 5;
                    tr[0] = tr0;
                    tr[1] = tr1;
                    tr[2] = tr2;
                    tr[3] = tr3;
                    tr[4] = clock64();
                }
            }
        }
    }
    __syncthreads();
    // phase 3: fused predict_frame + psnr SSE at the final vectors, records
    for (int g = wid; g < cols * rows; g += nw) {
        const int ty = s_type[g];
        if (ty == ME_TRANSPARENT) continue;  // warp-uniform
        const int h = g % cols, v = g / cols, x0 = h * 8, y0 = v * 8;
        const uint32_t mw = s_mv[g];
        const int fx = mv_dx(mw), fy = mv_dy(mw);
        uint32_t se = 0;
        if (lane < 8) {
            const uint2 cr = *reinterpret_cast<const uint2*>(s_cur + (y0 + lane) * W + x0);
            uint32_t r0, r1;
            srow8(s_ref + (y0 + lane + (fy >> 1)) * W, x0 + (fx >> 1), r0, r1);
            se = sq4(cr.y, r1, sq4(cr.x, r0, 0u));
        }
        se = __reduce_add_sync(FULL, se);
        if (lane == 0) {
            const uint32_t meta = s_meta[g];
            write_rec(a.recs + g, fx, fy, s_cost[g], 4, meta >> 8, meta & 0xFF, uint32_t(ty), false);
            my_sse += se;
            my_dpd += meta >> 8;
            if (ty == ME_BOUNDARY)
                ++n_boundary;
            else
                ++n_opaque;
        }
    }
    if (lane == 0) {
        atomicAdd(&s_sse, my_sse);
        atomicAdd(&s_dpd, my_dpd);
        atomicAdd(&s_cnt[0], n_opaque);
        atomicAdd(&s_cnt[1], n_boundary);
        atomicAdd(&s_cnt[2], n_transparent);
    }
    __syncthreads();
    if (tid == 0 && a.stats) {
        me_pair_stats st;
        st.block_comparisons = 4 * int64_t(s_cnt[0] + s_cnt[1]);  // brs_select: 4 per block (:290)
        st.dpd_refinement_steps = int64_t(s_dpd);
        st.blocks_opaque = s_cnt[0];
        st.blocks_boundary = s_cnt[1];
        st.blocks_transparent = s_cnt[2];
        st.sse = int64_t(s_sse);
        *a.stats = st;
    }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------


// Steps with at least this many estimated blocks run two blocks per warp.
int pa_wide_threshold(int num_sms, const Tuning& t) {
    return t.pa_wide_blocks > 0 ? t.pa_wide_blocks : num_sms * 40;  // measured: 3000-9000 within 1 %, duo-only 3 % slower
}

int pa_kernel_mode(const Batch& b, const me_config& cfg, const int32_t* prev0, bool prev0_integer,
                   int num_sms, const Tuning& t) {
    const int step = cfg.halfpel ? 1 : cfg.step;
    const bool fast = b.bs == 8 && step == 2 && cfg.max_iterations <= 4 && (!prev0 || prev0_integer) &&
                      size_t(b.n_seq) * b.F * b.W * b.H < (size_t(1) << 32);
    const int sched = t.pa_schedule;
    if (!fast || sched == ME_PA_SCHED_GENERIC) return 0;
    if (sched == ME_PA_SCHED_FAST) return 1;
    if (prev0) return 1;  // the two-blocks-per-warp kernel takes no external prev field
    if (sched == ME_PA_SCHED_DUO) return 2;
    if (sched == ME_PA_SCHED_DUO_HYBRID) return 3;
    if (sched == ME_PA_SCHED_QUAD_HYBRID) return 4;
    const int64_t per_step = b.nblocks() / std::max(1, b.steps());
    // measured on CIF batches (tools/pa_schedule_probe.py): the quad hybrid
    // from ~60 sequences on (120 blocks per step per SM), fast below
    return per_step >= int64_t(num_sms) * 120 ? 4 : 1;
}

bool pa_takes_bits(const Batch& b, const me_config& cfg, int num_sms, const Tuning& t) {
    const int mode = pa_kernel_mode(b, cfg, nullptr, false, num_sms, t);
    return mode == 1 || mode == 4;
}

// One small pair in one CTA (pa_smem_kernel) when it fits in shared memory;
// returns cudaErrorNotSupported when not eligible (the caller runs the
// batched pipeline instead).
cudaError_t launch_pa_smem(const Batch& b, const me_config& cfg, const int32_t* prev0, bool prev0_integer,
                           me_block_rec* recs, me_pair_stats* stats, cudaStream_t st, const Tuning& t) {
    const int step = cfg.halfpel ? 1 : cfg.step;
    if (!(b.n_seq == 1 && b.pairs == 1 && b.bs == 8 && step == 2 && cfg.max_iterations <= 4 &&
          (!prev0 || prev0_integer) && (size_t(b.W) * b.H) % 16 == 0) ||
        !t.pa_smem_pair || b.alpha_bits)
        return cudaErrorNotSupported;
    const int plane_pad = b.W * b.H + 16;
    const size_t smem = size_t(b.alpha ? 4 : 2) * plane_pad + size_t(b.cols) * b.rows * (prev0 ? 17 : 13) + 16;
    // (a CIF pair would fit in 227 KB, but one CTA's 32 warps hold only ~1.5 of
    // its ~22-block wavefront steps: 174 us vs 158 through the batched pipeline)
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    PaSmemArgs a;
    a.b = b;
    a.P = make_pa_params(b, cfg);
    a.prev0 = prev0;
    a.recs = recs;
    a.stats = stats;
    a.plane_pad = plane_pad;
    a.trace = nullptr;
    if (t.pa_trace) {
        cudaMalloc(&a.trace, size_t(b.cols) * b.rows * 5 * 8);
        cudaMemsetAsync(a.trace, 0, size_t(b.cols) * b.rows * 5 * 8, st);
    }
    static thread_local size_t attr_smem = 0;  // the attribute call costs microseconds: set once per size
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(pa_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e) return e;
        attr_smem = smem;
    }
    pa_smem_kernel<<<1, 1024, smem, st>>>(a);
    if (a.trace) {
        std::vector<long long> h(size_t(b.cols) * b.rows * 5);
        cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (FILE* f = fopen(t.pa_trace, "wb")) {
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
        cudaFree(a.trace);
    }
    return cudaGetLastError();
}

cudaError_t launch_pa(const Batch& b, const me_config& cfg, const int32_t* prev0, const uint2* list,
                      const int* nlist, const int* ranges, int pa_mode, me_block_rec* recs,
                      me_pair_stats* stats, int num_sms, cudaStream_t st, int* claims, const Tuning& t) {
    cudaError_t e;
    PaArgs pa_args;
    pa_args.b = b;
    pa_args.P = make_pa_params(b, cfg);
    pa_args.list = list;
    pa_args.nlist = nlist;
    pa_args.range = nullptr;
    pa_args.recs = recs;
    pa_args.prev0 = prev0;
    pa_args.stats = stats;
    pa_args.fast = (pa_args.P.step == 2 && cfg.max_iterations <= 4) ? 1 : 0;
    // pa_fast_kernel's staged search window: 2S + 16 rows of 16-byte chunks
    // from the 16-aligned column at or left of x0 - S - 4 (at most
    // (2S + 15) / 16 + 2 chunks), row stride padded by 4 words against bank
    // conflicts between the lanes' rows
    int fast_words = kFastWarpWords;
    pa_args.win_words = 0;
    pa_args.awin_words = 0;
    auto set_window = [&](int ctas_per_sm) {
        if (!t.pa_fast_window || cfg.search_range > 32) return;
        const int S = cfg.search_range, wsw = 4 * ((2 * S + 15) / 16 + 2) + 4;
        pa_args.win_words = wsw;
        int words = (2 * S + 16) * wsw;
        // the boundary blocks' alpha window when the shared memory allows (<= 2 CTAs per SM)
        if (b.alpha && !b.alpha_bits && ctas_per_sm <= 2) {
            pa_args.awin_words = 4 * ((2 * S + 8 + 15) / 16 + 1) + 4;
            words += (2 * S + 8) * pa_args.awin_words;
        }
        fast_words = std::max(4 * kFastPatch, words) + 20;
    };
    pa_args.poll_ns = t.pa_poll_ns;
    pa_args.pdl = 0;
    pa_args.trace = nullptr;
    pa_args.claim = nullptr;
    const char* trace_path = t.pa_trace;
    int n_host = 0;
    if (trace_path) {
        cudaStreamSynchronize(st);
        cudaMemcpy(&n_host, nlist, 4, cudaMemcpyDeviceToHost);
        cudaMalloc(&pa_args.trace, size_t(n_host) * 32);
        cudaMemset(pa_args.trace, 0, size_t(n_host) * 32);
    }
    using PaKernel = void (*)(const PaArgs);
    // pa_no_pdl launches the hybrid's grids in plain stream order
    const bool pdl = pa_mode == 4 && !trace_path && t.pa_pdl;
    // persistent grids: every warp of a launch must be co-resident (dependency spinning)
    const bool dyn = t.pa_claim;
    int n_launch = 0;
    auto launch = [&](PaKernel kern, int threads, int warp_words, const int* range, bool chained = false,
                      bool after_sort = false) -> cudaError_t {
        PaArgs la = pa_args;
        la.range = range;
        la.claim = dyn && claims ? claims + n_launch : nullptr;  // one zeroed counter per launch
        ++n_launch;
        la.pdl = pdl ? (after_sort ? 2 : 1) : 0;
        la.warp_words = std::max(la.P.bm_words, warp_words);
        const size_t smem = size_t(threads / 32) * la.warp_words * 4;
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e2) return e2;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (pdl && chained) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(num_sms * (occ > 0 ? occ : 1));
            lc.blockDim = dim3(threads);
            lc.dynamicSmemBytes = smem;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            return cudaLaunchKernelEx(&lc, kern, la);
        }
        kern<<<num_sms * (occ > 0 ? occ : 1), threads, smem, st>>>(la);
        return cudaGetLastError();
    };
    PaKernel fast = pa_fast_kernel<4>;
    {
        // a single sequence is latency-bound: one CTA per SM with 128
        // registers per thread runs each block sooner (measured 3-6 % on
        // configs 2, 3, 5); small batches (< 80 blocks per step per SM, up to
        // ~36 CIF sequences) need more blocks in flight: 2 CTAs below 60
        // blocks per step per SM (measured 4-25 % better than 1 or 4 at 8-16
        // CIF sequences, 5-7 % better than 3 at 16-24), 3 from 60 to 160
        // (1-1.5 % better than 2 or 4 at 32-64); wider ones 4 (the hybrid's
        // head and tail)
        const int64_t per_step = b.nblocks() / std::max(1, b.steps());
        // (a single sequence searched with per-candidate patches, S > 32: 2 CTAs,
        // config 5 2.37 -> 2.21 ms; with the staged window, S <= 32: 1)
        const int mb = t.pa_fast_ctas > 0 ? t.pa_fast_ctas
                       : pa_mode != 1      ? 4
                       : b.n_seq == 1      ? (cfg.search_range > 32 ? 2 : 1)
                       : per_step < int64_t(num_sms) * 60 ? 2
                       : per_step < int64_t(num_sms) * 160 ? 3 : 4;
        fast = mb == 1 ? pa_fast_kernel<1> : mb == 2 ? pa_fast_kernel<2> : mb == 3 ? pa_fast_kernel<3> : mb == 5 ? pa_fast_kernel<5> : mb == 6 ? pa_fast_kernel<6> : pa_fast_kernel<4>;
        set_window(mb);
        if (trace_path) fast = mb == 1 ? pa_fast_kernel<1, true> : mb == 2 ? pa_fast_kernel<2, true> : pa_fast_kernel<4, true>;
    }
    const int duo_threads = t.pa_duo_threads == 128 ? 128 : 256;
    PaKernel duo = pa_duo_kernel<256, 4>;
    {
        const int mb = t.pa_duo_ctas > 0 ? t.pa_duo_ctas : duo_threads == 128 ? 7 : 4;
        if (trace_path)
            duo = pa_duo_kernel<256, 4, true>;
        else if (duo_threads == 128)
            duo = mb == 8 ? pa_duo_kernel<128, 8> : mb == 6 ? pa_duo_kernel<128, 6> : pa_duo_kernel<128, 7>;
        else if (mb == 3)
            duo = pa_duo_kernel<256, 3>;
    }
    if (pa_mode == 0) {
        e = launch(b.bs == 8 ? pa_kernel<8> : pa_kernel<16>, 256,
                   b.bs == 8 ? WPatch<8>::WARP_WORDS : WPatch<16>::WARP_WORDS, nullptr);
    } else if (pa_mode == 1) {
        e = launch(fast, 256, fast_words, nullptr);
    } else if (pa_mode == 2) {
        e = launch(duo, trace_path ? 256 : duo_threads, kDuoWarpWords, nullptr);
    } else if (pa_mode == 4) {  // narrow steps -> fast, the wide middle -> quad, narrow tail -> fast
        // 3 CTAs (24 warps, 96 blocks in flight) per SM at 80 registers:
        // measured 8 % faster than 4 at 64 (spills) and 1 % than 2 at 112
        const int mb = t.pa_quad_ctas;
        PaKernel quad = mb == 4 ? pa_quad_kernel<4> : mb == 2 ? pa_quad_kernel<2> : pa_quad_kernel<3>;
        if (trace_path) quad = pa_quad_kernel<3, true>;
        if (!(e = launch(fast, 256, fast_words, ranges, t.sort_pdl, t.sort_pdl)) &&
            !(e = launch(quad, 256, kQuadWarpWords, ranges + 2, true)))
            e = launch(fast, 256, fast_words, ranges + 4, true);
    } else {  // narrow steps -> fast, the wide middle -> duo, narrow tail -> fast
        if (!(e = launch(fast, 256, fast_words, ranges)) &&
            !(e = launch(duo, trace_path ? 256 : duo_threads, kDuoWarpWords, ranges + 2)))
            e = launch(fast, 256, fast_words, ranges + 4);
    }
    if (e) return e;
    if (trace_path) {
        std::vector<unsigned long long> h(size_t(n_host) * 4);
        std::vector<uint2> lst(n_host);
        cudaMemcpyAsync(h.data(), pa_args.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(lst.data(), list, lst.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (FILE* f = fopen(trace_path, "wb")) {
            fwrite(h.data(), 8, h.size(), f);
            fwrite(lst.data(), 8, lst.size(), f);
            fclose(f);
        }
        cudaFree(pa_args.trace);
    }
    return cudaGetLastError();
}

static PaBlock single_block(const uint8_t* cur, const uint8_t* ref, const uint8_t* ca,
                            const uint8_t* ra, int W, int H, int x0, int y0, int size, int range) {
    PaBlock B;
    B.cur = cur;
    B.ref = ref;
    B.ca = ca;
    B.ra = ra;
    B.x0 = x0;
    B.y0 = y0;
    B.w.lo_x = std::max(-2 * range, -2 * x0);
    B.w.hi_x = std::min(2 * range, 2 * (W - x0 - size));
    B.w.lo_y = std::max(-2 * range, -2 * y0);
    B.w.hi_y = std::min(2 * range, 2 * (H - y0 - size));
    return B;
}

cudaError_t brs_single(const uint8_t* cur, const uint8_t* ref, const uint8_t* ca,
                       const uint8_t* ra, int W, int H, int x0, int y0, int size, int btype,
                       const int32_t* cands_dev, int range, int boundary_temporal, int64_t* out,
                       cudaStream_t st) {
    PaParams P{};
    P.W = W;
    P.H = H;
    P.bs = size;
    P.S = range;
    P.bt_shape = boundary_temporal == ME_BT_SHAPE;
    PaBlock B = single_block(cur, ref, ca, ra, W, H, x0, y0, size, range);
    brs_single_kernel<<<1, 32, 0, st>>>(P, B, btype == ME_BOUNDARY, cands_dev, out);
    return cudaGetLastError();
}

cudaError_t prs_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                       int size, int d0x, int d0y, int range, double eps, double theta,
                       int max_iter, int step, int64_t* out, cudaStream_t st) {
    Batch b{};
    b.W = W;
    b.H = H;
    b.bs = size;
    me_config c{};
    c.search_range = range;
    c.max_iterations = max_iter;
    c.step = step;
    c.halfpel = 0;
    c.epsilon = eps;
    c.theta = theta;
    PaParams P = make_pa_params(b, c);
    PaBlock B = single_block(cur, ref, nullptr, nullptr, W, H, x0, y0, size, range);
    const size_t smem = size_t(P.bm_words) * 4;
    cudaError_t e = cudaFuncSetAttribute(prs_single_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e) return e;
    prs_single_kernel<<<1, 32, smem, st>>>(P, B, d0x, d0y, out);
    return cudaGetLastError();
}

cudaError_t prs_update_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x, int y,
                              int dx, int dy, double eps, double theta, double* out, cudaStream_t st) {
    prs_update_kernel<<<1, 1, 0, st>>>(cur, ref, W, H, x, y, dx, dy, eps, theta, out);
    return cudaGetLastError();
}

}  // namespace mek
