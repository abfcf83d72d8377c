// batch.cu — the device pipeline of a batch of sequences (run_batch:
// classify -> wavefront sort -> search -> prediction) and the dispatch of the
// single-block searches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "device.cuh"

namespace mek {

namespace {

struct Scratch {
    uint8_t* types;
    uint2* list;
    int* hist;
    int* offs;
    int* cursor;
    int* counter;
    int* hist2;  // aligned PA keys: [n_seq][nbins] per-(sequence, step) counts, then tmin [n_seq]
    int* tmin;
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

Scratch carve(const Batch& b, int nbins, void* base) {
    Scratch s;
    uint8_t* p = static_cast<uint8_t*>(base);
    const size_t nb = size_t(b.nblocks());
    s.types = p;
    p += align_up(nb);
    s.list = reinterpret_cast<uint2*>(p);
    p += align_up((nb + 3 * size_t(nbins)) * 8);  // + padding of every step to a multiple of 4
    s.hist = reinterpret_cast<int*>(p);
    p += align_up(size_t(nbins) * 4);
    s.offs = reinterpret_cast<int*>(p);
    p += align_up(size_t(nbins + 1) * 4);
    s.cursor = reinterpret_cast<int*>(p);
    p += align_up(size_t(nbins) * 4 * kCursorStride);
    s.counter = reinterpret_cast<int*>(p);
    p += 256;
    s.hist2 = reinterpret_cast<int*>(p);
    p += align_up(size_t(b.n_seq) * nbins * 4);
    s.tmin = reinterpret_cast<int*>(p);
    return s;
}

}  // namespace

// Ordering of the PA work list: key = A * t + S * seq, t = h + 2v + p.  Any
// A >= 1 keeps every dependency (key - A or key - 2A) strictly earlier; S > 0
// staggers the sequences' wavefronts.  Overridable for experiments through
// ME_PA_KEY_A / ME_PA_KEY_S.
struct KeyParams {
    int a, s;
};

// Aligned keys pay off where the batch's lockstep step count sets the time
// (latency-bound wavefronts: cfg4 at 32 / 64 / 128 sequences, -5 / -9 / -4 %);
// at 256 the search is throughput-bound (-1 %) and the extra per-(sequence,
// step) counting in classify and the scan (+0.02 ms) outweighs it.  A single
// sequence has nothing to align.
bool pa_key_aligned(const Batch& b, const Tuning& t) {
    if (!t.key_align || b.n_seq < 2) return false;
    if (t.key_align_max_blocks_per_step >= 0 &&
        b.nblocks() > int64_t(t.key_align_max_blocks_per_step) * b.steps())
        return false;
    return int64_t(b.n_seq) * b.steps() <= (int64_t(1) << 24) && b.steps() + b.n_seq <= 48 * 1024;
}

KeyParams pa_key(const Batch& b, const Tuning& t) {
    if (pa_key_aligned(b, t)) return KeyParams{1, 0};  // key = t - tmin[seq] in [0, steps)
    KeyParams k{std::max(1, t.key_a), std::max(0, t.key_s)};
    if (int64_t(k.a) * (b.steps() - 1) + int64_t(k.s) * (b.n_seq - 1) + 1 > 12288) k = KeyParams{1, 0};
    return k;
}

int pa_bins(const Batch& b, const Tuning& t) {
    const KeyParams k = pa_key(b, t);
    return k.a * (b.steps() - 1) + k.s * (b.n_seq - 1) + 1;
}

Tuning resolve_tuning(const me_tuning* u) {
    Tuning t;
    if (!u) return t;
    if (u->pa_schedule) t.pa_schedule = u->pa_schedule;
    t.pa_wide_blocks = u->pa_wide_blocks;
    t.pa_fast_ctas = u->pa_fast_ctas;
    if (u->pa_quad_ctas) t.pa_quad_ctas = u->pa_quad_ctas;
    if (u->pa_duo_threads) t.pa_duo_threads = u->pa_duo_threads;
    t.pa_duo_ctas = u->pa_duo_ctas;
    if (u->pa_poll_ns) t.pa_poll_ns = u->pa_poll_ns;
    t.pa_claim = !u->pa_static_claim;
    t.pa_pdl = !u->pa_no_pdl;
    t.pa_smem_pair = !u->pa_no_smem_pair;
    t.pa_fast_window = !u->pa_fast_patches;
    if (u->pa_key_a) t.key_a = u->pa_key_a;
    t.key_s = u->pa_key_s;
    t.key_align = u->pa_key_plain != 1;
    if (u->pa_key_plain == -1) t.key_align_max_blocks_per_step = -1;  // -1: aligned at any batch width
    t.sort_pdl = !u->sort_no_pdl;
    t.fill_rows = u->fill_rows;
    if (u->fill_rows_per_cta) t.fill_rows_per_cta = u->fill_rows_per_cta;
    if (u->h2d_chunks) t.h2d_chunks = u->h2d_chunks;
    if (u->mask_pack) t.mask_pack = u->mask_pack;
    if (u->ring_ctas) t.ring_ctas = u->ring_ctas;
    t.host_threads = u->host_threads;
    t.pa_trace = u->pa_trace_path;
    return t;
}

size_t scratch_bytes(const Batch& b, int algo, const Tuning& t) {
    const int nbins = algo == ME_ALGO_PA ? pa_bins(b, t) : 1;
    const size_t nb = size_t(b.nblocks());
    return align_up(nb) + align_up((nb + 3 * size_t(nbins)) * 8) + align_up(size_t(nbins) * 4) +
           align_up(size_t(nbins + 1) * 4) + align_up(size_t(nbins) * 4 * kCursorStride) + 256 +
           align_up(size_t(b.n_seq) * nbins * 4) + align_up(size_t(b.n_seq) * 4);
}

// 0: pa_kernel (generic), 1: pa_fast_kernel, 2: pa_duo_kernel, 3: fast / duo /
// fast over the list's narrow / wide / narrow step ranges, 4: the same with
// pa_quad_kernel for the wide range (the default for wide batches).
// Wide wavefront steps (many independent blocks per step) are throughput-
// bound: four blocks per warp (quad) keep more blocks in flight for fewer
// instructions per block.  Narrow ones (single sequences, small batches) are
// latency-bound: a whole warp per block (fast) finishes each block sooner.
// Measured crossover (CIF, 148 SMs): between 64 and 128 sequences, i.e.
// ~25 000 blocks per step.

cudaError_t run_batch(const Batch& b, const me_config& cfg, const int32_t* prev0,
                      me_block_rec* recs, me_pair_stats* stats, uint8_t* pred, void* scratch,
                      size_t scratch_size, int num_sms, cudaStream_t st, const Tuning& tune,
                      cudaEvent_t* events, bool prev0_integer, int* launches) {
    const int algo = cfg.algo;
    const bool pa = algo == ME_ALGO_PA;
    if (pa) {  // one small pair: the whole pipeline in one shared-memory-resident CTA
        if (events)
            for (int i = 0; i < 3; ++i) cudaEventRecord(events[i], st);
        const cudaError_t e0 = launch_pa_smem(b, cfg, prev0, prev0_integer, recs, stats, st, tune);
        if (e0 == cudaSuccess) {
            if (launches) *launches = 1 + (pred ? 1 : 0);
            if (events) cudaEventRecord(events[3], st);
            if (pred) {
                const cudaError_t e1 = launch_mc_pred(b, recs, pred, st);
                if (e1) return e1;
            }
            if (events) cudaEventRecord(events[4], st);
            return cudaGetLastError();
        }
        if (e0 != cudaErrorNotSupported) return e0;
    }
    NvtxRange nv_batch(pa ? "me_b200/batch/pa" : "me_b200/batch/baseline");
    const int nbins = pa ? pa_bins(b, tune) : 1;
    if (scratch_size < scratch_bytes(b, algo, tune)) return cudaErrorInvalidValue;
    Scratch s = carve(b, nbins, scratch);
    cudaError_t e;
    // aligned keys (PA): every sequence's wavefront starts at key 0 — the list
    // interleaves the sequences by their own progress instead of the batch's
    // absolute step, so the batch has max(span) instead of max(end) - min(start)
    // lockstep steps (all dependencies stay within a sequence, hence earlier)
    const bool align = pa && pa_key_aligned(b, tune);  // (the scan holds the key histogram + tmin in shared memory)
    if ((e = cudaMemsetAsync(align ? s.hist2 : s.hist, 0, size_t(align ? b.n_seq : 1) * nbins * 4, st))) return e;
    if (align && (e = cudaMemsetAsync(s.tmin, 0x7F, size_t(b.n_seq) * 4, st))) return e;
    if ((e = cudaMemsetAsync(s.counter, 0, 256, st))) return e;  // ES ticket, PA claim counters, direct list count
    if (stats && (e = cudaMemsetAsync(stats, 0, sizeof(me_pair_stats) * size_t(b.n_seq) * b.pairs, st)))
        return e;

    if (events) cudaEventRecord(events[0], st);
    ClassArgs ca;
    ca.b = b;
    ca.pa = pa ? 1 : 0;
    ca.recs = recs;
    ca.types = s.types;
    ca.hist = s.hist;
    ca.nbins = nbins;
    ca.stats = stats;
    {
        const KeyParams k = pa_key(b, tune);
        ca.key_a = k.a;
        ca.key_s = k.s;
        ca.hist2 = align ? s.hist2 : nullptr;
        ca.tmin = align ? s.tmin : nullptr;
        ca.tmin_g = align ? s.tmin : nullptr;
    }
    // single-bin searches take their list straight from classify
    ca.list_direct = pa ? nullptr : s.list;
    ca.nlist_direct = pa ? nullptr : s.counter + 48;
    ca.es_runs = algo == ME_ALGO_ES && es_use_runs(b, cfg.search_range) && b.cols < 4096 ? 1 : 0;
    {
        NvtxRange nv("me_b200/classify");
        if ((e = launch_classify(ca, num_sms, st))) return e;
    }
    if (events) cudaEventRecord(events[1], st);
    // PA kernel choice (pa.cu): the duo / quad kernels take list entries in
    // pairs / fours, so every wavefront step is padded to a multiple of 2 / 4;
    // the hybrids split the list into narrow / wide / narrow step ranges.
    const int pa_mode = pa ? pa_kernel_mode(b, cfg, prev0, prev0_integer, num_sms, tune) : 0;
    int* ranges = pa_mode >= 3 ? s.counter + 8 : nullptr;
    if (pa) {
        NvtxRange nv("me_b200/sort");
        if ((e = launch_scan(s.hist, nbins, pa_mode == 4 ? 4 : pa_mode >= 2 ? 2 : 1, s.offs, s.cursor, s.list,
                             pa_wide_threshold(num_sms, tune), ranges, st, tune.sort_pdl, ca.hist2, b.n_seq,
                             s.tmin)))
            return e;
        if ((e = launch_fill(ca, s.cursor, s.list, num_sms, st, tune))) return e;
    }
    const int* nlist = pa ? s.offs + nbins : ca.nlist_direct;
    if (events) cudaEventRecord(events[2], st);

    NvtxRange nv_search("me_b200/search");
    if (algo == ME_ALGO_ES)
        e = launch_es(b, cfg.search_range, s.list, nlist, s.counter, recs, stats, num_sms, st, s.types);
    else if (algo == ME_ALGO_PA)
        e = launch_pa(b, cfg, prev0, s.list, nlist, ranges, pa_mode, recs, stats, num_sms, st, s.counter + 1, tune);
    else
        e = launch_ring(b, algo, cfg.search_range, s.list, nlist, recs, stats, num_sms, st, tune.ring_ctas);
    if (e) return e;

    if (events) cudaEventRecord(events[3], st);
    if (pred && (e = launch_mc_pred(b, recs, pred, st))) return e;
    // classify, scan + fill (PA), the search (three launches for the PA hybrid), MC
    if (launches) *launches = 1 + (pa ? 2 : 0) + (pa_mode >= 3 ? 3 : 1) + (pred ? 1 : 0);
    if (events) cudaEventRecord(events[4], st);
    return cudaGetLastError();
}

cudaError_t block_search(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H, int x0,
                         int y0, int size, int range, int64_t* out, cudaStream_t st) {
    if (algo == ME_ALGO_ES) return launch_es_single(cur, ref, W, H, x0, y0, size, range, out, st);
    return launch_ring_single(algo, cur, ref, W, H, x0, y0, size, range, out, st);
}

}  // namespace mek
