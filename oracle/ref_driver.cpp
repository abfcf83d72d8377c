// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" driver around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libme_ref.so).  It exposes the reference's own results in the
// record layout of include/me_b200.h so the Python tests can compare the CUDA
// path against the real reference on identical bytes:
//   * ref_run_sequence  — run_experiment's pair loop (bench.cpp:155-205):
//       estimate_field (estimators.cpp:384) + predict_frame
//       (compensation.cpp:30) + psnr (metrics.cpp:108), PA threading `prev`.
//     Per-block costs and counts are not returned by estimate_field, so each
//     estimated block is REPLAYED through the per-block entry points with a
//     fresh SearchStats (full_search/tss/fss/ds, or gather_candidates +
//     brs_select + prs_refine with a descent_log), and the replayed vector is
//     checked against estimate_field's; the aggregate SearchStats of the
//     replay must equal estimate_field's too (returns -1 otherwise).
//   * ref_run_experiment — the reference's own run_experiment (bench.cpp:120-227)
//       on a sequence file: writes its CSV and returns the AlgoSummary values
//       (golden source for the experiment-report tests).
//   * ref_* per-block wrappers used by the unit-level parity tests.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load this library.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "me/bench.hpp"
#include "me/compensation.hpp"
#include "me/estimators.hpp"
#include "me/video_io.hpp"
#include "me/frame.hpp"
#include "me/metrics.hpp"
#include "me_b200.h"

using namespace me;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::out_of_range*>(&e)) return ME_ERR_OUT_OF_RANGE;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return ME_ERR_INVALID_ARGUMENT;
    return ME_ERR_RUNTIME;
}

Frame frame_from(const uint8_t* p, int w, int h, int index) {
    Plane pl(w, h);
    std::memcpy(pl.data.data(), p, size_t(w) * h);
    Frame f;  // no make_frame: per-block tests use sizes that are not multiples of 16
    f.luma = std::move(pl);
    f.index = index;
    return f;
}

AlphaPlane alpha_from(const uint8_t* p, int w, int h) {
    AlphaPlane a;
    a.mask = Plane(w, h);
    std::memcpy(a.mask.data.data(), p, size_t(w) * h);
    return a;
}

SearchConfig scfg_of(const me_config* c) {
    SearchConfig s;
    s.search_range = c->search_range;
    s.block_size = c->block_size;
    s.ref_distance = c->ref_distance;
    s.halfpel = c->halfpel != 0;
    return s;
}

PrsConfig prs_of(const me_config* c) {
    PrsConfig p;
    p.epsilon = c->epsilon;
    p.theta = c->theta;
    p.max_iterations = c->max_iterations;
    p.step = c->step;
    return p;
}

uint32_t q4(double sad) { return uint32_t(std::llround(sad * 4.0)); }

// One pair: estimate_field + per-block replay + predict_frame + SSE.
int run_pair(const me_config* c, const Frame& cur, const Frame& ref, const AlphaPlane* ca,
             const AlphaPlane* ra, const MotionField* prev, MotionField& field_out,
             me_block_rec* recs, me_pair_stats* st, uint8_t* pred_out) {
    const Algo algo = static_cast<Algo>(c->algo);
    SearchConfig scfg = scfg_of(c);
    PrsConfig prs = prs_of(c);
    EstimateOptions opts;
    opts.boundary_temporal = static_cast<BoundaryTemporal>(c->boundary_temporal);
    auto [field, stats] = estimate_field(algo, cur, ref, ca, ra, prev, scfg, prs, opts);

    PrsConfig prs_eff = prs;
    if (scfg.halfpel) prs_eff.step = 1;
    SearchStats replay;
    for (const BlockRect& rect : block_grid(cur, scfg.block_size)) {
        const size_t i = size_t(rect.grid_v) * field.cols + rect.grid_h;
        me_block_rec& r = recs[i];
        std::memset(&r, 0, sizeof r);
        const BlockType bt = field.types[i];
        r.type = uint8_t(bt);
        if (bt == BlockType::Transparent) continue;
        SearchStats bs;
        MotionVector v;
        std::vector<double> log;
        switch (algo) {
            case Algo::ES: v = full_search(cur, ref, rect, scfg, bs); break;
            case Algo::TSS: v = tss_search(cur, ref, rect, scfg, bs); break;
            case Algo::FSS: v = fss_search(cur, ref, rect, scfg, bs); break;
            case Algo::DS: v = ds_search(cur, ref, rect, scfg, bs); break;
            case Algo::PA: {
                const CandidateSet cs = gather_candidates(field, prev, rect.grid_h, rect.grid_v);
                const MotionVector v0 =
                    brs_select(cur, ref, ca, ra, rect, bt, cs, scfg, opts, bs);
                v = prs_refine(cur, ref, rect, v0, scfg, prs_eff, bs, &log);
                break;
            }
        }
        if (!(v == field.vectors[i])) {
            g_err = "replay mismatch at block " + std::to_string(i);
            return -1;
        }
        r.dx = int16_t(v.dx);
        r.dy = int16_t(v.dy);
        r.comparisons = uint16_t(std::min<std::int64_t>(bs.block_comparisons, 65535));  // saturated (ES at S >= 128)
        r.dpd_steps = uint16_t(bs.dpd_refinement_steps);
        r.iterations = algo == Algo::PA ? uint8_t(log.size() - 1) : 0;
        r.cost_q4 = algo == Algo::PA ? q4(log.back()) : q4(sad_texture(cur, ref, rect, v));
        replay.block_comparisons += bs.block_comparisons;
        replay.dpd_refinement_steps += bs.dpd_refinement_steps;
    }
    if (replay.block_comparisons != stats.block_comparisons ||
        replay.dpd_refinement_steps != stats.dpd_refinement_steps) {
        g_err = "replay stats mismatch";
        return -1;
    }
    const Frame pred = predict_frame(ref, field, scfg);
    int64_t sse = 0;
    for (size_t k = 0; k < pred.luma.data.size(); ++k) {
        const int d = int(cur.luma.data[k]) - int(pred.luma.data[k]);
        sse += int64_t(d) * d;
    }
    // cross-check against the reference's own psnr()
    const PsnrResult pr = psnr(cur, pred);
    if (pr.mse != double(sse) / double(pred.luma.data.size())) {
        g_err = "psnr mse mismatch";
        return -1;
    }
    if (pred_out) std::memcpy(pred_out, pred.luma.data.data(), pred.luma.data.size());
    st->block_comparisons = stats.block_comparisons;
    st->dpd_refinement_steps = stats.dpd_refinement_steps;
    st->blocks_opaque = stats.blocks_opaque;
    st->blocks_boundary = stats.blocks_boundary;
    st->blocks_transparent = stats.blocks_transparent;
    st->sse = sse;
    field_out = std::move(field);
    return 0;
}

int run_sequence_impl(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                      const uint8_t* alpha, me_block_rec* recs, me_pair_stats* stats,
                      uint8_t* pred, bool replay_only_fast) {
    (void)replay_only_fast;
    const size_t plane = size_t(w) * h;
    std::vector<Frame> frames;
    std::vector<AlphaPlane> masks;
    for (int t = 0; t < n_frames; ++t) {
        frames.push_back(make_frame([&] {
            Plane p(w, h);
            std::memcpy(p.data.data(), luma + plane * t, plane);
            return p;
        }(), t));
        if (alpha) masks.push_back(alpha_from(alpha + plane * t, w, h));
    }
    const int d = c->ref_distance;
    const int bs = c->block_size;
    const size_t nblk = size_t(w / bs) * (h / bs);
    std::optional<MotionField> prev;
    for (int tau = d; tau < n_frames; ++tau) {
        const int p = tau - d;
        MotionField field;
        const int rc = run_pair(c, frames[tau], frames[tau - d], alpha ? &masks[tau] : nullptr,
                                alpha ? &masks[tau - d] : nullptr, prev ? &*prev : nullptr, field,
                                recs + nblk * p, stats + p, pred ? pred + plane * p : nullptr);
        if (rc != 0) return rc;
        if (c->algo == ME_ALGO_PA) prev = std::move(field);
    }
    return 0;
}

// Result digest of one sequence (order-dependent, uint64 wrap-around):
// sum over pairs p and blocks i (raster) of (dx * 0x9E37 + dy * 0x7F4B + 1) *
// (2 * (p * blocks + i) + 1), plus sum over pairs of the SearchStats counters
// and the exact SSE (psnr's mse * W * H, rounded) with fixed weights.  The same
// digest computed from the CUDA path's records and stats (bench.py) checks
// the benchmarked batch against the reference without shipping every record.
struct Digest {
    uint64_t v = 0;
    void field(const MotionField& f, uint64_t pair) {
        const uint64_t n = f.vectors.size();
        for (uint64_t i = 0; i < n; ++i) {
            const MotionVector& m = f.vectors[i];
            v += (uint64_t(int64_t(m.dx)) * 0x9E37u + uint64_t(int64_t(m.dy)) * 0x7F4Bu + 1u) * (2u * (pair * n + i) + 1u);
        }
    }
    void stats(const SearchStats& s, int64_t sse) {
        v += uint64_t(s.block_comparisons) * 1000003u + uint64_t(s.dpd_refinement_steps) * 7919u +
             uint64_t(s.blocks_opaque) * 131u + uint64_t(s.blocks_boundary) * 137u +
             uint64_t(s.blocks_transparent) * 139u + uint64_t(sse) * 17u;
    }
};

// Plain timing path: estimate_field + predict_frame + psnr exactly as
// run_experiment calls them (no replay), for the CPU baseline.
int time_sequence_impl(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                       const uint8_t* alpha, int64_t* mvsum, uint64_t* digest = nullptr) {
    const size_t plane = size_t(w) * h;
    std::vector<Frame> frames;
    std::vector<AlphaPlane> masks;
    for (int t = 0; t < n_frames; ++t) {
        Plane pl(w, h);
        std::memcpy(pl.data.data(), luma + plane * t, plane);
        frames.push_back(make_frame(std::move(pl), t));
        if (alpha) masks.push_back(alpha_from(alpha + plane * t, w, h));
    }
    SearchConfig scfg = scfg_of(c);
    PrsConfig prs = prs_of(c);
    EstimateOptions opts;
    opts.boundary_temporal = static_cast<BoundaryTemporal>(c->boundary_temporal);
    const Algo algo = static_cast<Algo>(c->algo);
    std::optional<MotionField> prev;
    int64_t acc = 0;
    Digest dg;
    for (int tau = c->ref_distance; tau < n_frames; ++tau) {
        const Frame& cur = frames[tau];
        const Frame& ref = frames[tau - c->ref_distance];
        auto [field, stats] = estimate_field(algo, cur, ref, alpha ? &masks[tau] : nullptr,
                                             alpha ? &masks[tau - c->ref_distance] : nullptr,
                                             prev ? &*prev : nullptr, scfg, prs, opts);
        const Frame pred = predict_frame(ref, field, scfg);
        const PsnrResult pr = psnr(cur, pred);
        if (digest) {
            dg.field(field, uint64_t(tau - c->ref_distance));
            dg.stats(stats, int64_t(std::llround(pr.mse * double(plane))));
        }
        acc += stats.block_comparisons + int64_t(pr.mse);
        for (const MotionVector& v : field.vectors) acc += v.dx + 3 * v.dy;
        if (algo == Algo::PA) prev = std::move(field);
    }
    if (mvsum) *mvsum = acc;
    if (digest) *digest = dg.v;
    return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_run_sequence(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                     const uint8_t* alpha, me_block_rec* recs, me_pair_stats* stats,
                     uint8_t* pred) {
    try {
        return run_sequence_impl(c, n_frames, w, h, luma, alpha, recs, stats, pred, false);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Times `n_seq` independent sequences of the same shape on `threads` host
// threads (one sequence per thread at a time), the reference's own code path.
// Returns 0; *checksum is an order-independent digest of the results.
int ref_time_sequences_digest(const me_config* c, int n_seq, int n_frames, int w, int h,
                              const uint8_t* luma, const uint8_t* alpha, int threads, int64_t* checksum,
                              uint64_t* digests);
int ref_time_sequences(const me_config* c, int n_seq, int n_frames, int w, int h,
                       const uint8_t* luma, const uint8_t* alpha, int threads, int64_t* checksum) {
    return ref_time_sequences_digest(c, n_seq, n_frames, w, h, luma, alpha, threads, checksum, nullptr);
}

// As ref_time_sequences, plus the per-sequence result digest (Digest above)
// into digests[n_seq] when non-null.
int ref_time_sequences_digest(const me_config* c, int n_seq, int n_frames, int w, int h,
                              const uint8_t* luma, const uint8_t* alpha, int threads, int64_t* checksum,
                              uint64_t* digests) {
    std::atomic<int> next{0};
    std::atomic<int64_t> sum{0};
    std::atomic<int> rc{0};
    const size_t seq = size_t(w) * h * n_frames;
    auto worker = [&] {
        for (;;) {
            const int s = next.fetch_add(1);
            if (s >= n_seq) return;
            int64_t cs = 0;
            try {
                time_sequence_impl(c, n_frames, w, h, luma + seq * s,
                                   alpha ? alpha + seq * s : nullptr, &cs, digests ? digests + s : nullptr);
            } catch (const std::exception& e) {
                rc = fail(e);
            }
            sum += cs;
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (checksum) *checksum = sum.load();
    return rc.load();
}

// Times a list of (sequence, pair) units for the pair-parallel baselines
// (ES/TSS/FSS/DS): each unit is one estimate_field + predict_frame + psnr.
int ref_time_pairs(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                   const uint8_t* alpha, int first_pair, int n_pairs, int threads,
                   int64_t* checksum) {
    std::atomic<int> next{0};
    std::atomic<int64_t> sum{0};
    std::atomic<int> rc{0};
    const size_t plane = size_t(w) * h;
    auto worker = [&] {
        for (;;) {
            const int k = next.fetch_add(1);
            if (k >= n_pairs) return;
            const int tau = c->ref_distance + first_pair + k;
            if (tau >= n_frames) return;
            try {
                const Frame cur = frame_from(luma + plane * tau, w, h, tau);
                const Frame ref = frame_from(luma + plane * (tau - c->ref_distance), w, h, 0);
                std::optional<AlphaPlane> ca, ra;
                if (alpha) {
                    ca = alpha_from(alpha + plane * tau, w, h);
                    ra = alpha_from(alpha + plane * (tau - c->ref_distance), w, h);
                }
                auto [field, stats] =
                    estimate_field(static_cast<Algo>(c->algo), cur, ref, ca ? &*ca : nullptr,
                                   ra ? &*ra : nullptr, nullptr, scfg_of(c), prs_of(c));
                const Frame pred = predict_frame(ref, field, scfg_of(c));
                const PsnrResult pr = psnr(cur, pred);
                int64_t cs = stats.block_comparisons + int64_t(pr.mse);
                for (const MotionVector& v : field.vectors) cs += v.dx + 3 * v.dy;
                sum += cs;
            } catch (const std::exception& e) {
                rc = fail(e);
            }
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (checksum) *checksum = sum.load();
    return rc.load();
}

// Times ES on a bounded list of blocks of one pair (the 4K ES CPU sample).
int ref_time_blocks(const me_config* c, int w, int h, const uint8_t* cur_p, const uint8_t* ref_p,
                    const int32_t* block_xy, int n_blocks, int threads, int64_t* comparisons) {
    const Frame cur = frame_from(cur_p, w, h, 1);
    const Frame ref = frame_from(ref_p, w, h, 0);
    std::atomic<int> next{0};
    std::atomic<int64_t> cmp{0};
    const SearchConfig scfg = scfg_of(c);
    auto worker = [&] {
        for (;;) {
            const int k = next.fetch_add(1);
            if (k >= n_blocks) return;
            const BlockRect r{block_xy[2 * k], block_xy[2 * k + 1], c->block_size,
                              block_xy[2 * k] / c->block_size, block_xy[2 * k + 1] / c->block_size};
            SearchStats st;
            switch (static_cast<Algo>(c->algo)) {
                case Algo::ES: full_search(cur, ref, r, scfg, st); break;
                case Algo::TSS: tss_search(cur, ref, r, scfg, st); break;
                case Algo::FSS: fss_search(cur, ref, r, scfg, st); break;
                default: ds_search(cur, ref, r, scfg, st); break;
            }
            cmp += st.block_comparisons;
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (comparisons) *comparisons = cmp.load();
    return 0;
}

// ---- per-block wrappers --------------------------------------------------

int ref_block_search(int algo, int w, int h, const uint8_t* cur_p, const uint8_t* ref_p, int x0,
                     int y0, int size, int range, int32_t* mv, int64_t* cmp, uint32_t* cost_q4) {
    try {
        const Frame cur = frame_from(cur_p, w, h, 1);
        const Frame ref = frame_from(ref_p, w, h, 0);
        SearchConfig s;
        s.search_range = range;
        s.block_size = size;
        const BlockRect r{x0, y0, size, 0, 0};
        SearchStats st;
        MotionVector v;
        switch (static_cast<Algo>(algo)) {
            case Algo::ES: v = full_search(cur, ref, r, s, st); break;
            case Algo::TSS: v = tss_search(cur, ref, r, s, st); break;
            case Algo::FSS: v = fss_search(cur, ref, r, s, st); break;
            case Algo::DS: v = ds_search(cur, ref, r, s, st); break;
            default: throw std::invalid_argument("not a block search");
        }
        mv[0] = v.dx;
        mv[1] = v.dy;
        *cmp = st.block_comparisons;
        *cost_q4 = q4(sad_texture(cur, ref, r, v));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_brs_select(int w, int h, const uint8_t* cur_p, const uint8_t* ref_p, const uint8_t* ca_p,
                   const uint8_t* ra_p, int x0, int y0, int size, int btype, const int32_t* cands,
                   int range, int boundary_temporal, int32_t* mv, uint8_t* kinds,
                   int64_t* cmp) {
    try {
        const Frame cur = frame_from(cur_p, w, h, 1);
        const Frame ref = frame_from(ref_p, w, h, 0);
        std::optional<AlphaPlane> ca, ra;
        if (ca_p) ca = alpha_from(ca_p, w, h);
        if (ra_p) ra = alpha_from(ra_p, w, h);
        SearchConfig s;
        s.search_range = range;
        s.block_size = size;
        const BlockRect r{x0, y0, size, x0 / size, y0 / size};
        CandidateSet cs;
        cs.a = {cands[0], cands[1]};
        cs.b = {cands[2], cands[3]};
        cs.c = {cands[4], cands[5]};
        cs.t = {cands[6], cands[7]};
        std::vector<ScoreEvent> log;
        EstimateOptions opts;
        opts.boundary_temporal = static_cast<BoundaryTemporal>(boundary_temporal);
        opts.scoring_log = &log;
        SearchStats st;
        const MotionVector v = brs_select(cur, ref, ca ? &*ca : nullptr, ra ? &*ra : nullptr, r,
                                          static_cast<BlockType>(btype), cs, s, opts, st);
        mv[0] = v.dx;
        mv[1] = v.dy;
        for (size_t i = 0; i < log.size() && i < 4; ++i) kinds[i] = uint8_t(log[i].kind);
        *cmp = st.block_comparisons;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_prs_refine(int w, int h, const uint8_t* cur_p, const uint8_t* ref_p, int x0, int y0,
                   int size, const int32_t* d0, int range, double eps, double theta, int max_iter,
                   int step, int32_t* mv, int64_t* dpd, uint32_t* log_q4, int* log_len) {
    try {
        const Frame cur = frame_from(cur_p, w, h, 1);
        const Frame ref = frame_from(ref_p, w, h, 0);
        SearchConfig s;
        s.search_range = range;
        s.block_size = size;
        PrsConfig p;
        p.epsilon = eps;
        p.theta = theta;
        p.max_iterations = max_iter;
        p.step = step;
        SearchStats st;
        std::vector<double> log;
        const MotionVector v =
            prs_refine(cur, ref, BlockRect{x0, y0, size, 0, 0}, {d0[0], d0[1]}, s, p, st, &log);
        mv[0] = v.dx;
        mv[1] = v.dy;
        *dpd = st.dpd_refinement_steps;
        *log_len = int(log.size());
        for (size_t i = 0; i < log.size(); ++i) log_q4[i] = q4(log[i]);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_prs_update(int w, int h, const uint8_t* cur_p, const uint8_t* ref_p, int x, int y,
                   const int32_t* d, double eps, double theta, double* out) {
    try {
        const Frame cur = frame_from(cur_p, w, h, 1);
        const Frame ref = frame_from(ref_p, w, h, 0);
        PrsConfig p;
        p.epsilon = eps;
        p.theta = theta;
        const Vec2 v = prs_update(cur, ref, x, y, {d[0], d[1]}, p);
        out[0] = v.x;
        out[1] = v.y;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_sad_texture(int w, int h, const uint8_t* cur_p, const uint8_t* ref_p, int x0, int y0,
                    int size, int dx, int dy, double* out) {
    try {
        *out = sad_texture(frame_from(cur_p, w, h, 1), frame_from(ref_p, w, h, 0),
                           BlockRect{x0, y0, size, 0, 0}, {dx, dy});
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_sad_shape(int w, int h, const uint8_t* ca, const uint8_t* ra, int x0, int y0, int size,
                  int dx, int dy, int64_t* out) {
    try {
        *out = sad_shape(alpha_from(ca, w, h), alpha_from(ra, w, h), BlockRect{x0, y0, size, 0, 0},
                         {dx, dy});
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_classify(int w, int h, const uint8_t* alpha, int size, uint8_t* types) {
    try {
        std::optional<AlphaPlane> a;
        if (alpha) a = alpha_from(alpha, w, h);
        for (const BlockRect& r : block_grid(w, h, size))
            types[size_t(r.grid_v) * (w / size) + r.grid_h] =
                uint8_t(classify_block(a ? &*a : nullptr, r));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_binarize(int w, int h, const uint8_t* gray, int threshold, uint8_t* out) {
    Plane p(w, h);
    std::memcpy(p.data.data(), gray, size_t(w) * h);
    const AlphaPlane a = binarize(p, threshold);
    std::memcpy(out, a.mask.data.data(), size_t(w) * h);
    return 0;
}

int ref_predict_frame(int w, int h, const uint8_t* ref_p, const int32_t* mv,
                      const uint8_t* types, int bs, uint8_t* pred) {
    try {
        const Frame ref = frame_from(ref_p, w, h, 0);
        MotionField f(w / bs, h / bs, bs);
        for (size_t i = 0; i < f.vectors.size(); ++i) {
            f.vectors[i] = {mv[2 * i], mv[2 * i + 1]};
            if (types) f.types[i] = static_cast<BlockType>(types[i]);
        }
        SearchConfig s;
        s.block_size = bs;
        const Frame p = predict_frame(ref, f, s);
        std::memcpy(pred, p.luma.data.data(), size_t(w) * h);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_psnr(int w, int h, const uint8_t* a, const uint8_t* b, double* mse, double* db,
             int* infinite) {
    const PsnrResult r = psnr(frame_from(a, w, h, 0), frame_from(b, w, h, 0));
    *mse = r.mse;
    *infinite = r.infinite() ? 1 : 0;
    *db = r.psnr_db ? *r.psnr_db : 0.0;
    return 0;
}


// run_experiment (bench.cpp:120-227) on an I420 (format 0) or Y4M (1) file.
// summaries: n_algos x 10 doubles {frame_pairs, mean_mse, mean_psnr_db,
// psnr_db_of_mean_mse, mean_psnr_linear, avg_search_points, indicator,
// total_comparisons, total_dpd_steps, total_blocks_estimated}; absent
// optionals are NaN.
int ref_run_experiment(const char* path, int format, int w, int h, const char* mask_pattern,
                       const int* algos, int n_algos, const me_config* c, int block_size_auto,
                       int frame_limit, const char* csv_path, const char* dump_dir, double* summaries) {
    try {
        ExperimentConfig cfg;
        cfg.source = format ? open_y4m(path) : open_i420(path, w, h);
        if (mask_pattern) cfg.masks.pattern = mask_pattern;
        for (int i = 0; i < n_algos; ++i) cfg.algos.push_back(static_cast<Algo>(algos[i]));
        cfg.search.search_range = c->search_range;
        cfg.search.block_size = c->block_size;
        cfg.search.ref_distance = c->ref_distance;
        cfg.search.halfpel = c->halfpel != 0;
        cfg.prs.epsilon = c->epsilon;
        cfg.prs.theta = c->theta;
        cfg.prs.max_iterations = c->max_iterations;
        cfg.prs.step = c->step;
        cfg.boundary_temporal = c->boundary_temporal ? BoundaryTemporal::Shape : BoundaryTemporal::Texture;
        cfg.block_size_auto = block_size_auto != 0;
        cfg.frame_limit = frame_limit;
        if (csv_path) cfg.csv_path = csv_path;
        if (dump_dir) cfg.dump_dir = dump_dir;
        const ExperimentResult r = run_experiment(cfg);
        const double nan = std::nan("");
        for (std::size_t i = 0; i < r.summaries.size(); ++i) {
            const AlgoSummary& s = r.summaries[i];
            double* o = summaries + 10 * i;
            o[0] = s.frame_pairs;
            o[1] = s.mean_mse;
            o[2] = s.mean_psnr_db ? *s.mean_psnr_db : nan;
            o[3] = s.psnr_db_of_mean_mse ? *s.psnr_db_of_mean_mse : nan;
            o[4] = s.mean_psnr_linear ? *s.mean_psnr_linear : nan;
            o[5] = s.avg_search_points;
            o[6] = s.indicator ? *s.indicator : nan;
            o[7] = double(s.total_comparisons);
            o[8] = double(s.total_dpd_steps);
            o[9] = double(s.total_blocks_estimated);
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
