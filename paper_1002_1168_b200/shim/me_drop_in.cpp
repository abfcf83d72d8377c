// me_drop_in.cpp — the C++ drop-in for the reference's motion-estimation
// entry points, backed by the sm_100a kernels through the C ABI
// (include/me_b200.h).
//
// It defines every symbol of the reference's proj/src/estimators.cpp and
// proj/src/compensation.cpp, compiled against the reference's OWN headers
// (proj/include/me/estimators.hpp, compensation.hpp) so the signatures cannot
// drift.  Linking it in place of those two translation units — next to the
// reference's unchanged frame.cpp / metrics.cpp / video_io.cpp / bench.cpp —
// turns any caller (run_experiment, the acceptance suite, an application)
// into a GPU user without a source change.  See INTEGRATION.md.
//
// Pixel work always runs on the GPU; only integer bookkeeping (window
// clipping, candidate gathering, validation) and two visualisation helpers
// off the hot path (residual, residual_to_gray) run on the host.  Errors map
// back to the reference's exception types.

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "me/compensation.hpp"
#include "me/estimators.hpp"
#include "me_b200.h"

namespace me {

namespace {

[[noreturn]] void raise(me_status s) {
    const std::string msg = me_b200_last_error();
    if (s == ME_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (s == ME_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error("me_b200: " + msg);
}

void check(me_status s) {
    if (s != ME_OK) raise(s);
}

// One context per host thread (the reference is re-entrant).
me_ctx* ctx() {
    struct Holder {
        me_ctx* c = nullptr;
        ~Holder() {
            if (c) me_b200_ctx_destroy(c);
        }
    };
    thread_local Holder h;
    if (!h.c) {
        const char* dev = std::getenv("ME_B200_DEVICE");
        check(me_b200_ctx_create(dev ? std::atoi(dev) : 0, &h.c));
    }
    return h.c;
}

me_config to_cfg(Algo algo, const SearchConfig& s, const PrsConfig& p, BoundaryTemporal bt) {
    me_config c{};
    c.algo = static_cast<int32_t>(algo);
    c.search_range = s.search_range;
    c.block_size = s.block_size;
    c.ref_distance = s.ref_distance;
    c.halfpel = s.halfpel ? 1 : 0;
    c.max_iterations = p.max_iterations;
    c.step = p.step;
    c.boundary_temporal = static_cast<int32_t>(bt);
    c.epsilon = p.epsilon;
    c.theta = p.theta;
    return c;
}

const uint8_t* luma(const Frame& f) { return f.luma.data.data(); }
const uint8_t* mask(const AlphaPlane* a) { return a ? a->mask.data.data() : nullptr; }

void require_inside(const Frame& cur, const BlockRect& rect) {  // estimators.cpp:105-110
    if (rect.x0 < 0 || rect.y0 < 0 || rect.size <= 0 || rect.x0 + rect.size > cur.luma.width ||
        rect.y0 + rect.size > cur.luma.height)
        throw std::invalid_argument("block rect outside the frame");
}

MotionVector block_search(Algo algo, const Frame& cur, const Frame& ref, const BlockRect& rect,
                          const SearchConfig& cfg, SearchStats& stats) {
    cfg.validate();
    require_inside(cur, rect);
    int32_t mv[2];
    int64_t cmp = 0;
    uint32_t cost = 0;
    check(me_b200_block_search(ctx(), static_cast<int>(algo), cur.luma.width, cur.luma.height,
                               luma(cur), luma(ref), rect.x0, rect.y0, rect.size, cfg.search_range,
                               mv, &cmp, &cost));
    stats.block_comparisons += cmp;
    return MotionVector{mv[0], mv[1]};
}

}  // namespace

// ---- estimators.hpp ---------------------------------------------------------

const char* to_string(Algo a) {  // estimators.cpp:116-125
    switch (a) {
        case Algo::ES: return "ES";
        case Algo::TSS: return "TSS";
        case Algo::FSS: return "FSS";
        case Algo::DS: return "DS";
        case Algo::PA: return "PA";
    }
    throw std::invalid_argument("unknown algorithm");
}

Algo algo_from_string(const std::string& name) {  // estimators.cpp:127-137
    std::string up;
    for (char ch : name) up.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(ch))));
    if (up == "ES") return Algo::ES;
    if (up == "TSS") return Algo::TSS;
    if (up == "FSS" || up == "4SS") return Algo::FSS;
    if (up == "DS") return Algo::DS;
    if (up == "PA") return Algo::PA;
    throw std::invalid_argument("unknown algorithm: " + name);
}

void SearchConfig::validate() const {  // estimators.cpp:139-143 (same checks as the C ABI)
    me_config c = to_cfg(Algo::ES, *this, PrsConfig{}, BoundaryTemporal::Texture);
    check(me_b200_validate_config(&c));
}

void PrsConfig::validate() const {  // estimators.cpp:145-150
    me_config c = to_cfg(Algo::ES, SearchConfig{}, *this, BoundaryTemporal::Texture);
    check(me_b200_validate_config(&c));
}

MotionField::MotionField(int cols_, int rows_, int block_size_)
    : cols(cols_),
      rows(rows_),
      block_size(block_size_),
      vectors(std::size_t(cols_ > 0 ? cols_ : 0) * (rows_ > 0 ? rows_ : 0)),
      types(std::size_t(cols_ > 0 ? cols_ : 0) * (rows_ > 0 ? rows_ : 0), BlockType::Opaque) {
    if (cols_ <= 0 || rows_ <= 0) throw std::invalid_argument("empty motion field grid");
}

MotionVector clip_to_window(MotionVector v, const BlockRect& rect, int width, int height,
                            int range_pels) {  // estimators.cpp:161-165
    const int lo_x = std::max(-2 * range_pels, -2 * rect.x0);
    const int hi_x = std::min(2 * range_pels, 2 * (width - rect.x0 - rect.size));
    const int lo_y = std::max(-2 * range_pels, -2 * rect.y0);
    const int hi_y = std::min(2 * range_pels, 2 * (height - rect.y0 - rect.size));
    return MotionVector{std::clamp(v.dx, lo_x, hi_x), std::clamp(v.dy, lo_y, hi_y)};
}

MotionVector full_search(const Frame& cur, const Frame& ref, const BlockRect& rect,
                         const SearchConfig& cfg, SearchStats& stats) {
    return block_search(Algo::ES, cur, ref, rect, cfg, stats);
}
MotionVector tss_search(const Frame& cur, const Frame& ref, const BlockRect& rect,
                        const SearchConfig& cfg, SearchStats& stats) {
    return block_search(Algo::TSS, cur, ref, rect, cfg, stats);
}
MotionVector fss_search(const Frame& cur, const Frame& ref, const BlockRect& rect,
                        const SearchConfig& cfg, SearchStats& stats) {
    return block_search(Algo::FSS, cur, ref, rect, cfg, stats);
}
MotionVector ds_search(const Frame& cur, const Frame& ref, const BlockRect& rect,
                       const SearchConfig& cfg, SearchStats& stats) {
    return block_search(Algo::DS, cur, ref, rect, cfg, stats);
}

CandidateSet gather_candidates(const MotionField& f, const MotionField* prev, int h, int v) {
    // estimators.cpp:238-255 (integer bookkeeping)
    if (h < 0 || v < 0 || h >= f.cols || v >= f.rows)
        throw std::out_of_range("block coordinates outside the motion field grid");
    CandidateSet cs;
    if (h - 1 >= 0) cs.a = f.at(h - 1, v);
    if (v - 1 >= 0) cs.b = f.at(h, v - 1);
    if (h + 1 < f.cols && v - 1 >= 0) cs.c = f.at(h + 1, v - 1);
    if (prev != nullptr) {
        if (prev->cols != f.cols || prev->rows != f.rows)
            throw std::invalid_argument("previous motion field grid mismatch");
        cs.t = prev->at(h, v);
    }
    return cs;
}

MotionVector brs_select(const Frame& cur, const Frame& ref, const AlphaPlane* cur_alpha,
                        const AlphaPlane* ref_alpha, const BlockRect& rect, BlockType btype,
                        const CandidateSet& cands, const SearchConfig& cfg,
                        const EstimateOptions& opts, SearchStats& stats) {
    cfg.validate();
    require_inside(cur, rect);
    const int32_t cd[8] = {cands.a.dx, cands.a.dy, cands.b.dx, cands.b.dy,
                           cands.c.dx, cands.c.dy, cands.t.dx, cands.t.dy};
    int32_t mv[2];
    uint8_t kinds[4];
    uint32_t scores[4];
    check(me_b200_brs_select(ctx(), cur.luma.width, cur.luma.height, luma(cur), luma(ref),
                             mask(cur_alpha), mask(ref_alpha), rect.x0, rect.y0, rect.size,
                             static_cast<int>(btype), cd, cfg.search_range,
                             static_cast<int>(opts.boundary_temporal), mv, kinds, scores));
    stats.block_comparisons += 4;
    if (opts.scoring_log != nullptr)
        for (int i = 0; i < 4; ++i)
            opts.scoring_log->push_back({rect.x0 / rect.size, rect.y0 / rect.size, btype, i,
                                         static_cast<ScoreKind>(kinds[i])});
    return MotionVector{mv[0], mv[1]};
}

Vec2 prs_update(const Frame& cur, const Frame& ref, int x, int y, MotionVector d_i,
                const PrsConfig& cfg) {
    const int32_t d[2] = {d_i.dx, d_i.dy};
    double out[2];
    check(me_b200_prs_update(ctx(), cur.luma.width, cur.luma.height, luma(cur), luma(ref), x, y, d,
                             cfg.epsilon, cfg.theta, out));
    return Vec2{out[0], out[1]};
}

MotionVector prs_refine(const Frame& cur, const Frame& ref, const BlockRect& rect,
                        MotionVector d0, const SearchConfig& scfg, const PrsConfig& cfg,
                        SearchStats& stats, std::vector<double>* descent_log) {
    scfg.validate();
    cfg.validate();
    require_inside(cur, rect);
    const int32_t d[2] = {d0.dx, d0.dy};
    int32_t mv[2];
    int64_t dpd = 0;
    uint32_t log_q4[64];
    int n = 0;
    check(me_b200_prs_refine(ctx(), cur.luma.width, cur.luma.height, luma(cur), luma(ref), rect.x0,
                             rect.y0, rect.size, d, scfg.search_range, cfg.epsilon, cfg.theta,
                             cfg.max_iterations, cfg.step, mv, &dpd, log_q4, &n));
    stats.dpd_refinement_steps += dpd;
    if (descent_log != nullptr)
        for (int i = 0; i < n && i < 64; ++i) descent_log->push_back(log_q4[i] / 4.0);
    return MotionVector{mv[0], mv[1]};
}

std::pair<MotionField, SearchStats> estimate_field(Algo algo, const Frame& cur, const Frame& ref,
                                                   const AlphaPlane* cur_alpha,
                                                   const AlphaPlane* ref_alpha,
                                                   const MotionField* prev_field,
                                                   const SearchConfig& cfg, const PrsConfig& prs,
                                                   const EstimateOptions& opts) {
    // estimators.cpp:384-440, one frame pair through the batched GPU pipeline
    cfg.validate();
    prs.validate();
    if (cur.luma.width != ref.luma.width || cur.luma.height != ref.luma.height)
        throw std::invalid_argument("current and reference frame dimensions differ");
    const int W = cur.luma.width, H = cur.luma.height, bs = cfg.block_size;
    if (bs <= 0 || W % bs != 0 || H % bs != 0)
        throw std::invalid_argument("block size " + std::to_string(bs) + " does not divide " +
                                    std::to_string(W) + "x" + std::to_string(H));
    MotionField field(W / bs, H / bs, bs);
    field.cur_index = cur.index;
    field.ref_index = ref.index;
    if (prev_field != nullptr && (prev_field->cols != field.cols || prev_field->rows != field.rows))
        throw std::invalid_argument("previous motion field grid mismatch");
    std::vector<int32_t> prev;
    if (prev_field != nullptr) {
        prev.resize(prev_field->vectors.size() * 2);
        for (std::size_t i = 0; i < prev_field->vectors.size(); ++i) {
            prev[2 * i] = prev_field->vectors[i].dx;
            prev[2 * i + 1] = prev_field->vectors[i].dy;
        }
    }
    const me_config c = to_cfg(algo, cfg, prs, opts.boundary_temporal);
    std::vector<me_block_rec> recs(field.vectors.size());
    me_pair_stats st{};
    const auto t0 = std::chrono::steady_clock::now();
    check(me_b200_estimate_field(ctx(), &c, W, H, luma(cur), luma(ref), mask(cur_alpha),
                                 mask(ref_alpha), prev_field ? prev.data() : nullptr, field.cols,
                                 field.rows, recs.data(), &st));
    SearchStats stats;
    stats.elapsed = std::chrono::duration_cast<std::chrono::microseconds>(
        std::chrono::steady_clock::now() - t0);
    stats.block_comparisons = st.block_comparisons;
    stats.dpd_refinement_steps = st.dpd_refinement_steps;
    stats.blocks_opaque = st.blocks_opaque;
    stats.blocks_boundary = st.blocks_boundary;
    stats.blocks_transparent = st.blocks_transparent;
    for (std::size_t i = 0; i < recs.size(); ++i) {
        field.vectors[i] = MotionVector{recs[i].dx, recs[i].dy};
        field.types[i] = static_cast<BlockType>(recs[i].type);
    }
    if (opts.scoring_log != nullptr && algo == Algo::PA) {
        // the scoring kind is a pure function of (type, candidate,
        // boundary_temporal) (estimators.cpp:277-279); raster block order
        for (std::size_t i = 0; i < recs.size(); ++i) {
            const BlockType t = field.types[i];
            if (t == BlockType::Transparent) continue;
            for (int k = 0; k < 4; ++k) {
                const bool shape = t == BlockType::Boundary &&
                                   (k < 3 || opts.boundary_temporal == BoundaryTemporal::Shape);
                opts.scoring_log->push_back({int(i % field.cols), int(i / field.cols), t, k,
                                             shape ? ScoreKind::Shape : ScoreKind::Texture});
            }
        }
    }
    return {std::move(field), stats};
}

// ---- compensation.hpp -------------------------------------------------------

ResidualPlane::ResidualPlane(int w, int h)
    : width(w), height(h), samples(std::size_t(w > 0 ? w : 0) * std::size_t(h > 0 ? h : 0)) {
    if (w <= 0 || h <= 0) throw std::invalid_argument("residual plane dimensions must be positive");
}

Frame predict_frame(const Frame& ref, const MotionField& field, const SearchConfig& cfg) {
    // compensation.cpp:30-71: luma on the GPU, chroma carried over from ref
    cfg.validate();
    if (field.block_size != cfg.block_size)
        throw std::invalid_argument("motion field block size does not match the configuration");
    if (field.cols * field.block_size != ref.luma.width ||
        field.rows * field.block_size != ref.luma.height)
        throw std::invalid_argument("motion field grid does not cover the frame");
    std::vector<int32_t> mv(field.vectors.size() * 2);
    std::vector<uint8_t> types(field.types.size());
    for (std::size_t i = 0; i < field.vectors.size(); ++i) {
        mv[2 * i] = field.vectors[i].dx;
        mv[2 * i + 1] = field.vectors[i].dy;
        types[i] = static_cast<uint8_t>(field.types[i]);
    }
    Frame pred = ref;
    pred.index = field.cur_index;
    check(me_b200_predict_frame(ctx(), ref.luma.width, ref.luma.height, luma(ref), mv.data(),
                                types.data(), field.block_size, nullptr, pred.luma.data.data(),
                                nullptr));
    return pred;
}

ResidualPlane residual(const Frame& cur, const Frame& pred) {
    // compensation.cpp:73-84 — host utility off the hot path (dumps, tests)
    if (cur.luma.width != pred.luma.width || cur.luma.height != pred.luma.height)
        throw std::invalid_argument("residual operands have different dimensions");
    ResidualPlane r(cur.luma.width, cur.luma.height);
    for (std::size_t i = 0; i < r.samples.size(); ++i)
        r.samples[i] = static_cast<std::int16_t>(int(cur.luma.data[i]) - int(pred.luma.data[i]));
    return r;
}

Plane residual_to_gray(const ResidualPlane& r) {
    // compensation.cpp:86-94 — visualisation, off the hot path
    Plane gray(r.width, r.height);
    for (std::size_t i = 0; i < r.samples.size(); ++i)
        gray.data[i] = static_cast<std::uint8_t>(std::clamp(int(r.samples[i]) + 128, 0, 255));
    return gray;
}

}  // namespace me
