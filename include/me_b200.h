/*
 * me_b200.h — C ABI of the B200-native shape-adaptive motion-estimation hot path.
 *
 * Every entry point replaces one C++ entry point of the reference library
 * (mebench, /root/reference/proj).  The reference has no FFI of its own: its
 * operator boundary is the C++ API in proj/include/me/estimators.hpp and
 * proj/include/me/compensation.hpp, and its per-algorithm dispatch is the
 * `switch (algo)` at proj/src/estimators.cpp:421-434.  This header is what a
 * foreign-language binding (ctypes, cgo, JNI, the C++ drop-in shim under
 * paper_1002_1168_b200/shim/) links against.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - Planes are 8-bit, row-major, pitch == width (reference me::Plane,
 *    frame.hpp:26-47).  Width and height are positive multiples of 16
 *    (check_dimensions, frame.cpp:34-40).
 *  - Motion vectors are half-pel units (MotionVector, frame.hpp:84-95).
 *  - Every function returns an me_status; no exception crosses the ABI.  The
 *    C++ shim maps ME_ERR_INVALID_ARGUMENT -> std::invalid_argument and
 *    ME_ERR_OUT_OF_RANGE -> std::out_of_range, the reference's error types
 *    (SURVEY §8b).  All argument validation happens before any device work.
 *  - Functions whose name ends in `_dev` take DEVICE pointers and enqueue on
 *    the given cudaStream_t (passed as void*); all others take HOST pointers
 *    and are synchronous.
 *  - There is no CPU fallback.  Without a usable sm_100 device every compute
 *    entry point returns ME_ERR_NO_DEVICE.
 */
#ifndef ME_B200_H
#define ME_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ME_B200_ABI_VERSION 1

typedef enum me_status {
    ME_OK = 0,
    ME_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    ME_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range in the reference */
    ME_ERR_CUDA = 3,             /* a CUDA runtime error (message in me_b200_last_error) */
    ME_ERR_NO_DEVICE = 4,        /* no sm_100 device: the product path refuses to run */
    ME_ERR_RUNTIME = 5           /* std::runtime_error-class failure (allocation, ...) */
} me_status;

/* me::Algo (estimators.hpp:29). */
typedef enum me_algo { ME_ALGO_ES = 0, ME_ALGO_TSS = 1, ME_ALGO_FSS = 2, ME_ALGO_DS = 3, ME_ALGO_PA = 4 } me_algo;

/* me::BlockType (frame.hpp:71). */
typedef enum me_block_type { ME_TRANSPARENT = 0, ME_OPAQUE = 1, ME_BOUNDARY = 2 } me_block_type;

/* me::BoundaryTemporal (estimators.hpp:82). */
typedef enum me_boundary_temporal { ME_BT_TEXTURE = 0, ME_BT_SHAPE = 1 } me_boundary_temporal;

/* SearchConfig + PrsConfig + EstimateOptions::boundary_temporal (estimators.hpp:34-50,96-99). */
typedef struct me_config {
    int32_t algo;              /* me_algo */
    int32_t search_range;      /* S, pels (default 7) */
    int32_t block_size;        /* 8 or 16 */
    int32_t ref_distance;      /* frames between current and reference (default 2) */
    int32_t halfpel;           /* 1 => PRS step forced to 1 (estimators.cpp:405-406) */
    int32_t max_iterations;    /* PRS cap (default 4) */
    int32_t step;              /* PRS grid step in half-pels: 2 or 1 */
    int32_t boundary_temporal; /* me_boundary_temporal */
    double epsilon;            /* PRS convergence factor (default 0.5) */
    double theta;              /* PRS gradient gate (default 2.0) */
} me_config;

/* Per-block result record (16 bytes).  `cost_q4` is 4x the texture SAD at the
 * returned vector (exact for half-pel vectors, whose SAD is a multiple of 1/4):
 * for ES/TSS/FSS/DS the winner's SAD, for PA the PRS final center cost
 * (descent_log.back(), estimators.cpp:379).  Transparent blocks are all zero
 * apart from `type`. */
typedef struct me_block_rec {
    int16_t dx, dy;          /* half-pel vector (MotionField::vectors) */
    uint32_t cost_q4;        /* 4 x SAD at (dx, dy) */
    uint16_t comparisons;    /* this block's share of SearchStats::block_comparisons (saturates at 65535) */
    uint16_t dpd_steps;      /* this block's share of SearchStats::dpd_refinement_steps */
    uint8_t iterations;      /* PRS recenters (descent_log size - 1); 0 for the baselines */
    uint8_t type;            /* me_block_type (MotionField::types) */
    uint16_t reserved;
} me_block_rec;

/* SearchStats (metrics.hpp:40-62) for one frame pair, plus the int64 luma SSE
 * of the motion-compensated prediction (psnr, metrics.cpp:108-124, before the
 * host-side division and log10). */
typedef struct me_pair_stats {
    int64_t block_comparisons;
    int64_t dpd_refinement_steps;
    int64_t blocks_opaque;
    int64_t blocks_boundary;
    int64_t blocks_transparent;
    int64_t sse;
} me_pair_stats;

/* Opaque per-thread context: device, stream, and a cache of device scratch
 * buffers (the reference is re-entrant; one context per host
 * thread keeps that property). */
typedef struct me_ctx me_ctx;

const char* me_b200_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* me_b200_last_error(void);
/* Number of usable sm_100 devices (0 on a machine without one). */
int me_b200_device_count(void);

me_status me_b200_ctx_create(int device, me_ctx** out);
void me_b200_ctx_destroy(me_ctx* ctx);
/* The cudaStream_t the host-pointer entry points of this context run on. */
void* me_b200_ctx_stream(me_ctx* ctx);

/* Per-kernel CUDA-event timing of the batched pipeline (off by default).
 * When enabled, every run records events on its stream around each stage;
 * me_b200_ctx_stage_ms waits for the last run and writes the stage durations
 * (ms) in the order ME_STAGE_* into out[n] (n <= ME_NUM_STAGES). */
enum { ME_STAGE_CLASSIFY = 0, ME_STAGE_SORT = 1, ME_STAGE_SEARCH = 2, ME_STAGE_MC_PSNR = 3, ME_NUM_STAGES = 4 };
me_status me_b200_ctx_set_profiling(me_ctx* ctx, int enable);

/* Kernel-schedule tuning of a context (defaults = the measured best; the
 * library reads no environment variables).  Every field's 0 selects the
 * default.  Results never depend on these: every schedule is bit-exact
 * (tests/test_gpu_parity.py runs them all). */
enum {
    ME_PA_SCHED_AUTO = 0,       /* by wavefront width: hybrid (quad middle) or fast */
    ME_PA_SCHED_GENERIC = 1,    /* pa_kernel: a warp per block, any configuration */
    ME_PA_SCHED_FAST = 2,       /* pa_fast_kernel over the whole list */
    ME_PA_SCHED_DUO = 3,        /* pa_duo_kernel (two blocks per warp) over the whole list */
    ME_PA_SCHED_DUO_HYBRID = 4, /* fast head/tail, duo middle */
    ME_PA_SCHED_QUAD_HYBRID = 5 /* fast head/tail, quad middle */
};
typedef struct me_tuning {
    int32_t pa_schedule;      /* ME_PA_SCHED_* */
    int32_t pa_wide_blocks;   /* hybrid: steps with at least this many blocks are "wide" (0: 40 x SMs) */
    int32_t pa_fast_ctas;     /* CTAs per SM of pa_fast_kernel, 1..6 (0: by wavefront width) */
    int32_t pa_quad_ctas;     /* CTAs per SM of pa_quad_kernel, 2..4 (0: 3) */
    int32_t pa_duo_threads;   /* 128 or 256 (0: 256) */
    int32_t pa_duo_ctas;      /* CTAs per SM of pa_duo_kernel (0: 4 at 256 threads, 7 at 128) */
    int32_t pa_poll_ns;       /* dependency poll back-off in ns (0: 16) */
    int32_t pa_static_claim;  /* 1: static round-robin work split (needs the whole grid resident);
                                 0: in-order CTA-batch claiming */
    int32_t pa_no_pdl;        /* 1: launch the hybrid's grids in plain stream order */
    int32_t pa_no_smem_pair;  /* 1: never use the one-CTA shared-memory kernel for a small pair */
    int32_t pa_fast_patches;  /* 1: pa_fast_kernel stages per-candidate patches after the dependency
                                 wait instead of the whole search window before it (S <= 32) */
    int32_t pa_key_a, pa_key_s; /* wavefront sort key a * (h + 2v + p) + s * seq (0: 1 and 0) */
    int32_t sort_no_pdl;      /* 1: scan and fill in plain stream order */
    int32_t fill_rows;        /* 1: a thread per block row, -1: a thread per block (0: by size) */
    int32_t fill_rows_per_cta;/* block rows per fill CTA (0: 64) */
    int32_t h2d_chunks;       /* host-buffer path: pipeline chunks, 1..32 (0: 16) */
    int32_t mask_pack;        /* host path alpha transfer: 1 bytes, 2 dense bits, 0/3 sparse bits */
    int32_t ring_ctas;        /* CTAs per SM of the TSS/FSS/DS kernel, 2..4 (0: 3) */
    int32_t host_threads;     /* host-buffer path: threads packing the masks (0: OpenMP default) */
    const char* pa_trace_path;/* debug: per-block PA trace written here (NULL: off; the context keeps a copy) */
    int32_t pa_key_plain;     /* 1: PA list keyed by the plain step t = h + 2v + p (with pa_key_a / pa_key_s);
                                 0: batches of <= 60000 blocks per step keyed by t - tmin(sequence), every
                                 sequence's wavefront starting at key 0 (wider batches: t);
                                 -1: t - tmin(sequence) at any width */
} me_tuning;
me_status me_b200_ctx_set_tuning(me_ctx* ctx, const me_tuning* tuning);
me_status me_b200_ctx_get_tuning(me_ctx* ctx, me_tuning* out);
me_status me_b200_ctx_stage_ms(me_ctx* ctx, float* out, int n);

/* Bytes the last me_b200_run_sequences call moved host->device and
 * device->host (binary alpha masks cross PCIe bit-packed: W*H/8 per frame). */
me_status me_b200_ctx_transfer_bytes(me_ctx* ctx, int64_t* h2d, int64_t* d2h);

/* Kernels the last batched call (me_b200_run_sequences[_dev], estimate_field)
 * launched: the stage kernels of every chunk (classify, scan, fill, the search
 * — three for the hybrid PA schedule — and the optional prediction pass) plus
 * the mask expansions of the host path. */
me_status me_b200_ctx_launches(me_ctx* ctx, int64_t* out);

/* The host path's transfer form of a binary alpha mask (n pixels, n % 64 ==
 * 0, every byte 0 or 255): G = ceil(n / 2048) groups of 32 64-pixel words;
 * uint32 presence[G] (bit i of group g: word 32g + i has a set pixel),
 * uint32 base[G] (index of the group's first stored word), zero padding to a
 * 16-byte boundary, then the stored (nonzero) words as uint64, bit i = pixel
 * i of the word.  *out_bytes receives the encoded size (<= 16 + n/256 + n/8);
 * ME_ERR_INVALID_ARGUMENT for a non-binary mask, n % 64 != 0 or a short
 * buffer.  Runs on the host cores (AVX-512BW when available). */
me_status me_b200_pack_mask(const uint8_t* mask, size_t n, uint8_t* out, size_t out_cap, size_t* out_bytes);

/* SearchConfig::validate + PrsConfig::validate (estimators.cpp:139-150). */
me_status me_b200_validate_config(const me_config* cfg);

/* ---------------------------------------------------------------------------
 * Batched sequence pipeline (the benchmark path).  Replaces the frame-pair
 * loop of run_experiment (bench.cpp:155-205) around estimate_field
 * (estimators.cpp:384-440), predict_frame (compensation.cpp:30-71) and psnr
 * (metrics.cpp:108-124): for each of n_seq sequences of n_frames frames, every
 * pair tau = ref_distance .. n_frames-1 (cur = frame tau, ref = frame
 * tau - ref_distance) is estimated; PA threads pair tau-1's field into pair
 * tau's temporal candidates (bench.cpp:204).
 *   luma   [n_seq][n_frames][height][width]
 *   alpha  [n_seq][n_frames][height][width] or NULL (no masks: all opaque)
 *   recs   [n_seq][pairs][rows][cols]       pairs = n_frames - ref_distance
 *   stats  [n_seq][pairs]
 *   pred   [n_seq][pairs][height][width] or NULL (prediction not stored; the
 *          SSE is computed either way)
 * Device pointers; enqueued on `stream` (a cudaStream_t; NULL is the CUDA
 * default stream, me_b200_ctx_stream gives the context's own), not
 * synchronised.  Calls on one context share its scratch: do not run two of
 * them concurrently on different streams.
 * ------------------------------------------------------------------------- */
me_status me_b200_run_sequences_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                                    int width, int height, const uint8_t* luma,
                                    const uint8_t* alpha, me_block_rec* recs,
                                    me_pair_stats* stats, uint8_t* pred, void* stream);

/* Same, with BINARY masks bit-packed in device memory: alpha_bits is
 * [n_seq][n_frames][height][width / 8] bytes, bit i of byte j = pel 8j + i,
 * set = inside (me_b200_pack_mask_dev makes it; 8-byte aligned).  1/8 of the
 * mask bytes in HBM; block classes come from the bits and boundary blocks'
 * shape SADs are popc(XOR) of bit rows (metrics.cpp:65-84 is a mismatch count,
 * which for 0/255 masks is the XOR count).  Results equal
 * me_b200_run_sequences_dev on the 0/255 byte masks. */
me_status me_b200_run_sequences_bits_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                                         int width, int height, const uint8_t* luma,
                                         const uint8_t* alpha_bits, me_block_rec* recs,
                                         me_pair_stats* stats, uint8_t* pred, void* stream);

/* Packs n device mask bytes (n % 64 == 0) into the bit plane above and sets
 * *binary (host) to 1 when every byte was 0 or 255 (the bit form is then
 * exact), else 0.  Synchronous on `stream`. */
me_status me_b200_pack_mask_dev(me_ctx* ctx, const uint8_t* alpha, size_t n, uint8_t* bits, int* binary,
                                void* stream);

/* One sequence (n_frames frames, device pointers) whose first pair takes its
 * temporal candidates from prev_mv — the previous pair's field as
 * [rows*cols][2] int32 (dx, dy) on the device, or NULL — exactly as
 * estimate_field's `prev` (estimators.cpp:384-440, bench.cpp:204): the unit of
 * chunked streaming, where chunk k's frames [s, s + n + d) continue chunk k-1
 * (PA only uses prev_mv).  prev_integer = 1 declares every prev vector
 * integer-pel (it is, for fields of an integer-pel search), which lets the
 * fast PA kernels take it. */
me_status me_b200_run_sequence_prev_dev(me_ctx* ctx, const me_config* cfg, int n_frames, int width,
                                        int height, const uint8_t* luma, const uint8_t* alpha,
                                        const int32_t* prev_mv, int prev_integer, me_block_rec* recs,
                                        me_pair_stats* stats, void* stream);

/* A block-row band [row0, row1) of the same batch (baselines ES/TSS/FSS/DS
 * only; PA blocks depend on the rows above -> ME_ERR_INVALID_ARGUMENT): the
 * unit of the row sharding across GPUs.  Records of the band's
 * blocks are written (the others are left untouched); stats are the band's
 * share of each pair's SearchStats + SSE, so the bands' stats of a pair sum
 * to the whole pair's.  Device pointers, enqueued on `stream`. */
me_status me_b200_run_band_dev(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                               int width, int height, const uint8_t* luma, const uint8_t* alpha,
                               int row0, int row1, me_block_rec* recs, me_pair_stats* stats,
                               void* stream);

/* The batch of me_b200_run_sequences over devices 0..n_gpus-1 of this
 * process (the reference's run_experiment pair loop, bench.cpp:155-205,
 * sharded): sequences split contiguously over the devices (a single
 * baseline sequence: its frame pairs), each shard end to end on its own host
 * thread and context, results written straight into the host arrays.  HOST
 * buffers; synchronous. */
me_status me_b200_run_sequences_multi(const me_config* cfg, int n_seq, int n_frames, int width,
                                      int height, const uint8_t* luma, const uint8_t* alpha,
                                      me_block_rec* recs, me_pair_stats* stats, int n_gpus);

/* Same, end to end from HOST buffers: H2D of the inputs, the device pipeline,
 * D2H of the records and stats (and pred when non-NULL), synchronous. */
me_status me_b200_run_sequences(me_ctx* ctx, const me_config* cfg, int n_seq, int n_frames,
                                int width, int height, const uint8_t* luma, const uint8_t* alpha,
                                me_block_rec* recs, me_pair_stats* stats, uint8_t* pred);

/* ---------------------------------------------------------------------------
 * Single frame pair: me::estimate_field (estimators.hpp:160-165,
 * estimators.cpp:384-440).  prev_mv is the previous field's vectors as
 * [rows*cols][2] int32 (dx, dy) or NULL; prev_cols/prev_rows must equal the
 * grid (ME_ERR_INVALID_ARGUMENT otherwise, estimators.cpp:401-403).  cur_alpha
 * / ref_alpha may be NULL (no mask).  Host pointers.
 * ------------------------------------------------------------------------- */
me_status me_b200_estimate_field(me_ctx* ctx, const me_config* cfg, int width, int height,
                                 const uint8_t* cur, const uint8_t* ref, const uint8_t* cur_alpha,
                                 const uint8_t* ref_alpha, const int32_t* prev_mv, int prev_cols,
                                 int prev_rows, me_block_rec* recs, me_pair_stats* stats);

/* ---------------------------------------------------------------------------
 * Per-block entry points (host pointers; one block per call).
 * ------------------------------------------------------------------------- */

/* full_search / tss_search / fss_search / ds_search (estimators.hpp:113-120,
 * estimators.cpp:167-236), selected by `algo` (ME_ALGO_ES..ME_ALGO_DS).
 * out_mv = (dx, dy) half-pel; *out_comparisons = unique evaluations added to
 * SearchStats::block_comparisons; *out_cost_q4 = 4 x SAD at the winner. */
me_status me_b200_block_search(me_ctx* ctx, int algo, int width, int height, const uint8_t* cur,
                               const uint8_t* ref, int x0, int y0, int size, int search_range,
                               int32_t out_mv[2], int64_t* out_comparisons, uint32_t* out_cost_q4);

/* brs_select (estimators.hpp:131-135, estimators.cpp:257-301).  cands =
 * {a.dx, a.dy, b.dx, b.dy, c.dx, c.dy, t.dx, t.dy}.  out_kinds[4] receives the
 * ScoreKind of each candidate (0 texture, 1 shape; the scoring_log payload),
 * out_scores_q4[4] 4 x each candidate's score.  Always 4 comparisons. */
me_status me_b200_brs_select(me_ctx* ctx, int width, int height, const uint8_t* cur,
                             const uint8_t* ref, const uint8_t* cur_alpha, const uint8_t* ref_alpha,
                             int x0, int y0, int size, int btype, const int32_t cands[8],
                             int search_range, int boundary_temporal, int32_t out_mv[2],
                             uint8_t out_kinds[4], uint32_t out_scores_q4[4]);

/* prs_refine (estimators.hpp:156-158, estimators.cpp:311-382).  descent_log
 * (capacity max_iterations + 1, may be NULL) receives 4 x the cost of every
 * accepted center; *log_len its length.  *out_dpd_steps = unique aggregate
 * evaluations. */
me_status me_b200_prs_refine(me_ctx* ctx, int width, int height, const uint8_t* cur,
                             const uint8_t* ref, int x0, int y0, int size, const int32_t d0[2],
                             int search_range, double epsilon, double theta, int max_iterations,
                             int step, int32_t out_mv[2], int64_t* out_dpd_steps,
                             uint32_t* descent_log_q4, int* log_len);

/* prs_update (estimators.hpp:144-145, estimators.cpp:303-309): the per-pixel
 * update d_i - eps * dpd * (u_x, u_y) in pels (out[0] = x, out[1] = y). */
me_status me_b200_prs_update(me_ctx* ctx, int width, int height, const uint8_t* cur,
                             const uint8_t* ref, int x, int y, const int32_t d[2], double epsilon,
                             double theta, double out[2]);

/* sad_texture (metrics.hpp:57, metrics.cpp:43-63), 4 x SAD, any vector
 * (edge-replicated reads, half-pel bilinear). */
me_status me_b200_sad_texture(me_ctx* ctx, int width, int height, const uint8_t* cur,
                              const uint8_t* ref, int x0, int y0, int size, int dx, int dy,
                              uint32_t* out_sad_q4);

/* sad_shape (metrics.hpp:61-62, metrics.cpp:65-84): 255 x mismatches.
 * Half-pel vectors are rejected with ME_ERR_INVALID_ARGUMENT. */
me_status me_b200_sad_shape(me_ctx* ctx, int width, int height, const uint8_t* cur_alpha,
                            const uint8_t* ref_alpha, int x0, int y0, int size, int dx, int dy,
                            int64_t* out_sad);

/* classify_block over the whole raster grid (frame.cpp:81-104 via
 * estimators.cpp:410-412): types[rows*cols]; alpha NULL => all opaque. */
me_status me_b200_classify_blocks(me_ctx* ctx, int width, int height, const uint8_t* alpha,
                                  int block_size, uint8_t* types);

/* binarize (frame.hpp:105, frame.cpp:50-56): out = gray >= threshold ? 255 : 0. */
me_status me_b200_binarize(me_ctx* ctx, int width, int height, const uint8_t* gray, int threshold,
                           uint8_t* out);

/* predict_frame (compensation.hpp:44, compensation.cpp:30-71): luma only.
 * mv = [rows*cols][2] int32, types = [rows*cols] (NULL => all opaque).  When
 * `cur` is non-NULL *out_sse receives the int64 SSE of cur vs the prediction
 * (the psnr numerator, metrics.cpp:108-124); pred may be NULL. */
me_status me_b200_predict_frame(me_ctx* ctx, int width, int height, const uint8_t* ref,
                                const int32_t* mv, const uint8_t* types, int block_size,
                                const uint8_t* cur, uint8_t* pred, int64_t* out_sse);

/* psnr numerator (metrics.cpp:108-124): int64 sum of squared luma differences. */
me_status me_b200_sse(me_ctx* ctx, int width, int height, const uint8_t* a, const uint8_t* b,
                      int64_t* out_sse);

/* The INT-pipe roofline denominator of the SAD kernels, measured on ctx's
 * device now: VABSDIFF4.U8.ACC byte-ops per second of independent chains at
 * full occupancy (best of 10 launches, CUDA events). */
me_status me_b200_probe_int_peak(me_ctx* ctx, double* byte_ops_per_s);

/* ---------------------------------------------------------------------------
 * Deterministic synthetic sequences (host code, integer-only so
 * every consumer sees identical bytes).  Not part of the reference API.
 * ------------------------------------------------------------------------- */
typedef struct me_synth_params {
    int32_t width, height, frames;
    uint64_t seed;
    int32_t blur_sigma_q8;       /* background/object blur sigma x 256 (1.5 -> 384) */
    int32_t bg_jitter;           /* >0: per-frame global shift drawn in [-j, j]^2 */
    int32_t bg_drift_q8[2];      /* else: global drift per frame, pels x 256 (rounded) */
    int32_t n_objects;
    int32_t obj_min, obj_max;    /* random object box size range (pels) when no fixed sizes */
    int32_t obj_w[4], obj_h[4];  /* fixed ellipse semi-axes for the first objects (0 = random) */
    int32_t obj_v[4][2];         /* fixed velocities (used when vel_fixed) */
    int32_t vel_fixed;           /* 1: obj_v for the fixed objects */
    int32_t vmax;                /* random integer velocities in [-vmax, vmax] */
    int32_t shapes;              /* 0 ellipses only, 1 ellipse/rectangle mix */
    int32_t noise_sigma_q8;      /* additive Gaussian noise sigma x 256 (0 = none) */
} me_synth_params;

/* Presets for BASELINE.json configs 1..5 (seed as given). */
me_status me_b200_synth_preset(int config_id, uint64_t seed, me_synth_params* out);
/* luma/alpha: [frames][height][width] each (alpha = union of object masks). */
me_status me_b200_synth(const me_synth_params* p, uint8_t* luma, uint8_t* alpha);
/* The same generator on the device for a batch of n_seq sequences (one params
 * entry per sequence, equal geometry; config 4 uses seed = base + i): luma and
 * alpha (nullable) are DEVICE buffers [n_seq][frames][height][width], written
 * on `stream` (NULL = default stream); byte-identical to me_b200_synth.
 * Returns after the stream has finished the batch. */
me_status me_b200_synth_dev(me_ctx* ctx, const me_synth_params* params, int n_seq, uint8_t* luma,
                            uint8_t* alpha, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ME_B200_H */
