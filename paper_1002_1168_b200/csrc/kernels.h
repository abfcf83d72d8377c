// kernels.h — host-side launchers of the sm_100a kernels (wavefront.cu, es.cu,
// ring.cu, pa.cu, frame_ops.cu; the pipeline in batch.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "me_b200.h"
#include <nvtx3/nvToolsExt.h>

namespace mek {

// NVTX range over a scope (host timeline: the pipeline's stages and the C ABI
// calls show up in Nsight Systems; no cost without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Geometry of a batch: n_seq sequences x n_frames frames of W x H luma; pairs
// tau = d .. F-1 (pair index p = tau - d, cur = frame p + d, ref = frame p).
struct Batch {
    const uint8_t* luma;   // [n_seq][F][H][W]
    const uint8_t* alpha;  // same shape, or null (all opaque)
    // binary masks bit-packed instead ([n_seq][F][H][W / 8], bit i of byte j =
    // pel 8j + i, set = inside): classify and the fast/quad PA kernels score
    // shapes with popc(XOR) on these (alpha is null then)
    const uint8_t* alpha_bits = nullptr;
    int n_seq, F, W, H, d, pairs, bs, cols, rows;
    // block-row band [v0, v1) of the baselines' row sharding (v1 < 0: every
    // row): blocks outside it are not estimated, their records are left
    // untouched and they add nothing to the pair's stats
    int v0 = 0, v1 = -1;
    __host__ __device__ bool in_band(int v) const { return v >= v0 && (v1 < 0 || v < v1); }
    __host__ __device__ int64_t nblocks() const { return int64_t(n_seq) * pairs * rows * cols; }
    __host__ __device__ int steps() const { return (cols - 1) + 2 * (rows - 1) + (pairs - 1) + 1; }
};

// Kernel-schedule tuning with the defaults applied (from a context's
// me_tuning, include/me_b200.h; the defaults are the measured best).
struct Tuning {
    int pa_schedule = ME_PA_SCHED_AUTO;
    int pa_wide_blocks = 0;  // 0: 40 x SMs
    int pa_fast_ctas = 0;    // 0: by wavefront width
    int pa_quad_ctas = 3;
    int pa_duo_threads = 256;
    int pa_duo_ctas = 0;     // 0: 4 (256 threads) or 7 (128)
    int pa_poll_ns = 16;
    bool pa_claim = true;    // in-order CTA-batch claiming
    bool pa_pdl = true;
    bool pa_smem_pair = true;
    bool pa_fast_window = true;  // pa_fast_kernel stages the whole search window at claim time (S <= 32)
    int key_a = 1, key_s = 0;
    bool key_align = true;   // PA batches: key = t - tmin[seq] (sequences' wavefronts aligned at their first estimated block)
    int key_align_max_blocks_per_step = 60000;  // ... up to this many blocks per lockstep step (-1: any)
    bool sort_pdl = true;
    int fill_rows = 0;       // 1 a thread per row, -1 a thread per block, 0 by size
    int fill_rows_per_cta = 64;
    int h2d_chunks = 16;
    int mask_pack = 3;       // 1 bytes, 2 dense bits, 3 sparse bits
    int ring_ctas = 3;       // CTAs per SM of ring_kernel (3: 80 registers, no spills)
    int host_threads = 0;    // host-path mask packing threads (0: OpenMP default)
    const char* pa_trace = nullptr;
};
Tuning resolve_tuning(const me_tuning* t);

// Scratch needed by run_batch (bytes), given the step-bin count.
size_t scratch_bytes(const Batch& b, int algo, const Tuning& t);

// Full device pipeline: classify -> (ES | rings | PA wavefront) -> MC + PSNR.
// `prev0` (nullable, [rows*cols][2] int32) supplies pair 0's temporal
// candidates (estimate_field's prev_field); stats must hold n_seq*pairs
// entries; pred is nullable.
// `events` (nullable) = 5 events recorded before classify, before the sort,
// before the search, before MC+PSNR and at the end.
// `prev0_integer`: every prev0 vector is integer-pel (even), which lets the
// fast PA kernels take it.
// `launches` (nullable) receives the number of kernels launched.
cudaError_t run_batch(const Batch& b, const me_config& cfg, const int32_t* prev0,
                      me_block_rec* recs, me_pair_stats* stats, uint8_t* pred, void* scratch,
                      size_t scratch_size, int num_sms, cudaStream_t st, const Tuning& tune,
                      cudaEvent_t* events = nullptr, bool prev0_integer = false, int* launches = nullptr);

// Single-block entry points (all pointers device pointers; outputs in `out`,
// an int64 array whose layout is documented at each launcher).
cudaError_t block_search(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H, int x0,
                         int y0, int size, int range, int64_t* out, cudaStream_t st);
cudaError_t brs_single(const uint8_t* cur, const uint8_t* ref, const uint8_t* ca,
                       const uint8_t* ra, int W, int H, int x0, int y0, int size, int btype,
                       const int32_t* cands_dev, int range, int boundary_temporal, int64_t* out,
                       cudaStream_t st);
cudaError_t prs_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                       int size, int d0x, int d0y, int range, double eps, double theta,
                       int max_iter, int step, int64_t* out, cudaStream_t st);
cudaError_t prs_update_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x, int y,
                              int dx, int dy, double eps, double theta, double* out, cudaStream_t st);
cudaError_t sad_texture_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                               int size, int dx, int dy, int64_t* out, cudaStream_t st);
cudaError_t sad_shape_single(const uint8_t* ca, const uint8_t* ra, int W, int H, int x0, int y0,
                             int size, int dx, int dy, int64_t* out, cudaStream_t st);
cudaError_t classify_frame(const uint8_t* alpha, int W, int H, int bs, uint8_t* types,
                           cudaStream_t st);
cudaError_t binarize(const uint8_t* gray, int n, int threshold, uint8_t* out, cudaStream_t st);
// Expands a bit-packed binary mask (bit i of byte j = pixel 8j + i) to bytes
// 0 / 255; n (pixels) is a multiple of 8.
cudaError_t unpack_mask(const uint8_t* bits, uint8_t* out, size_t n, cudaStream_t st);
// Sparse form of the same mask (n % 64 == 0): uint32 presence[G] (bit i of
// group g: 64-pixel word 32g + i is nonzero), uint32 base[G] (index of the
// group's first literal), then at sparse_mask_header_bytes(n) the nonzero
// words (uint64, bit i = pixel i); G = ceil(n / 64 / 32).
inline size_t sparse_mask_header_bytes(size_t n) { return ((n / 64 + 31) / 32 * 8 + 15) & ~size_t(15); }
cudaError_t unpack_mask_sparse(const uint8_t* packed, uint8_t* out, size_t n, cudaStream_t st);
// Device bytes -> dense bit plane (n % 64 == 0); *nonbinary (device int,
// zeroed by the caller) counts 64-pixel words with bytes other than 0 / 255.
cudaError_t pack_mask_dev(const uint8_t* alpha, size_t n, uint8_t* bits, int* nonbinary, cudaStream_t st);
// ... or to the dense bit plane (n / 8 bytes, the layout Batch::alpha_bits reads).
cudaError_t unpack_mask_sparse_bits(const uint8_t* packed, uint8_t* out_bits, size_t n, cudaStream_t st);
// PA on bit-packed masks: true when the batch's kernel schedule reads them
// (pa_fast_kernel / the quad hybrid); otherwise they are expanded to bytes.
bool pa_takes_bits(const Batch& b, const me_config& cfg, int num_sms, const Tuning& t);
cudaError_t predict(const uint8_t* ref, const uint8_t* cur, const int32_t* mv, const uint8_t* types,
                    int W, int H, int bs, uint8_t* pred, me_pair_stats* stats,
                    cudaStream_t st);
cudaError_t sse(const uint8_t* a, const uint8_t* b, int n, unsigned long long* out,
                cudaStream_t st);

}  // namespace mek
