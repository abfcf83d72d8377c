// stages.h — internal interface between the pipeline driver (batch.cu) and
// the kernel translation units (wavefront.cu, es.cu, ring.cu, pa.cu,
// frame_ops.cu).  Not installed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace mek {

// Each bin is padded to a multiple of `pad` entries (invalid markers), so a
// warp that claims `pad` aligned entries never straddles two bins.
constexpr uint32_t kInvalidEntry = 0xFFFFFFFFu;

// one 128-byte line per bin cursor: the fill's per-(CTA, bin) atomics would
// otherwise queue on a handful of L2 lines
constexpr int kCursorStride = 32;

struct ClassArgs {
    Batch b;
    int pa;              // key = wavefront step when 1
    me_block_rec* recs;  // [n_seq][pairs][rows][cols]
    uint8_t* types;      // same indexing
    int* hist;           // [nbins]
    int nbins;
    me_pair_stats* stats;  // [n_seq][pairs]: transparent blocks' count and SSE
    int key_a, key_s;      // PA: key = key_a * (h + 2v + p) + key_s * seq (sequence stagger)
    // PA, aligned keys (key = t - tmin[seq], tmin = the sequence's first step
    // holding an estimated block): classify counts estimated blocks per
    // (sequence, step) into hist2 [n_seq][steps]; the scan derives tmin and the
    // key histogram; the fill reads tmin.  Null: the key_a / key_s key.
    int* hist2;
    const int* tmin;  // fill: the keys' offsets (written by the scan)
    int* tmin_g;      // classify: atomicMin target (the same array, preset to 0x7F7F7F7F)
    // single-bin searches (ES, TSS, FSS, DS): classify appends the estimated
    // blocks' entries to the list itself (warp-aggregated, any order) and counts
    // them in *nlist_direct — no scan / fill.  Null: the sorted list.
    uint2* list_direct;
    int* nlist_direct;
    // ... as runs of 1, 2 or 4 horizontally adjacent estimated blocks (16x16
    // ES at the largest ranges, es_run_kernel): entry {h | count << 12 | v << 16, p | seq << 16}
    int es_runs;
};

// wavefront.cu: classify -> per-step histogram -> scan -> fill (the sorted list)
cudaError_t launch_classify(const ClassArgs& ca, int num_sms, cudaStream_t st);
// (pdl: scan, fill and the PA head chained by programmatic dependent launch)
// (hist2 / tmin non-null: aligned keys, hist2 [n_seq][nbins] is reduced into the key histogram
// with tmin [n_seq] from classify (0x7F7F7F7F for a sequence without estimated blocks: 0 is
// written back); hist is then unused)
cudaError_t launch_scan(const int* hist, int nbins, int pad, int* offs, int* cursor, uint2* list,
                        int wide, int* ranges, cudaStream_t st, bool pdl, const int* hist2 = nullptr,
                        int n_seq = 0, int* tmin = nullptr);
cudaError_t launch_fill(const ClassArgs& ca, int* cursor, uint2* list, int num_sms, cudaStream_t st,
                        const Tuning& t);

// es.cu: full search over the list; single-block full search
cudaError_t launch_es(const Batch& b, int S, const uint2* list, const int* nlist, int* counter,
                      me_block_rec* recs, me_pair_stats* stats, int num_sms, cudaStream_t st,
                      const uint8_t* types = nullptr);
// ES on 16x16 blocks at S > 32 takes runs of adjacent blocks (classify emits
// them when ClassArgs::es_runs is set; es_run_kernel shares their windows)
bool es_use_runs(const Batch& b, int S);
cudaError_t launch_es_single(const uint8_t* cur, const uint8_t* ref, int W, int H, int x0, int y0,
                             int size, int range, int64_t* out, cudaStream_t st);

// ring.cu: TSS / FSS / DS over the list; single-block ring search
cudaError_t launch_ring(const Batch& b, int algo, int S, const uint2* list, const int* nlist,
                        me_block_rec* recs, me_pair_stats* stats, int num_sms, cudaStream_t st, int ctas);
cudaError_t launch_ring_single(int algo, const uint8_t* cur, const uint8_t* ref, int W, int H,
                               int x0, int y0, int size, int range, int64_t* out, cudaStream_t st);

// pa.cu: the proposed algorithm's wavefront (kernel choice, list ranges)
int pa_wide_threshold(int num_sms, const Tuning& t);
int pa_kernel_mode(const Batch& b, const me_config& cfg, const int32_t* prev0, bool prev0_integer,
                   int num_sms, const Tuning& t);
cudaError_t launch_pa_smem(const Batch& b, const me_config& cfg, const int32_t* prev0, bool prev0_integer,
                           me_block_rec* recs, me_pair_stats* stats, cudaStream_t st, const Tuning& t);
// claims: 3 zeroed counters (in-order dynamic claiming, one per launch) or null
cudaError_t launch_pa(const Batch& b, const me_config& cfg, const int32_t* prev0, const uint2* list,
                      const int* nlist, const int* ranges, int pa_mode, me_block_rec* recs,
                      me_pair_stats* stats, int num_sms, cudaStream_t st, int* claims, const Tuning& t);

// frame_ops.cu: the prediction pass of a batch (only when asked for)
cudaError_t launch_mc_pred(const Batch& b, const me_block_rec* recs, uint8_t* pred, cudaStream_t st);

}  // namespace mek
