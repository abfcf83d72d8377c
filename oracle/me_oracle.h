/*
 * oracle/me_oracle.h — TEST INFRASTRUCTURE: the CPU restatement of the
 * reference's motion-estimation hot path (/root/reference/proj/src), used only
 * as the checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Never linked into or called by the product library.
 *
 * Parity pin: every function is checked bit-for-bit against the reference
 * itself (oracle/_ref/libme_ref.so, compiled from the unmodified reference
 * sources) and against tests/golden/ fixtures made from it
 * (tests/test_oracle_pin.py).
 */
#ifndef ME_ORACLE_H
#define ME_ORACLE_H

#include <stdint.h>

#include "me_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

void orc_binarize(int w, int h, const uint8_t* gray, int threshold, uint8_t* out);
int orc_classify(int w, int h, const uint8_t* alpha, int size, uint8_t* types);
double orc_sad_texture(int w, int h, const uint8_t* cur, const uint8_t* ref, int x0, int y0,
                       int size, int dx, int dy);
int orc_sad_shape(int w, int h, const uint8_t* ca, const uint8_t* ra, int x0, int y0, int size,
                  int dx, int dy, int64_t* out);
void orc_clip_to_window(int dx, int dy, int x0, int y0, int size, int w, int h, int range,
                        int32_t* out);
int orc_block_search(int algo, int w, int h, const uint8_t* cur, const uint8_t* ref, int x0,
                     int y0, int size, int range, int32_t* mv, int64_t* cmp, uint32_t* cost_q4);
int orc_brs_select(int w, int h, const uint8_t* cur, const uint8_t* ref, const uint8_t* ca,
                   const uint8_t* ra, int x0, int y0, int size, int btype, const int32_t* cands,
                   int range, int boundary_temporal, int32_t* mv, uint8_t* kinds,
                   uint32_t* scores_q4);
void orc_prs_update(int w, int h, const uint8_t* cur, const uint8_t* ref, int x, int y,
                    const int32_t* d, double eps, double theta, double* out);
int orc_prs_refine(int w, int h, const uint8_t* cur, const uint8_t* ref, int x0, int y0,
                   int size, const int32_t* d0, int range, double eps, double theta, int max_iter,
                   int step, int32_t* mv, int64_t* dpd, uint32_t* log_q4, int* log_len);
int orc_estimate_field(const me_config* c, int w, int h, const uint8_t* cur, const uint8_t* ref,
                       const uint8_t* ca, const uint8_t* ra, const int32_t* prev_mv,
                       int prev_cols, int prev_rows, me_block_rec* recs, me_pair_stats* st);
int orc_predict_frame(int w, int h, const uint8_t* ref, const int32_t* mv, const uint8_t* types,
                      int bs, uint8_t* pred);
int64_t orc_sse(int w, int h, const uint8_t* a, const uint8_t* b);
void orc_psnr_from_sse(int64_t sse, int64_t n, double* mse, double* db, double* linear,
                       int* infinite);
int orc_run_sequence(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                     const uint8_t* alpha, me_block_rec* recs, me_pair_stats* stats,
                     uint8_t* pred);
/* n_seq sequences on `threads` host threads (one sequence per thread at a time). */
int orc_run_sequences_threaded(const me_config* c, int n_seq, int n_frames, int w, int h,
                               const uint8_t* luma, const uint8_t* alpha, me_block_rec* recs,
                               me_pair_stats* stats, int threads);
/* One pair of a sequence, independent of the others (ES/TSS/FSS/DS units). */
int orc_run_pairs_threaded(const me_config* c, int n_frames, int w, int h, const uint8_t* luma,
                           const uint8_t* alpha, int first_pair, int n_pairs, me_block_rec* recs,
                           me_pair_stats* stats, int threads);
/* ES/ring search on an explicit list of blocks (bounded CPU samples). */
int orc_search_blocks(const me_config* c, int w, int h, const uint8_t* cur, const uint8_t* ref,
                      const int32_t* block_xy, int n_blocks, int threads, int32_t* mv_out,
                      int64_t* cmp_out);

#ifdef __cplusplus
}
#endif

#endif
