/*
 * tensorbleu.h — C ABI of the B200-native TensorBLEU hot path.
 *
 * Drop-in boundary for the reference package `batchbleu` (/root/reference/pkg).
 * The reference has no C ABI of its own: its operator/plugin surface is the
 * Python module `batchbleu._backend` (pkg/src/batchbleu/_backend.py:45-54)
 * dispatching to the Cython kernels in pkg/src/batchbleu/_kernels.pyx, and its
 * public entry points are `compute_stats` / `sentence_bleu` / `corpus_bleu`
 * (pkg/src/batchbleu/bleu.py:173-305).  Each function below names the
 * reference interface it replaces.  INTEGRATION.md shows the ctypes binding a
 * maintainer of the reference would add.
 *
 * Conventions
 *  - Every pointer documented "device" is a CUDA device pointer on the current
 *    device; "host" pointers are read before the call returns.
 *  - All calls are stream-ordered and asynchronous on `stream` (a
 *    cudaStream_t, NULL = legacy default stream).  Nothing synchronises.
 *  - Errors that depend only on host arguments are returned immediately as a
 *    TB_ERR_* code.  Errors that depend on device data (a length outside
 *    [0, width], a negative token ID in a valid position, a compact ID outside
 *    [0, U)) are OR-ed into the device int32 `*err_flag` (TB_FLAG_* bits;
 *    see tb_bleu_stats for its corpus-mode exception); the caller reads it
 *    after synchronising and raises.
 *  - Token IDs are int32 or int64 (`token_bytes` = 4 or 8), row-major with a
 *    leading dimension `ld` (elements).  Lengths are int64, as in
 *    `TokenBatch` (pkg/src/batchbleu/batch.py:22-37).
 *  - Integer statistics are int64; scores are fp64 (the reference epilogue
 *    is fp64 throughout, bleu.py:213-261).
 */
#ifndef TENSORBLEU_H
#define TENSORBLEU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define TB_OK 0
#define TB_ERR_INVALID_ARG 1  /* -> ValueError   (bleu.py:35-54, 97-105; ngrams.py:68-69) */
#define TB_ERR_CAPACITY 2     /* -> CapacityError (ngrams.py:23-27, 109-113)             */
#define TB_ERR_CUDA 3         /* -> RuntimeError                                          */
#define TB_ERR_UNSUPPORTED 4  /* -> ValueError   (limits of the device path, see below)   */
#define TB_ERR_WORKSPACE 5    /* -> RuntimeError (workspace smaller than *_workspace_bytes) */

/* ---- device-side error flag bits --------------------------------------- */
#define TB_FLAG_BAD_LENGTH 1   /* a length outside [0, width]   (batch.py:30-31)      */
#define TB_FLAG_NEGATIVE_ID 2  /* negative ID at a valid position (batch.py:32-34)    */
#define TB_FLAG_ID_RANGE 4     /* compact ID outside [0, U)  (_kernels.pyx:124-125)   */
#define TB_FLAG_SEGMENTS 8     /* segment lengths do not sum to the ID count (_kernels.pyx:96-97) */

/* ---- smoothing methods (bleu.py:15, 213-239) ----------------------------- */
#define TB_SMOOTH_NONE 0
#define TB_SMOOTH_FLOOR 1
#define TB_SMOOTH_ADD_K 2
#define TB_SMOOTH_EXP 3

/* Limits of the FUSED kernels (tb_bleu_stats / tb_bleu_host / tb_bleu_scores):
 * kernel-parameter array sizes.  Larger N or R are served by the n-gram
 * operator kernels below (tb_flatten_windows, tb_unique_rows,
 * tb_segment_bincount, tb_count_binary, tb_clipped_numerators) and
 * tb_bleu_scores_any / tb_bleu_totals, composed by the Python host
 * (paper_2510_05485_b200.bleu), so the public API has no limit. */
#define TB_MAX_ORDER 32
#define TB_MAX_REFS 32

/* Library identification. */
const char* tb_version(void);
/* Human-readable text for a TB_ERR_* code. */
const char* tb_strerror(int code);
/* Last CUDA error string recorded by a failing call on this thread. */
const char* tb_last_cuda_error(void);

/* ------------------------------------------------------------------------ *
 *  Fused hot path: batch -> per-sentence statistics (+ epilogue)            *
 * ------------------------------------------------------------------------ */

/* Workspace bytes `tb_bleu_stats` needs for this shape.  The first call on a
 * workspace needs it zero-filled; every call leaves it zero-filled again. */
size_t tb_bleu_workspace_bytes(int64_t batch, int32_t num_refs,
                               int64_t cand_width, const int64_t* ref_widths /* host (R,) */,
                               int32_t token_bytes, int32_t max_order);

/* Replaces `compute_stats` (bleu.py:173-210) — i.e. the whole counting engine
 * `_chunk_stats` -> `ngrams.packed_order_ids` -> `_backend.segment_bincount`
 * / `_backend.clipped_numerators` (bleu.py:117-159, ngrams.py:144-205,
 * _kernels.pyx:84-180) plus `_effective_ref_lens` (bleu.py:108-114) — fused
 * with the per-sentence epilogue `score_sentences_from_stats`
 * (bleu.py:274-279) and, optionally, the corpus aggregation
 * `score_corpus_from_stats` (bleu.py:293-305).
 *
 * One launch.  Per sentence group (candidate i and its R references) a CTA
 * stages the rows in shared memory with bulk-async (TMA) copies, builds a
 * per-group n-gram dictionary in shared memory (a Bloom filter + exact
 * matching of the survivors for unrelated text, a store-then-verify hash
 * table with exact key comparison otherwise), counts the reference n-grams
 * per reference, max-folds over references, min-clips the candidate counts,
 * and runs the fp64 epilogue.
 *
 *  cand_ids       device (B, cand_ld) int32|int64
 *  cand_len       device (B,) int64
 *  ref_ids        host (R,) array of device pointers, ref r is (B, ref_ld[r])
 *  ref_ld/ref_width host (R,)
 *  ref_len        host (R,) array of device (B,) int64 pointers
 *  weights        host (N,) normalised weights (BleuConfig.weights)
 *  num_out,den_out   device (B, N) int64            (SentenceStats.numerators/denominators)
 *  cand_len_out      device (B,) int64 or NULL      (SentenceStats.cand_lens)
 *  eff_ref_out       device (B,) int64 or NULL      (SentenceStats.eff_ref_lens)
 *  scores_out        device (B,) fp64 or NULL       (BleuResult.scores)       NULL -> no per-sentence epilogue
 *  precisions_out    device (B, N) fp64 or NULL     (BleuResult.precisions)
 *  bp_out            device (B,) fp64 or NULL       (BleuResult.brevity_penalty)
 *  totals_out        device (2N+2,) int64 or NULL   [sum num_n | sum den_n | sum c | sum r]
 *  corpus_out        device (N+2,) fp64 or NULL     [score, bp, precisions_n]  (corpus epilogue)
 *  err_flag          device int32.  Per-sentence launches OR TB_FLAG_* bits into
 *                    it (the caller zeroes it; it is sticky across launches);
 *                    launches with totals_out/corpus_out WRITE it (0 or bits).
 * num_out/den_out may be NULL when only scores or corpus outputs are wanted.
 */
int tb_bleu_stats(int32_t token_bytes,
                  const void* cand_ids, int64_t cand_ld, int64_t cand_width,
                  const int64_t* cand_len,
                  int32_t num_refs, const void* const* ref_ids,
                  const int64_t* ref_ld, const int64_t* ref_width,
                  const int64_t* const* ref_len,
                  int64_t batch, int32_t max_order,
                  int32_t smoothing, double eps, double k, const double* weights,
                  int64_t* num_out, int64_t* den_out,
                  int64_t* cand_len_out, int64_t* eff_ref_out,
                  double* scores_out, double* precisions_out, double* bp_out,
                  int64_t* totals_out, double* corpus_out,
                  int32_t* err_flag,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer form of tb_bleu_stats: the blocking call the reference's
 * `compute_stats` / `sentence_bleu` / `corpus_bleu` make on host arrays
 * (bleu.py:173-305; the buffer bindings _ext.pyx:87-110 call the same).
 * Same arguments and outputs as tb_bleu_stats, but
 *  - token and length arrays may be HOST memory, pinned (page-locked:
 *    cudaHostAlloc / torch pin_memory) or pageable, or device memory.  Pinned
 *    token rows are read by the kernel directly over PCIe — only the valid
 *    prefix of each row, overlapped with the counting — so there is no
 *    separate full-width H2D copy; when every token array is pageable, a pool
 *    of host threads copies the valid prefixes into library-owned pinned
 *    memory (int64 IDs narrowed to int32 when every valid ID fits, exactly as
 *    if the caller had passed int32) and the kernel reads those (batches of
 *    >= 1024 rows with per-sentence outputs in chunks: one launch per chunk,
 *    the copy of the next chunk overlapping the kernel on this one); other
 *    pageable rows (and every row when the shape needs the global-memory
 *    kernel) are copied whole to device staging first;
 *  - every non-NULL output is a HOST array; the kernel writes results into a
 *    pinned staging area that is copied out after the stream synchronises;
 *  - the workspace and staging buffers are owned by the library (cached per
 *    calling thread and device);
 *  - the call synchronises `stream` and returns the device-detected data
 *    errors in *flags_out (TB_FLAG_* bits, 0 = clean). */
int tb_bleu_host(int32_t token_bytes,
                 const void* cand_ids, int64_t cand_ld, int64_t cand_width,
                 const int64_t* cand_len,
                 int32_t num_refs, const void* const* ref_ids,
                 const int64_t* ref_ld, const int64_t* ref_width,
                 const int64_t* const* ref_len,
                 int64_t batch, int32_t max_order,
                 int32_t smoothing, double eps, double k, const double* weights,
                 int64_t* num_out, int64_t* den_out,
                 int64_t* cand_len_out, int64_t* eff_ref_out,
                 double* scores_out, double* precisions_out, double* bp_out,
                 int64_t* totals_out, double* corpus_out,
                 int32_t* flags_out, void* stream);

/* Replaces `apply_smoothing` + `_bp_vector` + `_geo_mean_scores`
 * (bleu.py:213-261) as used by `score_sentences_from_stats` (bleu.py:274-279).
 * With batch = 1 and pointers into a totals vector it is the corpus epilogue
 * of `score_corpus_from_stats` (bleu.py:301-305).  Any output may be NULL. */
int tb_bleu_scores(const int64_t* num, const int64_t* den,
                   const int64_t* cand_len, const int64_t* eff_ref,
                   int64_t batch, int32_t max_order,
                   int32_t smoothing, double eps, double k, const double* weights,
                   double* scores_out, double* precisions_out, double* bp_out,
                   void* stream);

/* tb_bleu_scores for ANY max_order (the reference caps neither N nor R;
 * bleu.py:24-56), with the normalised weights in DEVICE memory (N,) fp64.
 * fp32 = 0: fp64 in numpy's operation order (outputs double*); fp32 = 1: the
 * same operations in single precision, outputs float* (north_star: within
 * 1e-5 relative of the fp64 scores).  Any output may be NULL. */
int tb_bleu_scores_any(const int64_t* num, const int64_t* den,
                       const int64_t* cand_len, const int64_t* eff_ref,
                       int64_t batch, int32_t max_order,
                       int32_t smoothing, double eps, double k, const double* weights_dev,
                       int32_t fp32, void* scores_out, void* precisions_out, void* bp_out,
                       void* stream);

/* Corpus aggregation `score_corpus_from_stats` (bleu.py:295-300): column sums
 * of (B, N) num/den and (B,) lengths into totals (2N+2,) int64 (any N). */
int tb_bleu_totals(const int64_t* num, const int64_t* den,
                   const int64_t* cand_len, const int64_t* eff_ref,
                   int64_t batch, int32_t max_order, int64_t* totals_out,
                   void* stream);

/* `TokenBatch.__post_init__` validation (batch.py:22-37) for a device batch:
 * lengths in [0, width], valid IDs non-negative.  Sets TB_FLAG_BAD_LENGTH /
 * TB_FLAG_NEGATIVE_ID in *err_flag. */
int tb_validate_batch(int32_t token_bytes, const void* ids, int64_t ld, int64_t width,
                      const int64_t* lengths, int64_t batch, int32_t* err_flag,
                      void* stream);

/* The same validation for a HOST batch (numpy / torch CPU arrays), run on the
 * library's host threads — `TokenBatch.__post_init__` (batch.py:25-35) without
 * the per-element numpy masks.  Returns TB_FLAG_BAD_LENGTH when a length lies
 * outside [0, width] (checked first, as the reference does), else
 * TB_FLAG_NEGATIVE_ID when a valid position holds a negative ID, else 0;
 * -TB_ERR_* on an argument error.  Reads host memory only (no GPU needed). */
int tb_validate_host(int32_t token_bytes, const void* ids, int64_t ld, int64_t width,
                     const int64_t* lengths, int64_t batch);

/* ------------------------------------------------------------------------ *
 *  Reference operator/plugin surface (_backend.py:45-54) on the device      *
 * ------------------------------------------------------------------------ */

/* Workspace bytes for tb_flatten_windows over `batch` rows. */
size_t tb_windows_workspace_bytes(int64_t batch);

/* Replaces `extract_ngrams` + `flatten_valid` (ngrams.py:63-83): the valid
 * order-n windows of every row (row i contributes max(len_i - n + 1, 0),
 * lengths clamped to [0, width]) concatenated row-major into out (T, n)
 * int64, T written to *total_out (device).  `out` must hold the upper bound
 * batch * max(width - n + 1, 0) rows.  ids device (batch, ld) int32|int64;
 * lengths device (batch,) int64. */
int tb_flatten_windows(int32_t token_bytes, const void* ids, int64_t ld, int64_t width,
                       const int64_t* lengths, int64_t batch, int32_t n, int64_t* out,
                       int64_t* total_out, void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes for tb_unique_rows on t rows of n columns. */
size_t tb_unique_rows_workspace_bytes(int64_t t, int32_t n);

/* Replaces `_backend.unique_rows` (_backend.py:45-46; _kernels.pyx:36-81) and
 * the dictionary step of `build_dictionary` (ngrams.py:86-106).  Exact
 * deduplication of the rows of a (t, n) int64 matrix with a global-memory
 * hash table; dense IDs are assigned in FIRST-OCCURRENCE order (the SPEC
 * leaves the order implementation-defined, SPEC.md "Dictionary ordering").
 *  unique_out   device (t, n) int64 capacity; first U rows written
 *  inverse_out  device (t,) int64
 *  num_unique   device int64 scalar (U) */
int tb_unique_rows(const int64_t* rows, int64_t t, int32_t n,
                   int64_t* unique_out, int64_t* inverse_out, int64_t* num_unique,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes for tb_segment_bincount / tb_clipped_numerators. */
size_t tb_segment_workspace_bytes(int64_t b, int64_t num_unique);

/* Replaces `_backend.segment_bincount` (_backend.py:49-50; _kernels.pyx:84-126;
 * ngrams.py:116-120): counts[i, id] over the concatenated per-segment IDs.
 *  ids (num_ids,) int64, seg_lengths (b,) int64 — device; counts_out (b, u)
 *  int32 device (fully overwritten).  Returns TB_ERR_CAPACITY when b*u
 *  overflows int64 (ngrams.py:109-113). */
int tb_segment_bincount(const int64_t* ids, int64_t num_ids,
                        const int64_t* seg_lengths, int64_t b, int64_t num_unique,
                        int32_t* counts_out, int32_t* err_flag,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Replaces `_backend.clipped_numerators` (_backend.py:53-54;
 * _kernels.pyx:129-180; ngrams.py:201-205): per segment, the sum over IDs of
 * min(candidate count, ref_max[i, id]).  ref_max (b, u) int32 device;
 * num_out (b,) int64 device. */
int tb_clipped_numerators(const int64_t* ids, int64_t num_ids,
                          const int64_t* seg_lengths, int64_t b,
                          const int32_t* ref_max, int64_t num_unique,
                          int64_t* num_out, int32_t* err_flag,
                          void* workspace, size_t workspace_bytes, void* stream);

/* `max_reference_counts` / `clip_counts` (ngrams.py:208-227): elementwise
 * out = max(a, b) (op = 0) or min(a, b) (op = 1) over `count` int32 values.
 * `out` may alias `a`. */
int tb_count_binary(const int32_t* a, const int32_t* b, int32_t* out, int64_t count,
                    int32_t op, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TENSORBLEU_H */
