// tb_common.cuh — device-side pieces shared by the TensorBLEU kernels:
// kernel parameters, PTX helpers (mbarrier, bulk async copy, PDL), row
// staging, hashing, the fp64 epilogue, the completion protocol and the
// shared-memory table helpers of the pair / multi kernels.
//
// Sources of libtensorbleu_b200.so:
//   tb_common.cuh        this file
//   tb_launch.cuh        shape planning types + the launch helper
//   tb_kernel_sparse.cu  bleu_sparse_kernel (R <= 8: warp per group; dense groups listed)
//   tb_kernel_pair.cu    bleu_pair_kernel (R = 1, CTA per group; the listed dense groups)
//   tb_kernel_multi.cu   bleu_multi_kernel (2 <= R <= 8, CTA per group; the listed dense groups)
//   tb_kernel_group.cu   bleu_group_kernel (R > 8) and bleu_stats_kernel (global memory)
//   tb_runtime.cu        planning, launches, host-buffer path, C ABI
//   plugin.cu            the _backend operator surface
#pragma once

#include "../../include/tensorbleu.h"
#include "tb_guard.h"

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#define TB_VERSION_STRING "tensorbleu-b200 0.2.0 (sm_100a)"

namespace tbk {

constexpr int kThreads = 256;
constexpr int kPairCtasPerSm = 4;  // single-reference kernel: 4 CTAs of kThreads per SM
constexpr int kMultiMaxRefs = 8;  // references handled by the multi-reference kernel
constexpr int kSparseMaxRefs = 8;  // references handled by the warp-per-group kernel
constexpr int kSparseMaxWidth = 4096;  // row widths handled by the warp-per-group kernel
constexpr int kSmallSet = 128;    // positions matched without a table (<= kThreads)
constexpr int kMultiThreads = 512;  // multi-reference kernel: 16 warps, 2 CTAs per SM
constexpr int kAccCopies = 32;         // replicated corpus accumulators (spread L2 atomics)
constexpr int kGlobalKeyShift = 26;    // global-mode key = (ref << 26) | position
constexpr uint32_t kFull = 0xffffffffu;

// records the CUDA error for tb_last_cuda_error() (tb_runtime.cu)
int cuda_fail(cudaError_t e);

#define TB_CUDA(expr)                        \
  do {                                       \
    cudaError_t _e = (expr);                 \
    if (_e != cudaSuccess) return cuda_fail(_e); \
  } while (0)

// --------------------------------------------------------------------------
// Kernel parameters (passed by value as __grid_constant__).
// --------------------------------------------------------------------------
struct RefDesc {
  const void* ids;
  int64_t ld;
  int64_t width;
  const int64_t* len;
};

struct StatsParams {
  const void* cand_ids;
  int64_t cand_ld;
  int64_t cand_width;
  const int64_t* cand_len;
  RefDesc refs[TB_MAX_REFS];
  int num_refs;
  int max_order;
  int64_t batch;
  // epilogue
  int smoothing;
  double eps;
  double k;
  double weights[TB_MAX_ORDER];
  // outputs
  int64_t* num;
  int64_t* den;
  int64_t* cand_len_out;
  int64_t* eff_ref;
  double* scores;
  double* precisions;
  double* bp;
  int64_t* totals;
  double* corpus;
  unsigned long long* acc;  // kAccCopies x (2N+2), zero on entry and on exit
  unsigned int* done;       // CTA completion counter, zero on entry and on exit
  int* ws_flag;             // OR of CTA flags, zero on entry and on exit
  int32_t* err;             // written by the last CTA
  // hash table
  int cap_log2;
  int filter_log2;  // pair kernel: 32-bit words per side of the order-1 filter (log2)
  // shared-memory layout (elements of the token type)
  int cand_pad;
  int ref_off[TB_MAX_REFS + 1];
  // pruned shared-memory kernel: byte offsets of the per-position / table arrays
  int off_id1, off_idn, off_live, off_ent, off_mref, off_kc, off_lists, off_seg;
  int off_tok2;  // pair kernel: second token buffer (prefetch of the next group), 0 = none
  // global-memory mode
  unsigned char* gtab;
  size_t gtab_stride;
  // host-buffer mode (tb_bleu_host): stage only valid prefixes (rows come over
  // PCIe); report flags through the completion protocol with a plain store
  int prefix_only;
  int err_store;
  int no_tails;  // every row is taken whole by the bulk copies: copy_row_tails has nothing to do
  // warp-group kernel: per-group shared-memory bytes, byte offsets, and the
  // element offsets of the staged rows (candidate, then reference r)
  int sp_off_fc, sp_off_fs, sp_off_tok, sp_off_ps, sp_off_aux, sp_off_rows;
  int sp_row_off[TB_MAX_REFS + 1];
  int sp_buf_elems;          // elements per row buffer
  int sp_nbuf;               // row buffers (1 or 2)
  unsigned int sp_tma_mask;  // bit s: row set s is bulk-copied (16-byte base and pitch)
  // dense groups listed by the warp-per-group kernel for the CTA-per-group kernel
  // (list mode when glist != nullptr: that kernel scores glist[0, *gcount))
  int* glist;
  unsigned int* gcount;
};

struct EpiParams {
  int smoothing;
  double eps;
  double k;
  double weights[TB_MAX_ORDER];
};

}  // namespace tbk

using namespace tbk;

namespace {

template <bool kSmem>
struct Word;
template <>
struct Word<false> {
  using T = unsigned long long;
  static constexpr int kShift = 32;
};

// --------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA engine, 1-D form).
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (the stats kernels are launched with
// programmatic stream serialization): wait until the preceding grid in the
// stream has completed and its writes are visible — before the first global
// read — then let the next grid start launching its CTAs into free SM slots,
// where they do their own prologue and wait here in turn.  This hides the
// kernel-to-kernel launch gap; without the launch attribute both are no-ops.
__device__ __forceinline__ void griddep_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// TB_DEBUG_NO_PDL=1: launch the stats kernels without programmatic stream
// serialization (A/B measurements of the launch overlap)
// TB_DEBUG_PDL_MODE (A/B only): 1 = list-mode launches keep PDL, 3 = the filter kernel takes it
inline int pdl_mode() {
  static const int v = [] {
    const char* e = getenv("TB_DEBUG_PDL_MODE");
    return e ? atoi(e) : 0;
  }();
  return v;
}
inline bool no_pdl() {
  static const bool v = [] {
    const char* e = getenv("TB_DEBUG_NO_PDL");
    return e && e[0] == '1';
  }();
  return v;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --------------------------------------------------------------------------
// Row staging shared by the shared-memory kernels.  Row s of group b is the
// candidate (s = 0) or reference s-1; it lands at element offset
// row_dst(s) of the token buffer.  Normally the full width is staged (widths
// are known without reading lengths, so the copy starts at once).  In
// prefix mode — token rows read over PCIe straight from pinned host memory
// (tb_bleu_host) — thread 0 first reads the lengths and only the valid
// prefixes cross the bus.
// --------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ const T* row_src(const StatsParams& p, int s, int64_t b) {
  return s == 0 ? static_cast<const T*>(p.cand_ids) + b * p.cand_ld
                : static_cast<const T*>(p.refs[s - 1].ids) + b * p.refs[s - 1].ld;
}
__device__ __forceinline__ int64_t row_width(const StatsParams& p, int s) {
  return s == 0 ? p.cand_width : p.refs[s - 1].width;
}
__device__ __forceinline__ int row_dst(const StatsParams& p, int s) {
  return s == 0 ? 0 : p.cand_pad + p.ref_off[s - 1];
}
__device__ __forceinline__ bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// Thread 0 only.  Prefix mode records the clamped lengths in stage_len[0..R]
// and ORs TB_FLAG_BAD_LENGTH into *flags.
template <typename T>
__device__ void issue_rows(const StatsParams& p, int64_t b, int nrows, T* tok, uint64_t* mbar, int64_t* stage_len,
                           int* flags) {
  fence_proxy_async_smem();
  if (p.prefix_only) {
    for (int s = 0; s < nrows; ++s) {
      int64_t len = s == 0 ? p.cand_len[b] : p.refs[s - 1].len[b];
      const int64_t w = row_width(p, s);
      if (len < 0 || len > w) {
        *flags |= TB_FLAG_BAD_LENGTH;
        len = len < 0 ? 0 : w;
      }
      stage_len[s] = len;
    }
  }
  uint32_t total = 0;
  for (int s = 0; s < nrows; ++s) {
    const int64_t n = p.prefix_only ? stage_len[s] : row_width(p, s);
    if (aligned16(row_src<T>(p, s, b))) total += static_cast<uint32_t>((n * sizeof(T)) & ~int64_t(15));
  }
  mbar_arrive_expect_tx(mbar, total);
  for (int s = 0; s < nrows; ++s) {
    const T* src = row_src<T>(p, s, b);
    const int64_t n = p.prefix_only ? stage_len[s] : row_width(p, s);
    const uint32_t bytes = static_cast<uint32_t>((n * sizeof(T)) & ~int64_t(15));
    if (aligned16(src) && bytes > 0) bulk_g2s(tok + row_dst(p, s), src, bytes, mbar);
  }
}

// All threads: the < 16-byte tails and rows whose address is unaligned.
template <typename T>
__device__ __forceinline__ void copy_row_tails(const StatsParams& p, int64_t b, int nrows, T* tok,
                                               const int64_t* stage_len, int tid, int nthreads) {
  for (int s = 0; s < nrows; ++s) {
    const T* src = row_src<T>(p, s, b);
    const int64_t n = p.prefix_only ? stage_len[s] : row_width(p, s);
    const int64_t start = aligned16(src) ? static_cast<int64_t>(((n * sizeof(T)) & ~int64_t(15)) / sizeof(T)) : 0;
    T* dst = tok + row_dst(p, s);
    for (int64_t j = start + tid; j < n; j += nthreads) dst[j] = src[j];
  }
}

// --------------------------------------------------------------------------
// n-gram hashing / comparison.
// --------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ uint32_t ngram_hash(const T* tok, int n) {
  uint64_t h = 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(n);
  for (int i = 0; i < n; ++i) {
    h ^= static_cast<uint64_t>(tok[i]);
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  h *= 0x94D049BB133111EBull;
  h ^= h >> 29;
  return static_cast<uint32_t>(h);
}

template <typename T>
__device__ __forceinline__ bool ngram_equal(const T* a, const T* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// Key -> pointer to the first token of the reference n-gram it names.
template <typename T, bool kSmem>
struct RefTokens {
  const T* base;                 // smem: concatenated reference rows
  const T* const* rows;          // global: per-reference row pointers (smem array)
  __device__ __forceinline__ int32_t key(int r, int64_t j, const int* ref_off) const {
    if constexpr (kSmem)
      return ref_off[r] + static_cast<int32_t>(j);
    else
      return (r << kGlobalKeyShift) | static_cast<int32_t>(j);
  }
  __device__ __forceinline__ const T* ptr(int32_t key) const {
    if constexpr (kSmem)
      return base + key;
    else
      return rows[key >> kGlobalKeyShift] + (key & ((1 << kGlobalKeyShift) - 1));
  }
};

// Insert-or-find.  Keys only ever go EMPTY(-1) -> key once per order, so a
// stale EMPTY read is repaired by the CAS and a non-empty read is final.
template <typename T, bool kSmem>
__device__ __forceinline__ int32_t table_insert(int32_t* keys, uint32_t mask, const T* gram, int n,
                                                int32_t my_key, const RefTokens<T, kSmem>& rt) {
  uint32_t s = ngram_hash(gram, n) & mask;
  while (true) {
    int32_t k = *reinterpret_cast<volatile int32_t*>(&keys[s]);
    if (k < 0) {
      k = atomicCAS(&keys[s], -1, my_key);
      if (k < 0) return static_cast<int32_t>(s);
    }
    if (ngram_equal(rt.ptr(k), gram, n)) return static_cast<int32_t>(s);
    s = (s + 1) & mask;
  }
}

template <typename T, bool kSmem>
__device__ __forceinline__ int32_t table_find(const int32_t* keys, uint32_t mask, const T* gram,
                                              int n, const RefTokens<T, kSmem>& rt) {
  uint32_t s = ngram_hash(gram, n) & mask;
  while (true) {
    const int32_t k = keys[s];
    if (k < 0) return -1;
    if (ngram_equal(rt.ptr(k), gram, n)) return static_cast<int32_t>(s);
    s = (s + 1) & mask;
  }
}

// --------------------------------------------------------------------------
// fp64 epilogue with numpy's operation order (bleu.py:213-261).
// __d*_rn intrinsics keep nvcc from contracting into FMAs that numpy does
// not perform.
// --------------------------------------------------------------------------
__device__ void bleu_epilogue(const int64_t* num, const int64_t* den, int64_t c, int64_t r, int N,
                              int smoothing, double eps, double kk, const double* w,
                              double* prec_out, double* bp_out, double* score_out) {
  double p[TB_MAX_ORDER];
  double counter = 1.0;
  for (int n = 0; n < N; ++n) {
    const double nd = static_cast<double>(num[n]);
    const double dd = static_cast<double>(den[n]);
    const bool has_den = den[n] > 0;
    double pn = has_den ? __ddiv_rn(nd, dd) : 0.0;            // bleu.py:222
    const bool zero_num = (num[n] == 0) && has_den;           // bleu.py:223
    if (smoothing == TB_SMOOTH_FLOOR) {
      if (zero_num) pn = __ddiv_rn(eps, dd);                  // bleu.py:228
    } else if (smoothing == TB_SMOOTH_ADD_K) {
      if (n >= 1 && has_den) pn = __ddiv_rn(__dadd_rn(nd, kk), __dadd_rn(dd, kk));  // bleu.py:230-232
    } else if (smoothing == TB_SMOOTH_EXP) {
      if (zero_num) {                                         // bleu.py:234-238
        pn = __ddiv_rn(1.0, __dmul_rn(ldexp(1.0, static_cast<int>(counter)), dd));  // np.exp2 of an integer: exact
        counter = __dadd_rn(counter, 1.0);
      }
    }
    p[n] = pn;
    if (prec_out) prec_out[n] = pn;
  }
  // _bp_vector, bleu.py:256-261
  const double cd = static_cast<double>(c);
  const double rd = static_cast<double>(r);
  double bp = (cd > rd) ? 1.0 : exp(__dsub_rn(1.0, __ddiv_rn(rd, cd > 0.0 ? cd : 1.0)));
  if (!(cd > 0.0)) bp = 0.0;
  // _geo_mean_scores, bleu.py:242-253 (sequential sum over active orders)
  bool ok = true;
  double s = 0.0;
  for (int n = 0; n < N; ++n) {
    if (!(w[n] > 0.0)) continue;
    if (p[n] > 0.0)
      s = __dadd_rn(s, __dmul_rn(log(p[n]), w[n]));
    else
      ok = false;
  }
  double score = ok ? __dmul_rn(bp, exp(s)) : 0.0;
  score = fmin(fmax(score, 0.0), 1.0);
  if (bp_out) *bp_out = bp;
  if (score_out) *score_out = score;
}

// effective reference length: closest to c, ties -> shorter (bleu.py:108-114)
__device__ __forceinline__ int64_t closest_ref_len(int64_t c, const int64_t* ref_lens, int R) {
  int64_t best = ref_lens[0];
  int64_t best_d = best > c ? best - c : c - best;
  for (int r = 1; r < R; ++r) {
    const int64_t v = ref_lens[r];
    const int64_t d = v > c ? v - c : c - v;
    if (d < best_d || (d == best_d && v < best)) {
      best = v;
      best_d = d;
    }
  }
  return best;
}

// --------------------------------------------------------------------------
// Warp-parallel epilogue (lane n owns order n; N <= 32).  Same operations and
// order as bleu_epilogue / numpy: the log terms are summed sequentially by
// lane 0.  All 32 lanes of the warp must call it.
// --------------------------------------------------------------------------
// brevity penalty, bleu.py:256-261 (1 if c > r, 0 if c == 0, else exp(1 - r/c))
__device__ __forceinline__ double brevity_penalty_fp64(int64_t c, int64_t r) {
  const double cd = static_cast<double>(c);
  const double rd = static_cast<double>(r);
  double bp = (cd > rd) ? 1.0 : exp(__dsub_rn(1.0, __ddiv_rn(rd, cd > 0.0 ? cd : 1.0)));
  if (!(cd > 0.0)) bp = 0.0;
  return bp;
}

// `bp_in` >= 0: the brevity penalty was computed beforehand (by another warp)
__device__ void warp_epilogue(int64_t num, int64_t den, int64_t c, int64_t r, int N, int smoothing,
                              double eps, double kk, double w, double* prec_out, double* bp_out,
                              double* score_out, double bp_in = -1.0) {
  const int lane = threadIdx.x & 31;
  const bool act = lane < N;
  const double nd = static_cast<double>(num);
  const double dd = static_cast<double>(den);
  const bool has_den = act && den > 0;
  const bool zero_num = has_den && num == 0;
  // divisors of lanes without a denominator are replaced by 1: a division by 0
  // takes the slow path of the fp64 divide (hundreds of cycles) even though its
  // result is discarded
  const double ds = has_den ? dd : 1.0;
  // 0 / den is +0 exactly; a zero numerator would also take the divide's slow
  // path (its operand-range check fails for |x| < 2^-120), and one such lane
  // stalls the warp for hundreds of cycles
  double pn = (has_den && num != 0) ? __ddiv_rn(nd, ds) : 0.0;
  if (smoothing == TB_SMOOTH_FLOOR) {
    if (zero_num) pn = __ddiv_rn(eps, ds);
  } else if (smoothing == TB_SMOOTH_ADD_K) {
    if (lane >= 1 && has_den) pn = __ddiv_rn(__dadd_rn(nd, kk), __dadd_rn(ds, kk));
  } else if (smoothing == TB_SMOOTH_EXP) {
    const unsigned zb = __ballot_sync(kFull, zero_num);
    const double counter = 1.0 + static_cast<double>(__popc(zb & ((1u << lane) - 1u)));
    if (zero_num) pn = __ddiv_rn(1.0, __dmul_rn(ldexp(1.0, static_cast<int>(counter)), ds));  // exact 2^counter
  }
  if (act && prec_out) prec_out[lane] = pn;
  const double bp = bp_in >= 0.0 ? bp_in : brevity_penalty_fp64(c, r);
  const bool wpos = act && w > 0.0;
  const bool bad = __any_sync(kFull, wpos && !(pn > 0.0));  // an active precision is 0: score 0
  double score = 0.0;
  if (!bad) {
    const double term = wpos ? __dmul_rn(log(pn), w) : 0.0;
    double s = 0.0;
    for (int n = 0; n < N; ++n) {
      const double t = __shfl_sync(kFull, term, n);
      if (__shfl_sync(kFull, wpos ? 1 : 0, n)) s = __dadd_rn(s, t);
    }
    score = fmin(fmax(__dmul_rn(bp, exp(s)), 0.0), 1.0);
  }
  if (lane == 0) {
    if (bp_out) *bp_out = bp;
    if (score_out) *score_out = score;
  }
}

// --------------------------------------------------------------------------
// Completion protocol shared by the stats kernels: CTA flags (+ corpus
// totals) reach the last CTA to finish, which writes *err, runs the corpus
// epilogue and leaves the workspace zeroed for the next launch.
// --------------------------------------------------------------------------
// The last CTA of a launch: the replicated accumulators summed (one parallel
// read of all copies) into the totals + the corpus epilogue, the flags moved
// to *err, and the workspace left zeroed for the next launch.  All threads of
// the CTA call it; s_tot has >= 2N+2 words.
__device__ void finalize_launch(const StatsParams& p, unsigned long long* s_tot) {
  const int tid = threadIdx.x;
  const int N = p.max_order;
  const int nt = 2 * N + 2;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  if (corpus) {  // thread j sums slot j over the copies (measured faster than
    // spreading the copies over the CTA with shared atomics: c4 40.4 vs 41.7 us)
    for (int j = tid; j < nt; j += blockDim.x) {
      unsigned long long sum = 0;
      for (int c = 0; c < kAccCopies; ++c) sum += atomicExch(&p.acc[c * nt + j], 0ull);
      s_tot[j] = sum;
      if (p.totals) p.totals[j] = static_cast<int64_t>(sum);
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int f = atomicExch(p.ws_flag, 0);
    if (corpus)
      *p.err = f;  // corpus launches write the flag word
    else if (f && p.err_store)
      *p.err |= f;  // host mapped memory: plain stores only (the warp-group kernel may have set bits)
    else if (f)
      atomicOr(p.err, f);
    *p.done = 0;
    if (p.gcount) *p.gcount = 0;
  }
  if (p.corpus && tid < 32) {
    const int lane = tid;
    warp_epilogue(lane < N ? static_cast<int64_t>(s_tot[lane]) : 0,
                  lane < N ? static_cast<int64_t>(s_tot[N + lane]) : 0, static_cast<int64_t>(s_tot[2 * N]),
                  static_cast<int64_t>(s_tot[2 * N + 1]), N, p.smoothing, p.eps, p.k,
                  lane < N ? p.weights[lane] : 0.0, p.corpus + 2, p.corpus + 1, p.corpus);
  }
}

// Arrival of one CTA at the completion counter (release its updates, acquire
// everyone else's); true for the last of `participants`.
__device__ __forceinline__ bool arrive_last(const StatsParams& p, unsigned int participants) {
  unsigned int prev;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.done) : "memory");
  return prev == participants - 1;
}

// End of a CTA of the CTA-per-group kernels.  nb (list mode): the number of
// listed groups; only the CTAs that got one take part (none when nothing was
// listed: the warp-group kernel has finished the launch).
template <bool listed = false>
__device__ void finish_cta(const StatsParams& p, unsigned long long* s_tot, int& s_flags, int& s_last,
                           int64_t nb = -1) {
  const int tid = threadIdx.x;
  const int N = p.max_order;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  if (!corpus && !p.err_store && !listed) {  // no cross-CTA work: report flags directly (the caller zeroed *err)
    __syncthreads();
    if (tid == 0 && s_flags) atomicOr(p.err, s_flags);
    return;
  }
  unsigned int participants = gridDim.x;
  if constexpr (listed) {
    if (nb < 1) return;
    participants = static_cast<unsigned int>(nb < gridDim.x ? nb : gridDim.x);
    if (blockIdx.x >= participants) return;  // no group, no flags, no totals
  }
  const int nt = 2 * N + 2;
  __syncthreads();  // s_tot of the last group (warp 0's epilogue) before other threads read it
  if (corpus && tid < nt && s_tot[tid]) atomicAdd(&p.acc[(blockIdx.x % kAccCopies) * nt + tid], s_tot[tid]);
  if (tid == 0 && s_flags) atomicOr(p.ws_flag, s_flags);
  __syncthreads();
  if (tid == 0) s_last = arrive_last(p, participants);
  __syncthreads();
  if (s_last) finalize_launch(p, s_tot);
}



// Debug-only phase timestamps (build with -DTB_PHASES; see tools/phase_profile.py)
#ifdef TB_PHASES
__device__ unsigned long long* g_tb_phases;  // per translation unit
#define TB_MARK(k)                                                                        \
  do {                                                                                   \
    if (threadIdx.x == 0 && g_tb_phases && (k) < 32) {                                   \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
      g_tb_phases[blockIdx.x * 32 + (k)] = t_;                                           \
    }                                                                                    \
  } while (0)
#else
#define TB_MARK(k) \
  do {             \
  } while (0)
#endif
#ifdef TB_PHASES
#define TB_NOTE(k, v)                                                   \
  do {                                                                  \
    if (threadIdx.x == 0 && g_tb_phases) g_tb_phases[blockIdx.x * 32 + (k)] = (v); \
  } while (0)
#else
#define TB_NOTE(k, v) \
  do {                \
  } while (0)
#endif

// 32-bit multiplicative hash of a token; use the TOP bits (h >> (32 - bits))
#ifdef TB_PHASES
// every kernel TU has its own g_tb_phases (no relocatable device code)
inline int set_phase_buffer_here(void* buf) {
  TB_CUDA(cudaMemcpyToSymbol(g_tb_phases, &buf, sizeof(buf)));
  return TB_OK;
}
#endif

// 1 << (s & 31) in one funnel shift
__device__ __forceinline__ uint32_t bit_of(uint32_t s) { return __funnelshift_l(1u, 1u, s); }

template <typename T>
__device__ __forceinline__ uint32_t tok_hash32(T t) {
  if constexpr (sizeof(T) == 4) {
    return static_cast<uint32_t>(t) * 0x9E3779B1u;
  } else {
    uint64_t h = static_cast<uint64_t>(t);
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    return static_cast<uint32_t>(h >> 32);
  }
}

// warp-aggregated append of `val` to list[*count] for lanes with `pred`;
// every lane of the warp must call it

//           [ref 16 | cand 16] (the only atomic of the common path); a
//           different token is lost and retries in rounds with fresh hashes
//           (plain stores again), then serial CAS probing for leftovers.
// Reference tokens only look up (an absent token can neither be counted nor
// start a matching n-gram).  The liveness pass adds min(cand, ref) once per
// slot (by its owner) and lists the positions whose token occurs on the other
// side; only those are extended at the next order (exact pruning).
// Orders >= 2 run the same claim / verify-or-look-up / live rounds over that
// list (owners, counts and next-order ids are list indices); their keys live
// in `kc`, which aliases the token buffer (dead after order 1).
// --------------------------------------------------------------------------
// 32-bit CAS on a shared-memory address (explicit state space: the address is
// computed with integer arithmetic, which would otherwise become a generic,
// GPU-scope ATOM instead of ATOMS).
__device__ __forceinline__ uint32_t atom_cas_shared(uint32_t saddr, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.shared::cta.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(saddr), "r"(cmp), "r"(val) : "memory");
  return old;
}

// claim the EMPTY (0xffff) u16 slot `slot` of `own` for `desired`
__device__ __forceinline__ bool cas16(uint16_t* own, uint32_t slot, uint16_t desired, uint16_t* seen) {
  const uint32_t waddr = smem_u32(own) + 4 * (slot >> 1);
  const int sh = static_cast<int>((slot & 1) * 16);
  uint32_t cur;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(cur) : "r"(waddr));
  while (true) {
    const uint16_t h = static_cast<uint16_t>(cur >> sh);
    if (h != 0xffffu) {
      *seen = h;
      return false;
    }
    const uint32_t nw = (cur & ~(0xffffu << sh)) | (static_cast<uint32_t>(desired) << sh);
    const uint32_t prev = atom_cas_shared(waddr, cur, nw);
    if (prev == cur) return true;
    cur = prev;
  }
}

// Deferred insert of a position whose home slot was won by a different key:
// linear probing from the home slot (8 slots per 16-byte read).  All plain
// round-1 stores are complete, so entries are EMPTY or owned; CAS claims an
// EMPTY one, an equal key adds to its owner's count.
template <typename EqF>
__device__ __forceinline__ uint32_t pair_insert_loser(uint16_t* own, uint32_t* cnt, uint32_t home, uint32_t mask,
                                                      uint16_t me, uint32_t inc, EqF eq) {
  const uint32_t base = smem_u32(own);
  uint32_t s = (home + 1) & mask;
  while (true) {
    uint16_t v;
    asm volatile("ld.volatile.shared.u16 %0, [%1];" : "=h"(v) : "r"(base + 2 * s));
    if (v == 0xffffu && cas16(own, s, me, &v)) return s;
    if (eq(v)) {
      atomicAdd(&cnt[v], inc);
      return s;
    }
    s = (s + 1) & mask;
  }
}

// Barriers of a thread subset: BAR == 0 is the whole CTA (__syncthreads);
// otherwise named barrier BAR over the NT threads that take part.
template <int NT, int BAR>
__device__ __forceinline__ void bsync() {
  if constexpr (BAR == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}
template <int NT, int BAR>
__device__ __forceinline__ int bsync_or(int v) {
  if constexpr (BAR == 0) {
    return __syncthreads_or(v);
  } else {
    int r;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t"
        "bar.red.or.pred p, %2, %3, p;\n\tselp.s32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(v), "n"(BAR), "n"(NT)
        : "memory");
    return r;
  }
}

// Round-r slot of a key whose round-1 home is the top bits of h (r >= 1):
// independent multiplicative remixes of the same 32-bit hash.
__device__ __forceinline__ uint32_t rehash(uint32_t h, int r, uint32_t hshift) {
  constexpr uint32_t kMul[4] = {0x85EBCA6Bu, 0xC2B2AE35u, 0x27D4EB2Fu, 0x165667B1u};
  h ^= h >> 15;
  return (h * kMul[r - 1]) >> hshift;
}

constexpr int kRetryRounds = 4;

// Store half of retry round r for a lost position: claim slot rehash_r if it is
// EMPTY (plain store; racing stores of the same round are resolved when verifying).
__device__ __forceinline__ void pair_retry_store(uint16_t* own, uint32_t h, int r, uint32_t hshift, uint16_t pos) {
  const uint32_t cs = rehash(h, r, hshift);
  if (own[cs] == 0xffffu) own[cs] = pos;
}

// Resolve the positions on `lost` (their round-1 home slot is owned by a
// different key).  All occurrences of a key share its home, so all of them
// are on the list, and they move together: retry round r stores every lost
// position into slot rehash_r(key) if that slot was EMPTY when read (plain
// stores, one wins), a barrier, then every position verifies — the owner
// keeps the slot, an equal key adds one to the owner's count, a different
// key stays lost.  A key is either settled or entirely still lost after
// each round, so the serial linear probing from the home slot that handles
// the (rare) leftovers after kRetryRounds is self-consistent.
// The store half of round r+1 runs in the same pass as the verify half of
// round r: stores only ever target EMPTY slots, and every slot being verified
// in round r is non-empty, so the two halves cannot interfere.  The caller has
// done the store half of round 1 (in its home-slot verify pass) and a barrier
// (with first_round > 1, rounds before it are complete and the store half of
// first_round is done).  `ids[pos]` receives the final slot.  All threads call it.
template <int NT = kThreads, int BAR = 0, typename HashF, typename EqF>
__device__ __forceinline__ void pair_resolve_lost(uint16_t* own, uint32_t* cnt, uint16_t* lost, int nl, uint16_t* ids,
                                                  uint32_t mask, uint32_t hshift, int roff, int tid, HashF hash,
                                                  EqF eq, int first_round = 1) {
  for (int r = first_round; r <= kRetryRounds; ++r) {
    int left = 0;
    for (int i = tid; i < nl; i += NT) {
      const uint16_t pos = lost[i];
      if (pos == 0xffffu) continue;
      const uint32_t h = hash(pos);
      const uint32_t cs = rehash(h, r, hshift);
      const uint16_t w = own[cs];
      if (w == pos || eq(pos, w)) {
        if (w != pos) atomicAdd(&cnt[w], pos < roff ? 1u : (1u << 16));
        ids[pos] = static_cast<uint16_t>(cs);
        lost[i] = 0xffffu;
      } else {
        left = 1;
        if (r < kRetryRounds) pair_retry_store(own, h, r + 1, hshift, pos);
      }
    }
    if (!bsync_or<NT, BAR>(left)) return;
  }
  for (int i = tid; i < nl; i += NT) {
    const uint16_t pos = lost[i];
    if (pos == 0xffffu) continue;
    ids[pos] = static_cast<uint16_t>(pair_insert_loser(own, cnt, ids[pos], mask, pos, pos < roff ? 1u : (1u << 16),
                                                       [&](uint16_t x) { return eq(pos, x); }));
  }
  bsync<NT, BAR>();
}

// pair_resolve_lost for the live-list passes of orders >= 2: `lost` holds list
// indices e (owners are list indices, keys kc[e], hash key * 0x9E3779B1), all of
// candidate entries; settling e writes its owner's list index to idn[lin[e]].
template <int NT = kThreads, int BAR = 0>
__device__ __forceinline__ void list_resolve_lost(uint16_t* own, uint32_t* cnt, const uint32_t* kc, uint16_t* lost,
                                                  int nl, const uint16_t* lin, uint16_t* idn, uint32_t mask,
                                                  uint32_t hshift, int tid) {
  for (int r = 1; r <= kRetryRounds; ++r) {
    int left = 0;
    for (int i = tid; i < nl; i += NT) {
      const uint16_t e = lost[i];
      if (e == 0xffffu) continue;
      const uint32_t key = kc[e];
      const uint32_t h = key * 0x9E3779B1u;
      const uint16_t w = own[rehash(h, r, hshift)];
      if (w == e || kc[w] == key) {
        if (w != e) atomicAdd(&cnt[w], 1u);
        idn[lin[e]] = w;
        lost[i] = 0xffffu;
      } else {
        left = 1;
        if (r < kRetryRounds) pair_retry_store(own, h, r + 1, hshift, e);
      }
    }
    if (!bsync_or<NT, BAR>(left)) return;
  }
  for (int i = tid; i < nl; i += NT) {
    const uint16_t e = lost[i];
    if (e == 0xffffu) continue;
    const uint32_t key = kc[e];
    const uint32_t sl = pair_insert_loser(own, cnt, (key * 0x9E3779B1u) >> hshift, mask, e, 1u,
                                          [&](uint16_t x) { return kc[x] == key; });
    uint16_t w;
    asm volatile("ld.volatile.shared.u16 %0, [%1];" : "=h"(w) : "r"(smem_u32(own) + 2 * sl));
    idn[lin[e]] = w;
  }
  bsync<NT, BAR>();
}

// Warp-aggregated appends to a shared list (one atomic per warp).  All 32 lanes
// call.  warp_append: one value per lane.
__device__ __forceinline__ void warp_append(uint16_t* list, int* count, bool want, int v, int lane) {
  const unsigned m = __ballot_sync(kFull, want);
  if (!m) return;
  const int src = __ffs(m) - 1;
  int base = 0;
  if (lane == src) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, src);
  if (want) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(v);
}
// warp_append_quad: the values v(k) for the set bits k of m (4 bits per lane),
// offsets by a warp prefix sum of the per-lane counts
template <typename V>
__device__ __forceinline__ void warp_append_quad(uint16_t* list, int* count, uint32_t m, V v, int lane) {
  if (!__any_sync(kFull, m != 0)) return;
  const int n = __popc(m);
  int incl = n;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  int base = 0;
  if (lane == 31) base = atomicAdd(count, incl);
  base = __shfl_sync(kFull, base, 31) + incl - n;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (m >> k & 1u) list[base++] = static_cast<uint16_t>(v(k));
}

// Slot of token t among the inserted (candidate) tokens, or -1; *owner gets its
// owner position.  Follows an inserted key's placement order: home slot, the
// retry rounds' slots, then linear probing from home + 1 — a key sits at the
// first slot of that chain that it owns, and every earlier slot of the chain is
// owned by another key (slots never empty again), so an EMPTY slot ends the search.
// pair_find_retry continues after a home slot owned by a different token.
template <typename T>
__device__ __forceinline__ int pair_find_retry(const uint16_t* own, const T* tok, T t, uint32_t h, uint32_t hshift,
                                            uint32_t mask, uint16_t* owner) {
  const uint32_t home = h >> hshift;
  uint16_t o;
#pragma unroll 1
  for (int r = 1; r <= kRetryRounds; ++r) {
    const uint32_t cs = rehash(h, r, hshift);
    o = own[cs];
    if (o == 0xffffu) return -1;
    if (tok[o] == t) {
      *owner = o;
      return static_cast<int>(cs);
    }
  }
  for (uint32_t s = (home + 1) & mask;; s = (s + 1) & mask) {
    o = own[s];
    if (o == 0xffffu) return -1;
    if (tok[o] == t) {
      *owner = o;
      return static_cast<int>(s);
    }
  }
}


// --------------------------------------------------------------------------
// Exact clipped counts of a short element list (the filter kernel's listed
// survivors, the pair kernel's finisher warp): elements sorted by (row,
// position), counted per order with match.any (S <= 32) or a tiny hash table
// per order (S <= kSparseMax).
// --------------------------------------------------------------------------
constexpr int kSparseMax = 128;  // listed elements handled per group
constexpr int kTinySlots = 256;  // tiny table (>= 2 * kSparseMax)

// Element list key: (row << 23) | (position << 7) | list slot — sorting keys
// sorts by (row, position) and carries the slot of the element's token.
__device__ __forceinline__ uint32_t elem_key(uint32_t side, uint32_t pos, uint32_t slot) {
  return (side << 23) | (pos << 7) | slot;
}

// Bitonic sort (ascending) of 32 * K keys in a warp; element i = j * 32 + lane is key[j].
template <int K>
__device__ __forceinline__ void warp_sort(uint32_t (&key)[K], int lane) {
  constexpr int n = 32 * K;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
    for (int s = k >> 1; s > 0; s >>= 1) {
      if (s >= 32) {  // partner in another register of this lane
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const int pj = j ^ (s / 32);
          if (pj > j) {
            const int i = j * 32 + lane;
            const bool up = (i & k) == 0;
            const uint32_t a = key[j], b = key[pj];
            const bool swap = up ? (a > b) : (a < b);
            key[j] = swap ? b : a;
            key[pj] = swap ? a : b;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const int i = j * 32 + lane;
          const uint32_t o = __shfl_xor_sync(kFull, key[j], s);
          const bool up = (i & k) == 0;
          const bool lower = (lane & s) == 0;
          key[j] = (lower == up) ? (key[j] < o ? key[j] : o) : (key[j] > o ? key[j] : o);
        }
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ T lane_sentinel(int lane) {
  return static_cast<T>(-1 - lane);
}

// Exact clipped counts of the S listed elements (one warp; etok / eps hold the
// list, 1 <= S <= kSparseMax).  Returns order n's clipped count in lane n-1.
template <typename T>
__device__ __noinline__ unsigned int exact_counts(T* etok, uint32_t* eps, uint32_t* ekey, uint8_t* eid1,
                                                  uint8_t* epid, uint8_t* eval, uint16_t* town, uint32_t* tcnt,
                                                  int S, int R, int N, int lane) {
  unsigned int hits = 0;
  if (S > 0 && S <= 32) {
    uint32_t key[1] = {lane < S ? elem_key(eps[lane] >> 16, eps[lane] & 0xffffu, lane) : 0xffffffffu};
    warp_sort<1>(key, lane);
    const bool v = lane < S;
    const int e = static_cast<int>(key[0] & 127u);
    const int side = v ? static_cast<int>(key[0] >> 23) : 15;
    const int pos = static_cast<int>((key[0] >> 7) & 0xffffu);
    const T tk = v ? etok[e] : lane_sentinel<T>(lane);
    using MT = typename std::conditional<sizeof(T) == 4, unsigned int, unsigned long long>::type;
    unsigned peers = __match_any_sync(kFull, static_cast<MT>(tk));
    auto clip = [&](unsigned pr, bool valid, unsigned& c, unsigned& x) {
      const unsigned vb = __ballot_sync(kFull, valid);
      c = __popc(pr & vb & __ballot_sync(kFull, side == 0));
      x = 0;
      for (int r = 1; r <= R; ++r) {
        const unsigned xr = __popc(pr & vb & __ballot_sync(kFull, side == r));
        x = xr > x ? xr : x;
      }
    };
    unsigned c, x;
    clip(peers, v, c, x);
    int leader = __ffs(peers) - 1;
    unsigned h = (v && lane == leader) ? (c < x ? c : x) : 0u;
    h = __reduce_add_sync(kFull, h);
    if (lane == 0) hits = h;
    bool valid = v && (side == 0 ? x > 0 : c > 0);  // its token matched: live at order 1
    const int id1 = leader;
    // the next element is the next position of the same row
    const int pos_nx = __shfl_down_sync(kFull, pos, 1);
    const int side_nx = __shfl_down_sync(kFull, side, 1);
    const bool consec = lane + 1 < S && side_nx == side && pos_nx == pos + 1;
    int pid = leader;
    for (int n = 2; n <= N; ++n) {
      if (!__any_sync(kFull, valid && side == 0)) break;  // no candidate (n-1)-gram matched
      const bool up = __shfl_down_sync(kFull, valid, 1);
      const int last = __shfl_sync(kFull, id1, (lane + n - 1) & 31);
      valid = valid && consec && up;
      const unsigned nkey = valid ? static_cast<unsigned>(pid * 32 + last) : 1024u + lane;
      peers = __match_any_sync(kFull, nkey);
      clip(peers, valid, c, x);
      leader = __ffs(peers) - 1;
      h = (valid && lane == leader) ? (c < x ? c : x) : 0u;
      h = __reduce_add_sync(kFull, h);
      if (lane == n - 1) hits = h;
      valid = valid && (side == 0 ? x > 0 : c > 0);
      pid = leader;
    }
  } else if (S > 32) {
    // sort, rewrite the list in (row, position) order, then a tiny table per order
    constexpr int kJ = kSparseMax / 32;
    const int W = (R + 1 + 3) >> 2;  // count words per owner: 8-bit count per row
    uint32_t key[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int e = j * 32 + lane;
      key[j] = e < S ? elem_key(eps[e] >> 16, eps[e] & 0xffffu, e) : 0xffffffffu;
    }
    warp_sort<kJ>(key, lane);
    T tj[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) tj[j] = j * 32 + lane < S ? etok[key[j] & 127u] : T(0);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int e = j * 32 + lane;
      if (e < S) {
        etok[e] = tj[j];
        eps[e] = ((key[j] >> 23) << 16) | ((key[j] >> 7) & 0xffffu);
      }
    }
    uint32_t own_e[kJ];
    for (int i = lane; i < kTinySlots / 2; i += 32) reinterpret_cast<uint32_t*>(town)[i] = 0xffffffffu;
    for (int i = lane; i < S * W; i += 32) tcnt[i] = 0;
    __syncwarp();
    // order 1: keys are the tokens
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int e = lane + 32 * j;
      own_e[j] = 0xffffu;
      if (e < S) {
        const T tk = etok[e];
        uint32_t s = tok_hash32(tk) >> 24;
        uint16_t o;
        while (true) {
          uint16_t seen;
          if (cas16(town, s, static_cast<uint16_t>(e), &seen)) {
            o = static_cast<uint16_t>(e);
            break;
          }
          if (etok[seen] == tk) {
            o = seen;
            break;
          }
          s = (s + 1) & (kTinySlots - 1);
        }
        own_e[j] = o;
        const int side = static_cast<int>(eps[e] >> 16);
        atomicAdd(&tcnt[o * W + (side >> 2)], 1u << (8 * (side & 3)));
      }
    }
    __syncwarp();
    auto counts = [&](uint32_t o, unsigned& c, unsigned& x) {
      c = tcnt[o * W] & 0xffu;
      x = 0;
      for (int s = 1; s <= R; ++s) {
        const unsigned xs = (tcnt[o * W + (s >> 2)] >> (8 * (s & 3))) & 0xffu;
        x = xs > x ? xs : x;
      }
    };
    unsigned acc = 0;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int e = lane + 32 * j;
      if (e < S) {
        unsigned c, x;
        counts(own_e[j], c, x);
        if (own_e[j] == static_cast<uint32_t>(e)) acc += c < x ? c : x;
        const int side = static_cast<int>(eps[e] >> 16);
        eval[e] = (side == 0 ? x > 0 : c > 0) ? 1 : 0;
        eid1[e] = static_cast<uint8_t>(own_e[j]);
        epid[e] = static_cast<uint8_t>(own_e[j]);
      }
    }
    acc = __reduce_add_sync(kFull, acc);
    if (lane == 0) hits = acc;
    __syncwarp();
    for (int n = 2; n <= N; ++n) {
      // (a) keys of the valid order-n elements
      bool any_c = false;
      bool vj[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int e = lane + 32 * j;
        vj[j] = false;
        if (e + 1 < S && eval[e] && eval[e + 1]) {
          const uint32_t a = eps[e], nx = eps[e + 1];
          // the next element is the next position of the same row and its
          // (n-1)-gram matched too
          vj[j] = (nx >> 16) == (a >> 16) && (nx & 0xffffu) == (a & 0xffffu) + 1;
        }
        if (vj[j]) any_c |= (eps[e] >> 16) == 0;
        ekey[e] = vj[j] ? (static_cast<uint32_t>(epid[e]) << 8) | eid1[e + n - 1] : 0xffffffffu;
      }
      if (!__any_sync(kFull, any_c)) break;
      for (int i = lane; i < kTinySlots / 2; i += 32) reinterpret_cast<uint32_t*>(town)[i] = 0xffffffffu;
      for (int i = lane; i < S * W; i += 32) tcnt[i] = 0;
      __syncwarp();
      // (b) insert / count
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int e = lane + 32 * j;
        own_e[j] = 0xffffu;
        if (vj[j]) {
          const uint32_t k2 = ekey[e];
          uint32_t s = (k2 * 0x9E3779B1u) >> 24;
          uint16_t o;
          while (true) {
            uint16_t seen;
            if (cas16(town, s, static_cast<uint16_t>(e), &seen)) {
              o = static_cast<uint16_t>(e);
              break;
            }
            if (ekey[seen] == k2) {
              o = seen;
              break;
            }
            s = (s + 1) & (kTinySlots - 1);
          }
          own_e[j] = o;
          const int side = static_cast<int>(eps[e] >> 16);
          atomicAdd(&tcnt[o * W + (side >> 2)], 1u << (8 * (side & 3)));
        }
      }
      __syncwarp();
      // (c) clipped counts; the matched stay valid; ids for the next order
      acc = 0;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int e = lane + 32 * j;
        if (e < S) {
          bool nv = false;
          if (vj[j]) {
            unsigned c, x;
            counts(own_e[j], c, x);
            if (own_e[j] == static_cast<uint32_t>(e)) acc += c < x ? c : x;
            nv = (eps[e] >> 16) == 0 ? x > 0 : c > 0;
            epid[e] = static_cast<uint8_t>(own_e[j]);
          }
          eval[e] = nv ? 1 : 0;
        }
      }
      acc = __reduce_add_sync(kFull, acc);
      if (lane == n - 1) hits = acc;
      __syncwarp();
    }
  }

  return hits;
}

}  // namespace
