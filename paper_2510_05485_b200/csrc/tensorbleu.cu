// tensorbleu.cu — B200 (sm_100a) kernels + C ABI for the TensorBLEU hot path.
//
// See include/tensorbleu.h for the contract of every exported symbol and
// DESIGN.md for the data layout and the roofline of each kernel.
//
// Reference behaviour followed (paths relative to /root/reference):
//   counting   pkg/src/batchbleu/bleu.py:117-159   (_chunk_stats)
//              pkg/src/batchbleu/ngrams.py:144-205 (packed_order_ids, segmented_bincount,
//                                                   clipped_row_sums)
//              pkg/src/batchbleu/_kernels.pyx:84-180 (segment_bincount, clipped_numerators)
//   eff. ref   pkg/src/batchbleu/bleu.py:108-114
//   epilogue   pkg/src/batchbleu/bleu.py:213-261, 274-305
//
// Design (one sentence group = candidate i + its R references):
//   * one CTA owns a group at a time (grid-stride over groups, all CTAs
//     resident, programmatic dependent launch hides the launch gap);
//   * the group's rows are staged in shared memory with bulk-async copies
//     (cp.async.bulk -> UBLKCP, completion on an mbarrier) — only the valid
//     prefixes when the rows come over PCIe from pinned host memory;
//   * bleu_pair_kernel (R = 1): an order-1 Bloom filter drops the tokens absent
//     from the other side; the few survivors of unrelated text are matched
//     exactly with match.any (or by direct comparison), otherwise candidate
//     tokens are inserted store-then-verify into a shared-memory table (plain
//     stores, retry rounds with fresh hashes for the rare collisions) and
//     reference tokens look up; min(cand, ref) is added once per key by its
//     owner;
//   * orders >= 2 visit only n-grams whose (n-1)-prefix and last token matched:
//     key = (id of the prefix, order-1 id of the last token); <= 32 live
//     positions finish in one warp with match.any, more run one table round
//     per order over the LIST of live positions (three barrier phases);
//   * bleu_multi_kernel (2 <= R <= 8): the same passes with one count per
//     (reference, candidate owner), clip = min(cand, max_r ref_r);
//     bleu_group_kernel (R > 8) walks the references one by one;
//   * warp 0 finishes the group: effective reference length, smoothing, BP,
//     weighted geometric mean, in fp64 with numpy's operation order;
//   * corpus mode accumulates the int64 totals per CTA and the last CTA to
//     finish runs the corpus epilogue (one launch in total).
// Rows too wide for shared memory run bleu_stats_kernel with the table and
// tokens in global memory (64-bit count words).

#include "../../include/tensorbleu.h"

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

#define TB_VERSION_STRING "tensorbleu-b200 0.1.0 (sm_100a)"

namespace {

constexpr int kThreads = 256;
constexpr int kPairCtasPerSm = 4;  // single-reference kernel: 4 CTAs of kThreads per SM
constexpr int kMultiMaxRefs = 8;  // references handled by the multi-reference kernel
constexpr int kSmallSet = 128;    // positions matched without a table (<= kThreads)
constexpr int kMultiThreads = 512;  // multi-reference kernel: 16 warps, 2 CTAs per SM
constexpr int kAccCopies = 32;         // replicated corpus accumulators (spread L2 atomics)
constexpr int kGlobalKeyShift = 26;    // global-mode key = (ref << 26) | position
constexpr uint32_t kFull = 0xffffffffu;

thread_local char g_last_cuda_error[256] = "";

int cuda_fail(cudaError_t e) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
  return TB_ERR_CUDA;
}

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
};

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
__device__ void finish_cta(const StatsParams& p, unsigned long long* s_tot, int& s_flags, int& s_last) {
  const int tid = threadIdx.x;
  const int N = p.max_order;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  if (!corpus && !p.err_store) {  // no cross-CTA work: report flags directly (the caller zeroed *err)
    __syncthreads();
    if (tid == 0 && s_flags) atomicOr(p.err, s_flags);
    return;
  }
  const int nt = 2 * N + 2;
  __syncthreads();  // s_tot of the last group (warp 0's epilogue) before other threads read it
  if (corpus && tid < nt && s_tot[tid]) atomicAdd(&p.acc[(blockIdx.x % kAccCopies) * nt + tid], s_tot[tid]);
  if (tid == 0 && s_flags) atomicOr(p.ws_flag, s_flags);
  __syncthreads();
  if (tid == 0) {
    // release this CTA's accumulator/flag updates, acquire everyone else's
    unsigned int prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.done) : "memory");
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    if (corpus && tid < nt) {
      unsigned long long sum = 0;
      for (int c = 0; c < kAccCopies; ++c) sum += atomicExch(&p.acc[c * nt + tid], 0ull);
      s_tot[tid] = sum;
      if (p.totals) p.totals[tid] = static_cast<int64_t>(sum);
    }
    __syncthreads();
    if (tid == 0) {
      *p.err = atomicExch(p.ws_flag, 0);
      *p.done = 0;
    }
    if (p.corpus && tid < 32) {
      const int lane = tid;
      warp_epilogue(lane < N ? static_cast<int64_t>(s_tot[lane]) : 0,
                    lane < N ? static_cast<int64_t>(s_tot[N + lane]) : 0, static_cast<int64_t>(s_tot[2 * N]),
                    static_cast<int64_t>(s_tot[2 * N + 1]), N, p.smoothing, p.eps, p.k,
                    lane < N ? p.weights[lane] : 0.0, p.corpus + 2, p.corpus + 1, p.corpus);
    }
  }
}

// --------------------------------------------------------------------------
// The fused per-sentence-group kernel.
// --------------------------------------------------------------------------
template <typename T, bool kSmem>
__global__ void __launch_bounds__(kThreads)
    bleu_stats_kernel(const __grid_constant__ StatsParams p) {
  using W = typename Word<kSmem>::T;
  constexpr int kShift = Word<kSmem>::kShift;
  constexpr W kLow = (W(1) << kShift) - 1;

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int s_hits[TB_MAX_ORDER];
  __shared__ int64_t s_len[TB_MAX_REFS + 1];  // [0] candidate, [1 + r] reference r
  __shared__ const T* s_rows[TB_MAX_REFS];    // global mode: reference rows of this group
  __shared__ unsigned long long s_tot[2 * TB_MAX_ORDER + 2];
  __shared__ int s_last;
  __shared__ int s_flags;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int R = p.num_refs;
  const int N = p.max_order;
  const uint32_t cap = 1u << p.cap_log2;
  const uint32_t mask = cap - 1;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;

  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  T* s_cand = reinterpret_cast<T*>(smem + 16);
  T* s_ref = s_cand + p.cand_pad;
  int32_t* keys;
  W* words;
  if constexpr (kSmem) {
    keys = reinterpret_cast<int32_t*>(s_ref + p.ref_off[R]);
    words = reinterpret_cast<W*>(keys + cap);
  } else {
    unsigned char* g = p.gtab + static_cast<size_t>(blockIdx.x) * p.gtab_stride;
    words = reinterpret_cast<W*>(g);
    keys = reinterpret_cast<int32_t*>(g + static_cast<size_t>(cap) * sizeof(W));
  }
  griddep_wait_and_release();

  if (tid < 2 * N + 2) s_tot[tid] = 0;
  if (tid == 0) s_flags = 0;
  if constexpr (kSmem) {
    if (tid == 0) mbar_init(mbar, 1);
  }
  __syncthreads();

  uint32_t phase = 0;
  const T* cand_g_base = static_cast<const T*>(p.cand_ids);

  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    // ---- 1. lengths (validated; clamped so that nothing reads out of bounds)
    if (tid <= R) {
      int64_t len, width;
      if (tid == 0) {
        len = p.cand_len[b];
        width = p.cand_width;
      } else {
        len = p.refs[tid - 1].len[b];
        width = p.refs[tid - 1].width;
        if constexpr (!kSmem)
          s_rows[tid - 1] = static_cast<const T*>(p.refs[tid - 1].ids) + b * p.refs[tid - 1].ld;
      }
      if (len < 0 || len > width) {
        atomicOr(&s_flags, TB_FLAG_BAD_LENGTH);
        len = len < 0 ? 0 : width;
      }
      s_len[tid] = len;
    }
    if (tid < N) s_hits[tid] = 0;
    __syncthreads();

    // ---- 2. stage the group's valid tokens in shared memory (bulk async copy)
    if constexpr (kSmem) {
      if (tid == 0) {
        fence_proxy_async_smem();  // prior generic reads of the buffers before async writes
        uint32_t total = 0;
        for (int s = 0; s <= R; ++s) {
          const T* src = s == 0 ? cand_g_base + b * p.cand_ld
                                : static_cast<const T*>(p.refs[s - 1].ids) + b * p.refs[s - 1].ld;
          if ((reinterpret_cast<uintptr_t>(src) & 15) == 0)
            total += static_cast<uint32_t>((s_len[s] * sizeof(T)) & ~static_cast<int64_t>(15));
        }
        mbar_arrive_expect_tx(mbar, total);
        for (int s = 0; s <= R; ++s) {
          const T* src = s == 0 ? cand_g_base + b * p.cand_ld
                                : static_cast<const T*>(p.refs[s - 1].ids) + b * p.refs[s - 1].ld;
          T* dst = s == 0 ? s_cand : s_ref + p.ref_off[s - 1];
          const uint32_t bytes =
              static_cast<uint32_t>((s_len[s] * sizeof(T)) & ~static_cast<int64_t>(15));
          if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && bytes > 0) bulk_g2s(dst, src, bytes, mbar);
        }
      }
      // tails (< 16 B) and rows whose global address is not 16-B aligned
      for (int s = 0; s <= R; ++s) {
        const T* src = s == 0 ? cand_g_base + b * p.cand_ld
                              : static_cast<const T*>(p.refs[s - 1].ids) + b * p.refs[s - 1].ld;
        T* dst = s == 0 ? s_cand : s_ref + p.ref_off[s - 1];
        const int64_t len = s_len[s];
        const int64_t start = ((reinterpret_cast<uintptr_t>(src) & 15) == 0)
                                  ? static_cast<int64_t>(((len * sizeof(T)) & ~static_cast<int64_t>(15)) / sizeof(T))
                                  : 0;
        for (int64_t j = start + tid; j < len; j += kThreads) dst[j] = src[j];
      }
    }

    // ---- 3. clear the table for order 1 (overlaps the bulk copy)
    for (uint32_t s = tid; s < cap; s += kThreads) {
      keys[s] = -1;
      words[s] = 0;
    }
    if constexpr (kSmem) {
      mbar_wait(mbar, phase);
      phase ^= 1;
    }
    __syncthreads();

    RefTokens<T, kSmem> rt;
    rt.base = s_ref;
    rt.rows = s_rows;
    const T* cand = kSmem ? s_cand : cand_g_base + b * p.cand_ld;

    // ---- 4. per order: reference counting, max-fold, clipped candidate count
    for (int n = 1; n <= N; ++n) {
      if (n > 1) {
        for (uint32_t s = tid; s < cap; s += kThreads) {
          keys[s] = -1;
          words[s] = 0;
        }
        __syncthreads();
      }
      for (int r = 0; r < R; ++r) {
        const int64_t cnt = s_len[1 + r] - n + 1;
        const T* rrow = kSmem ? s_ref + p.ref_off[r] : s_rows[r];
        // R == 1: count straight into the "max" half (no fold needed)
        const W unit = (R == 1) ? (W(1) << kShift) : W(1);
        for (int64_t base = 0; base < cnt; base += kThreads) {
          const int64_t j = base + tid;
          int32_t slot = -1;
          if (j < cnt) slot = table_insert<T, kSmem>(keys, mask, rrow + j, n, rt.key(r, j, p.ref_off), rt);
          const unsigned act = __ballot_sync(kFull, slot >= 0);
          if (slot >= 0) {
            const unsigned peers = __match_any_sync(act, slot);
            if (lane == __ffs(peers) - 1) atomicAdd(&words[slot], unit * static_cast<W>(__popc(peers)));
          }
        }
        __syncthreads();
        if (R > 1) {  // fold: max(refmax, count_r) -> high half, reset running count
          for (uint32_t s = tid; s < cap; s += kThreads) {
            const W w = words[s];
            const W c = w & kLow;
            const W m = w >> kShift;
            if (c) words[s] = (c > m ? c : m) << kShift;
          }
          __syncthreads();
        }
      }
      // candidate pass: the old word carries (refmax, running count) -> clipped hit count
      {
        const int64_t cnt = s_len[0] - n + 1;
        unsigned int hits = 0;
        for (int64_t base = 0; base < cnt; base += kThreads) {
          const int64_t j = base + tid;
          int32_t slot = -1;
          if (j < cnt) slot = table_find<T, kSmem>(keys, mask, cand + j, n, rt);
          const unsigned act = __ballot_sync(kFull, slot >= 0);
          if (slot >= 0) {
            const unsigned peers = __match_any_sync(act, slot);
            if (lane == __ffs(peers) - 1) {
              const W k = static_cast<W>(__popc(peers));
              const W old = atomicAdd(&words[slot], k);
              const W oc = old & kLow;
              const W m = old >> kShift;
              const W avail = m > oc ? m - oc : 0;
              hits += static_cast<unsigned int>(avail < k ? avail : k);
            }
          }
        }
        hits = __reduce_add_sync(kFull, hits);
        if (lane == 0 && hits) atomicAdd(&s_hits[n - 1], hits);
      }
      __syncthreads();
    }

    // ---- 5. per-sentence epilogue
    if (tid == 0) {
      int64_t num[TB_MAX_ORDER], den[TB_MAX_ORDER];
      const int64_t c = s_len[0];
      for (int n = 0; n < N; ++n) {
        num[n] = s_hits[n];
        const int64_t d = c - n;  // max(len - (n+1) + 1, 0)
        den[n] = d > 0 ? d : 0;
        if (p.num) p.num[b * N + n] = num[n];
        if (p.den) p.den[b * N + n] = den[n];
      }
      const int64_t r = closest_ref_len(c, &s_len[1], R);
      if (p.cand_len_out) p.cand_len_out[b] = c;
      if (p.eff_ref) p.eff_ref[b] = r;
      if (p.scores || p.precisions || p.bp)
        bleu_epilogue(num, den, c, r, N, p.smoothing, p.eps, p.k, p.weights,
                      p.precisions ? p.precisions + b * N : nullptr, p.bp ? p.bp + b : nullptr,
                      p.scores ? p.scores + b : nullptr);
      if (corpus) {
        for (int n = 0; n < N; ++n) {
          s_tot[n] += static_cast<unsigned long long>(num[n]);
          s_tot[N + n] += static_cast<unsigned long long>(den[n]);
        }
        s_tot[2 * N] += static_cast<unsigned long long>(c);
        s_tot[2 * N + 1] += static_cast<unsigned long long>(r);
      }
    }
    __syncthreads();
  }

  finish_cta(p, s_tot, s_flags, s_last);
}

// --------------------------------------------------------------------------
// Pruned progressive kernel (shared-memory path).
//
// Only n-grams that can be in the clipped intersection are ever hashed:
//   * order 1: every candidate token is inserted (count kept in the entry),
//     every reference token is looked up;
//   * order n >= 2: a position is visited only if its (n-1)-gram matched the
//     other side at order n-1 (it is on that order's live list) and its last
//     token matched at order 1 — an n-gram occurring on both sides has both
//     properties, so skipping everything else is exact;
//   * order-n keys are (slot of the (n-1)-prefix, slot of the last token),
//     16 + 16 bits: one integer compare, no token re-reads (the progressive
//     packing of ngrams.py:144-198, restricted to the live set).
// Entry (64 bit): [key 32 | candidate count 16 | reference count 16]; a new
// key is inserted and counted with one CAS.  The numerator is the clipped
// intersection sum_g min(cand_g, max_r ref_{r,g}) (oracle.py:36-37).
// Live lists are built with warp-aggregated appends, so orders >= 2 cost
// time proportional to the matching n-grams only.
// --------------------------------------------------------------------------

// Debug-only phase timestamps (build with -DTB_PHASES; see tools/phase_profile.py)
#ifdef TB_PHASES
__device__ unsigned long long* g_tb_phases;
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
__device__ __forceinline__ void list_append(uint16_t* list, int* count, bool pred, int val) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(val);
}

// Lookup of `key` (order n >= 2 packed key, or a token at order 1) in the
// bucketed table.  A present key always sits in its home bucket unless that
// bucket was full when it was inserted, so a lookup stops at the first bucket
// with an empty entry.  The home slot is checked first (keys usually win their
// home slot), which makes most lookups a single 4-byte load.
template <typename EqF>
__device__ __forceinline__ int table_find(const uint32_t* ent, uint32_t home, uint32_t bmask, EqF eq) {
  const uint32_t e0 = ent[home];
  if (e0 == ~0u) return -1;
  if (eq(e0 >> 16)) return static_cast<int>(home);
  uint32_t bk = home >> 2;
  while (true) {
    const uint4 q = reinterpret_cast<const uint4*>(ent)[bk];
    const uint32_t e[4] = {q.x, q.y, q.z, q.w};
    bool full = true;
    int slot = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] == ~0u)
        full = false;
      else if (slot < 0 && 4 * bk + k != home && eq(e[k] >> 16))
        slot = static_cast<int>(4 * bk + k);
    }
    if (slot >= 0 || !full) return slot;
    bk = (bk + 1) & bmask;
  }
}

// Round 2 of the candidate insert for a position that lost its home slot to a
// different key: CAS into the first empty entry from the home bucket on, or add
// to an equal key inserted by another loser.
template <typename EqF>
__device__ __forceinline__ uint32_t table_insert_loser(uint32_t* ent, uint32_t home, uint32_t bmask,
                                                       uint32_t mine, EqF eq) {
  uint32_t bk = home >> 2;
  while (true) {
    uint4 q;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "r"(smem_u32(ent + 4 * bk)));
    const uint32_t e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = e[k];
      if (v == ~0u) {
        v = atomicCAS(&ent[4 * bk + k], ~0u, mine);
        if (v == ~0u) return 4 * bk + k;
      }
      if (eq(v >> 16)) {
        atomicAdd(&ent[4 * bk + k], 1u);
        return 4 * bk + k;
      }
    }
    bk = (bk + 1) & bmask;
  }
}

// reference-count half-words packed in u32 words (32-bit atomics only)
__device__ __forceinline__ void xc_add(uint32_t* xcw, int s) { atomicAdd(&xcw[s >> 1], 1u << ((s & 1) * 16)); }
__device__ __forceinline__ uint32_t xc_get(const uint32_t* xcw, int s) { return (xcw[s >> 1] >> ((s & 1) * 16)) & 0xffffu; }
__device__ __forceinline__ uint32_t xc_take(uint32_t* xcw, int s) {
  const uint32_t m = 0xffffu << ((s & 1) * 16);
  return (atomicAnd(&xcw[s >> 1], ~m) & m) >> ((s & 1) * 16);
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 4)
    bleu_group_kernel(const __grid_constant__ StatsParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int s_hits[TB_MAX_ORDER];
  __shared__ int64_t s_len[TB_MAX_REFS + 1];
  __shared__ int s_pos[TB_MAX_REFS + 1];  // position offset of row s (0 = candidate)
  __shared__ unsigned long long s_tot[2 * TB_MAX_ORDER + 2];
  __shared__ int s_last, s_flags;
  __shared__ int s_nlc[2], s_nins[2];    // candidate live / inserted list lengths (by order parity)
  __shared__ int s_nlr[2][TB_MAX_REFS];  // live reference list lengths
  __shared__ int64_t s_stage_len[TB_MAX_REFS + 1];  // prefix mode: lengths read by issue_rows

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int R = p.num_refs;
  const int N = p.max_order;
  const int cap_log2 = p.cap_log2;
  const uint32_t cap = 1u << cap_log2;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;

  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  T* tok = reinterpret_cast<T*>(smem + 16);
  uint16_t* id1 = reinterpret_cast<uint16_t*>(smem + p.off_id1);
  uint16_t* idn = reinterpret_cast<uint16_t*>(smem + p.off_idn);
  uint8_t* live = smem + p.off_live;
  uint32_t* ent = reinterpret_cast<uint32_t*>(smem + p.off_ent);   // [cand position 16 | cand count 16]
  uint32_t* xcw = ent + cap;                                        // reference counts, 16 bit, paired
  uint16_t* mref = reinterpret_cast<uint16_t*>(smem + p.off_mref);  // max over references (R > 1)
  uint32_t* kc = reinterpret_cast<uint32_t*>(smem + p.off_kc);      // order-n key of candidate positions
  uint16_t* lc = reinterpret_cast<uint16_t*>(smem + p.off_lists);   // candidate positions live at order n-1 / n
  const int cpad = p.cand_pad;
  const int rtot = p.ref_off[R];
  uint16_t* lins = lc + cpad;                                       // candidate positions inserted at order n
  uint16_t* lrbase = lc + 2 * cpad;                                 // reference lists, two parities
  const uint32_t hshift = 32 - cap_log2;  // home slot = top bits of the hash
  const uint32_t bmask = (cap >> 2) - 1;  // buckets of 4 slots (one 16-byte load)

  // Stage the rows of group b: bulk copies of the 16-byte-aligned body (full
  // width, or the valid prefix in prefix mode); the < 16-byte tails and rows
  // whose global address is unaligned are copied by the threads before the barrier.
  auto issue_stage = [&](int64_t b) {
    if (tid == 0) issue_rows<T>(p, b, R + 1, tok, mbar, s_stage_len, &s_flags);
  };

  if (tid < 2 * N + 2) s_tot[tid] = 0;
  if (tid <= R) s_pos[tid] = tid == 0 ? 0 : cpad + p.ref_off[tid - 1];
  if (tid == 0) {
    s_flags = 0;
    mbar_init(mbar, 1);
  }
  griddep_wait_and_release();
  if (static_cast<int64_t>(blockIdx.x) < p.batch) issue_stage(blockIdx.x);
  __syncthreads();
  TB_MARK(0);
  uint32_t phase = 0;

  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    // ---- lengths, per-group state (the token copy is already in flight)
    if (p.prefix_only) {
      __syncthreads();  // s_stage_len of this group, written by thread 0 in issue_rows
      if (tid <= R) s_len[tid] = s_stage_len[tid];
    } else if (tid <= R) {
      int64_t len, width;
      if (tid == 0) {
        len = p.cand_len[b];
        width = p.cand_width;
      } else {
        len = p.refs[tid - 1].len[b];
        width = p.refs[tid - 1].width;
      }
      if (len < 0 || len > width) {
        atomicOr(&s_flags, TB_FLAG_BAD_LENGTH);
        len = len < 0 ? 0 : width;
      }
      s_len[tid] = len;
    }
    if (tid < N) s_hits[tid] = 0;
    if (tid < 2) {
      s_nlc[tid] = 0;
      s_nins[tid] = 0;
    }
    if (tid < 2 * R) s_nlr[tid / R][tid % R] = 0;
    copy_row_tails<T>(p, b, R + 1, tok, s_stage_len, tid, kThreads);  // tails / unaligned rows
    // clear the table (entries EMPTY, reference counts 0); later orders clear only used slots
    for (uint32_t s = tid; s < cap / 4; s += kThreads) reinterpret_cast<uint4*>(ent)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (uint32_t s = tid; s < cap / 8; s += kThreads) {
      reinterpret_cast<uint4*>(xcw)[s] = make_uint4(0, 0, 0, 0);
      if (R > 1) reinterpret_cast<uint4*>(mref)[s] = make_uint4(0, 0, 0, 0);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    __syncthreads();
    TB_MARK(2);

    const int clen = static_cast<int>(s_len[0]);

    // ================= order 1: tokens =================
    {
      // P1 round 1: every candidate position stores itself into its token's home slot
      for (int j = tid; j < clen; j += kThreads) {
        const uint32_t home = tok_hash32(tok[j]) >> hshift;
        ent[home] = (static_cast<uint32_t>(j) << 16) | 1u;
      }
      __syncthreads();
      // P1 round 2: winners own their slot; equal tokens count; collisions probe
      for (int j = tid; j < clen; j += kThreads) {
        const T t = tok[j];
        const uint32_t home = tok_hash32(t) >> hshift;
        uint32_t slot = home;
        const uint32_t w = ent[home] >> 16;
        if (w != static_cast<uint32_t>(j)) {
          if (tok[w] == t)
            atomicAdd(&ent[home], 1u);
          else
            slot = table_insert_loser(ent, home, bmask, (static_cast<uint32_t>(j) << 16) | 1u,
                                      [&](uint32_t x) { return tok[x] == t; });
        }
        id1[j] = static_cast<uint16_t>(slot);
        idn[j] = static_cast<uint16_t>(slot);
      }
      __syncthreads();
      TB_MARK(3);
      // P2: reference tokens
      for (int r = 0; r < R; ++r) {
        const int off = s_pos[1 + r];
        const int rlen = static_cast<int>(s_len[1 + r]);
        uint16_t* lrout = lrbase + rtot + p.ref_off[r];  // parity 1
        for (int base = 0; base < rlen; base += kThreads) {
          const int i = base + tid;
          const int q = off + i;
          int slot = -1;
          if (i < rlen) {
            const T t = tok[q];
            slot = table_find(ent, tok_hash32(t) >> hshift, bmask, [&](uint32_t x) { return tok[x] == t; });
            if (slot >= 0) {
              xc_add(xcw, slot);
              id1[q] = static_cast<uint16_t>(slot);
              idn[q] = static_cast<uint16_t>(slot);
            }
            live[q] = slot >= 0 ? 1 : 0;
          }
          list_append(lrout, &s_nlr[1][r], slot >= 0, q);
        }
        __syncthreads();
        if (R > 1) {
          const int nf = s_nlr[1][r];
          for (int i = tid; i < nf; i += kThreads) {
            const int s = id1[lrout[i]];
            const uint32_t x = xc_take(xcw, s);
            if (x > mref[s]) mref[s] = static_cast<uint16_t>(x);
          }
          __syncthreads();
        }
      }
      TB_MARK(4);
      // P3: candidate liveness + clipped count (added once per slot by its owner)
      unsigned int hits = 0;
      for (int base = 0; base < clen; base += kThreads) {
        const int j = base + tid;
        bool ok = false;
        if (j < clen) {
          const int s = id1[j];
          const uint32_t e = ent[s];
          const uint32_t m = (R == 1) ? xc_get(xcw, s) : mref[s];
          ok = m != 0;
          if ((e >> 16) == static_cast<uint32_t>(j)) {
            const uint32_t c = e & 0xffffu;
            hits += c < m ? c : m;
          }
          live[j] = ok ? 1 : 0;
        }
        list_append(lc, &s_nlc[1], ok, j);
      }
      hits = __reduce_add_sync(kFull, hits);
      if (lane == 0 && hits) atomicAdd(&s_hits[0], hits);
      __syncthreads();
      TB_MARK(5);
    }

    // ================= orders n >= 2: packed (prefix slot, last-token slot) keys =================
    for (int n = 2; n <= N; ++n) {
      const int par = n & 1;
      const int nlive = s_nlc[par ^ 1];
      if (nlive == 0) break;  // no candidate (n-1)-gram matched: orders >= n have no hits
      // P0: clear the slots used at order n-1, compute this order's candidate keys
      {
        const int cnt = n == 2 ? clen : s_nins[par ^ 1];
        for (int i = tid; i < cnt; i += kThreads) {
          const int s = n == 2 ? id1[i] : idn[lins[i]];
          ent[s] = ~0u;
          reinterpret_cast<uint16_t*>(xcw)[s] = 0;  // half-word s of the paired counts
          if (R > 1) mref[s] = 0;
        }
        for (int i = tid; i < nlive; i += kThreads) {
          const int j = lc[i];
          const bool el = j + n - 1 < clen && live[j + n - 1] >= 1;
          kc[j] = el ? ((static_cast<uint32_t>(idn[j]) << 16) | id1[j + n - 1]) : ~0u;
        }
        if (tid == 0) s_nins[par] = 0;
        if (tid < R) s_nlr[par][tid] = 0;
        __syncthreads();
      }
      // P1 round 1
      for (int i = tid; i < nlive; i += kThreads) {
        const int j = lc[i];
        const uint32_t key = kc[j];
        if (key != ~0u) ent[(key * 0x9E3779B1u) >> hshift] = (static_cast<uint32_t>(j) << 16) | 1u;
      }
      __syncthreads();
      // P1 round 2 (+ inserted list)
      for (int base = 0; base < nlive; base += kThreads) {
        const int i = base + tid;
        int j = 0;
        bool el = false;
        if (i < nlive) {
          j = lc[i];
          const uint32_t key = kc[j];
          el = key != ~0u;
          if (el) {
            const uint32_t home = (key * 0x9E3779B1u) >> hshift;
            uint32_t slot = home;
            const uint32_t w = ent[home] >> 16;
            if (w != static_cast<uint32_t>(j)) {
              if (kc[w] == key)
                atomicAdd(&ent[home], 1u);
              else
                slot = table_insert_loser(ent, home, bmask, (static_cast<uint32_t>(j) << 16) | 1u,
                                          [&](uint32_t x) { return kc[x] == key; });
            }
            idn[j] = static_cast<uint16_t>(slot);
          }
        }
        list_append(lins, &s_nins[par], el, j);
      }
      if (tid == 0) s_nlc[par] = 0;  // lc is consumed; it is rebuilt in P3
      __syncthreads();
      // P2: live reference positions
      for (int r = 0; r < R; ++r) {
        const int off = s_pos[1 + r];
        const int rlen = static_cast<int>(s_len[1 + r]);
        uint16_t* lrin = lrbase + (par ^ 1) * rtot + p.ref_off[r];
        uint16_t* lrout = lrbase + par * rtot + p.ref_off[r];
        const int cnt = s_nlr[par ^ 1][r];
        for (int base = 0; base < cnt; base += kThreads) {
          const int i = base + tid;
          int q = 0;
          int slot = -1;
          if (i < cnt) {
            q = lrin[i];
            if (q - off + n - 1 < rlen && live[q + n - 1] >= 1) {
              const uint32_t key = (static_cast<uint32_t>(idn[q]) << 16) | id1[q + n - 1];
              slot = table_find(ent, (key * 0x9E3779B1u) >> hshift, bmask, [&](uint32_t x) { return kc[x] == key; });
              if (slot >= 0) {
                xc_add(xcw, slot);
                idn[q] = static_cast<uint16_t>(slot);
                live[q] = static_cast<uint8_t>(n);
              }
            }
          }
          list_append(lrout, &s_nlr[par][r], slot >= 0, q);
        }
        __syncthreads();
        if (R > 1) {
          const int nf = s_nlr[par][r];
          for (int i = tid; i < nf; i += kThreads) {
            const int s = idn[lrout[i]];
            const uint32_t x = xc_take(xcw, s);
            if (x > mref[s]) mref[s] = static_cast<uint16_t>(x);
          }
          __syncthreads();
        }
      }
      // P3
      {
        const int cnt = s_nins[par];
        unsigned int hits = 0;
        for (int base = 0; base < cnt; base += kThreads) {
          const int i = base + tid;
          bool ok = false;
          int j = 0;
          if (i < cnt) {
            j = lins[i];
            const int s = idn[j];
            const uint32_t e = ent[s];
            const uint32_t m = (R == 1) ? xc_get(xcw, s) : mref[s];
            ok = m != 0;
            if ((e >> 16) == static_cast<uint32_t>(j)) {
              const uint32_t c = e & 0xffffu;
              hits += c < m ? c : m;
            }
            if (ok) live[j] = static_cast<uint8_t>(n);
          }
          list_append(lc, &s_nlc[par], ok, j);
        }
        hits = __reduce_add_sync(kFull, hits);
        if (lane == 0 && hits) atomicAdd(&s_hits[n - 1], hits);
      }
      __syncthreads();
      TB_MARK(3 + 4 * (n - 1) + 3);
    }

    // ---- epilogue (warp 0)
    if (tid < 32) {
      const int64_t c = s_len[0];
      const int64_t num = lane < N ? static_cast<int64_t>(s_hits[lane]) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      if (lane < N) {
        if (p.num) p.num[b * N + lane] = num;
        if (p.den) p.den[b * N + lane] = den;
      }
      const int64_t r = closest_ref_len(c, &s_len[1], R);
      if (lane == 0) {
        if (p.cand_len_out) p.cand_len_out[b] = c;
        if (p.eff_ref) p.eff_ref[b] = r;
      }
      if (p.scores || p.precisions || p.bp)
        warp_epilogue(num, den, c, r, N, p.smoothing, p.eps, p.k, lane < N ? p.weights[lane] : 0.0,
                      p.precisions ? p.precisions + b * N : nullptr, p.bp ? p.bp + b : nullptr,
                      p.scores ? p.scores + b : nullptr);
      if (corpus) {
        if (lane < N) {
          s_tot[lane] += static_cast<unsigned long long>(num);
          s_tot[N + lane] += static_cast<unsigned long long>(den);
        }
        if (lane == 0) {
          s_tot[2 * N] += static_cast<unsigned long long>(c);
          s_tot[2 * N + 1] += static_cast<unsigned long long>(r);
        }
      }
    }
    __syncthreads();
    TB_MARK(30);
    if (b + gridDim.x < p.batch) issue_stage(b + gridDim.x);
  }
  finish_cta(p, s_tot, s_flags, s_last);
  TB_MARK(31);
}

// --------------------------------------------------------------------------
// Single-reference kernel (R == 1, the headline configuration).
//
// Order 1: a blocked two-bit Bloom filter per side (in the table + count
// region) drops the tokens absent from the other side; when <= kSmallSet
// positions survive (unrelated text) they are matched exactly without a
// table.  Otherwise only CANDIDATE tokens are inserted, store-then-verify:
//   claim:  every candidate position stores itself (u16) into its token's
//           home slot — plain stores, one wins;
//   verify: the winner owns the slot (its own occurrence is counted
//           implicitly); an equal token adds one to the owner's count word
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
template <int NT = kThreads, typename HashF, typename EqF>
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
    if (!__syncthreads_or(left)) return;
  }
  for (int i = tid; i < nl; i += NT) {
    const uint16_t pos = lost[i];
    if (pos == 0xffffu) continue;
    ids[pos] = static_cast<uint16_t>(pair_insert_loser(own, cnt, ids[pos], mask, pos, pos < roff ? 1u : (1u << 16),
                                                       [&](uint16_t x) { return eq(pos, x); }));
  }
  __syncthreads();
}

// pair_resolve_lost for the live-list passes of orders >= 2: `lost` holds list
// indices e (owners are list indices, keys kc[e], hash key * 0x9E3779B1), all of
// candidate entries; settling e writes its owner's list index to idn[lin[e]].
template <int NT = kThreads>
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
    if (!__syncthreads_or(left)) return;
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
  __syncthreads();
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

template <typename T>
__global__ void __launch_bounds__(kThreads, 4)
    bleu_pair_kernel(const __grid_constant__ StatsParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int s_hits[TB_MAX_ORDER];
  __shared__ int64_t s_len[2];
  __shared__ unsigned long long s_tot[2 * TB_MAX_ORDER + 2];
  __shared__ int s_last, s_flags;
  __shared__ int s_nlost, s_nc, s_nr, s_ndef, s_nf;  // s_nc / s_nr: live candidate / reference entries
  __shared__ uint16_t s_flist[kSmallSet];  // positions that pass the order-1 filter
  __shared__ int64_t s_stage_len[2];  // prefix mode: lengths read by issue_rows
  __shared__ double s_bp;             // brevity penalty of the current group

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int N = p.max_order;
  const int cap_log2 = p.cap_log2;
  const uint32_t cap = 1u << cap_log2;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  const int cpad = p.cand_pad;
  const int roff = cpad;  // first reference position (multiple of 4)

  uint64_t* mbars = reinterpret_cast<uint64_t*>(smem);  // one mbarrier per token buffer
  T* const tokb[2] = {reinterpret_cast<T*>(smem + 16), reinterpret_cast<T*>(smem + p.off_tok2)};
  const bool dbuf = p.off_tok2 != 0;  // prefetch the next group into the other buffer
  int cur = 0;
  T* tok = tokb[0];
  uint32_t* kc = reinterpret_cast<uint32_t*>(tok);                 // aliases tok (orders >= 2)
  uint16_t* id1 = reinterpret_cast<uint16_t*>(smem + p.off_id1);   // order-1 slot; 0xffff: token unmatched
  uint16_t* idn = reinterpret_cast<uint16_t*>(smem + p.off_idn);   // order-n slot; 0xffff: n-gram unmatched
  uint16_t* own = reinterpret_cast<uint16_t*>(smem + p.off_ent);   // slot -> owner position, 0xffff = empty
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + p.off_mref);  // owner -> [ref 16 | cand 16], owner excluded
  // two position lists of ptot entries: the live positions of an order (input of
  // the next; candidate positions from index 0, reference positions from index
  // roff) and, in the other, the lost (from 0) / deferred (from roff) entries of
  // the current order.  Owners are always candidate entries: cnt has cand_pad words.
  const int ptot = roff + p.ref_off[1];
  uint16_t* const lx = reinterpret_cast<uint16_t*>(smem + p.off_lists);
  uint16_t* const ly = lx + ptot;
  const uint32_t hshift = 32 - cap_log2;
  const uint32_t mask = cap - 1;

  auto issue_stage = [&](int64_t b, int buf) {
    if (tid == 0) issue_rows<T>(p, b, 2, tokb[buf], mbars + buf, s_stage_len, &s_flags);
  };

  if (tid < 2 * N + 2) s_tot[tid] = 0;
  if (tid == 0) {
    s_flags = 0;
    mbar_init(mbars, 1);
    if (dbuf) mbar_init(mbars + 1, 1);
  }
  griddep_wait_and_release();
  if (static_cast<int64_t>(blockIdx.x) < p.batch) issue_stage(blockIdx.x, 0);
  __syncthreads();
  TB_MARK(0);
  uint32_t phases = 0;  // bit i: parity of mbarrier i
  bool try_filter = true;  // off after a group of this CTA needed the hash passes (related text)

  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    tok = tokb[cur];
    kc = reinterpret_cast<uint32_t*>(tok);
    if (p.prefix_only) {
      __syncthreads();  // s_stage_len of this group, written by thread 0 in issue_rows
      if (tid < 2) s_len[tid] = s_stage_len[tid];
    } else if (tid < 2) {
      const int64_t len = tid == 0 ? p.cand_len[b] : p.refs[0].len[b];
      const int64_t width = tid == 0 ? p.cand_width : p.refs[0].width;
      int64_t l = len;
      if (len < 0 || len > width) {
        atomicOr(&s_flags, TB_FLAG_BAD_LENGTH);
        l = len < 0 ? 0 : width;
      }
      s_len[tid] = l;
    }
    if (tid < N) s_hits[tid] = 0;
    if (tid == 0) {
      s_nlost = 0;
      s_nc = 0;
      s_nr = 0;
      s_ndef = 0;
      s_nf = 0;
    }
    copy_row_tails<T>(p, b, 2, tok, s_stage_len, tid, kThreads);  // tails / unaligned rows
    // the table region starts as the two filter bitmaps (zero; they extend over
    // the count array) or as the empty table
    if (try_filter) {
      for (uint32_t s = tid; s < (1u << p.filter_log2) / 2; s += kThreads)
        reinterpret_cast<uint4*>(own)[s] = make_uint4(0, 0, 0, 0);
    } else {
      for (uint32_t s = tid; s < cap / 8; s += kThreads)
        reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    mbar_wait(mbars + cur, (phases >> cur) & 1u);
    phases ^= 1u << cur;
    __syncthreads();
    // every thread is past the previous group: its buffer takes the next group
    if (dbuf && b + gridDim.x < p.batch) issue_stage(b + gridDim.x, cur ^ 1);
    TB_MARK(2);

    const int clen = static_cast<int>(s_len[0]);
    const int rlen = static_cast<int>(s_len[1]);
    // positions are processed in quads (4 consecutive positions of one row)
    const int ncq = (clen + 3) >> 2;
    const int nq = ncq + ((rlen + 3) >> 2);
    // quad -> (first position, mask of valid positions)
    auto quad = [&](int qi, int& p0) -> uint32_t {
      int left;
      if (qi < ncq) {
        p0 = 4 * qi;
        left = clen - p0;
      } else {
        p0 = roff + 4 * (qi - ncq);
        left = rlen - (p0 - roff);
      }
      return left >= 4 ? 0xfu : ((1u << left) - 1u);
    };
    auto load4 = [&](int pos, T (&t)[4]) {
      if constexpr (sizeof(T) == 4) {
        const int4 v = *reinterpret_cast<const int4*>(tok + pos);
        t[0] = v.x;
        t[1] = v.y;
        t[2] = v.z;
        t[3] = v.w;
      } else {
        const longlong2 u = *reinterpret_cast<const longlong2*>(tok + pos);
        const longlong2 v = *reinterpret_cast<const longlong2*>(tok + pos + 2);
        t[0] = u.x;
        t[1] = u.y;
        t[2] = v.x;
        t[3] = v.y;
      }
    };
    auto inc_of = [&](int pos) { return pos < roff ? 1u : (1u << 16); };

    // ================= order 1: filter =================
    // Each side marks its tokens in a blocked two-bit Bloom filter (the table
    // region: a 32-bit word per 4 slots per side, both bits of a token in one
    // word); a token not in the other side's filter cannot match (false
    // positives ~0.1% at the table's load).  When at most kSmallSet positions pass (unrelated
    // text: the ~1% that match plus ~1% false positives), their tokens are
    // matched exactly among themselves — one warp with match.any up to 32, the
    // block by direct comparison up to kSmallSet — and the hash passes below are
    // skipped.  Otherwise (related text) the table is reset and they run.
    bool filtered = false;
    if (try_filter) {
      // blocked: both bits of a token in one 32-bit word (one atomic / one load)
      uint32_t* bmc = reinterpret_cast<uint32_t*>(own);  // candidate tokens
      uint32_t* bmr = bmc + (1u << p.filter_log2);        // reference tokens
      const uint32_t wshift = 32 - p.filter_log2;
      auto fmask = [](uint32_t h) {
        const uint32_t g = h * 0x85EBCA6Bu;
        return (1u << (g >> 27)) | (1u << ((g >> 22) & 31u));
      };
      for (int qi = tid; qi < nq; qi += kThreads) {
        int p0;
        const uint32_t vm = quad(qi, p0);
        T t[4];
        load4(p0, t);
        uint32_t* bm = p0 < roff ? bmc : bmr;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (vm >> k & 1u) {
            const uint32_t h = tok_hash32(t[k]);
            atomicOr(&bm[h >> wshift], fmask(h));
          }
      }
      __syncthreads();
      TB_MARK(20);
      for (int qi = tid; qi < nq; qi += kThreads) {
        int p0;
        const uint32_t vm = quad(qi, p0);
        T t[4];
        load4(p0, t);
        const uint32_t* bm = p0 < roff ? bmr : bmc;  // the other side's
        uint32_t pm = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (vm >> k & 1u) {
            const uint32_t h = tok_hash32(t[k]);
            const uint32_t m = fmask(h);
            if ((bm[h >> wshift] & m) == m) pm |= 1u << k;
          }
        // every valid position starts "unmatched" at order 1 (the exact match below
        // marks the matched ones)
        *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);
        *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
        for (; pm; pm &= pm - 1) {
          const int j = atomicAdd(&s_nf, 1);
          if (j < kSmallSet) s_flist[j] = static_cast<uint16_t>(p0 + __ffs(pm) - 1);
        }
      }
      __syncthreads();
      TB_MARK(21);
      TB_NOTE(25, s_nf);
      const int S = s_nf;
      if (S <= kSmallSet && tid == kThreads - 32)  // the last warp is idle below
        s_bp = brevity_penalty_fp64(s_len[0], s_len[1]);
      if (S <= 32) {
        filtered = true;
        if (tid < 32) {  // exact order-1 match of the S listed positions
          const int pos = lane < S ? static_cast<int>(s_flist[lane]) : -1;
          const T t = pos >= 0 ? tok[pos] : T(0);
          const unsigned peers = __match_any_sync(kFull, pos >= 0 ? t : static_cast<T>(-1 - lane));
          const unsigned c = __popc(peers & __ballot_sync(kFull, pos >= 0 && pos < roff));
          const unsigned x = __popc(peers & __ballot_sync(kFull, pos >= roff));
          const int leader = __ffs(peers) - 1;
          unsigned h = (pos >= 0 && lane == leader) ? (c < x ? c : x) : 0u;
          h = __reduce_add_sync(kFull, h);
          const bool live = pos >= 0 && (pos < roff ? x > 0 : c > 0);
          if (live) {
            id1[pos] = static_cast<uint16_t>(leader);
            idn[pos] = static_cast<uint16_t>(leader);
          }
          const unsigned lc = __ballot_sync(kFull, live && pos < roff);
          const unsigned lr = __ballot_sync(kFull, live && pos >= roff);
          const unsigned below = (1u << lane) - 1u;
          if (live) lx[pos < roff ? __popc(lc & below) : roff + __popc(lr & below)] = static_cast<uint16_t>(pos);
          if (lane == 0) {
            s_hits[0] = h;
            s_nc = __popc(lc);
            s_nr = __popc(lr);
          }
        }
      } else if (S <= kSmallSet) {
        filtered = true;  // the block compares the S listed tokens directly
        const int pos = tid < S ? static_cast<int>(s_flist[tid]) : -1;
        bool live = false;
        if (pos >= 0) {
          const T t = tok[pos];
          unsigned c = 0, x = 0;
          int leader = tid;
          for (int j = 0; j < S; ++j) {
            const int q = s_flist[j];
            if (tok[q] != t) continue;
            leader = j < leader ? j : leader;
            if (q < roff) ++c; else ++x;
          }
          if (leader == tid) {
            const unsigned h = c < x ? c : x;
            if (h) atomicAdd(&s_hits[0], h);
          }
          live = pos < roff ? x > 0 : c > 0;
          if (live) {
            id1[pos] = static_cast<uint16_t>(leader);
            idn[pos] = static_cast<uint16_t>(leader);
            if (pos < roff) lx[atomicAdd(&s_nc, 1)] = static_cast<uint16_t>(pos);
            else lx[roff + atomicAdd(&s_nr, 1)] = static_cast<uint16_t>(pos);
          }
        }
      } else {  // related text: reset the table region for the hash passes
        for (uint32_t s = tid; s < cap / 8; s += kThreads)
          reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
        try_filter = false;  // uniform across the CTA (S is)
      }
      __syncthreads();
      TB_MARK(22);
    }

    if (__builtin_expect(!filtered, 0)) {  // (unlikely: keeps the filter path's code contiguous)
    // ================= order 1: tokens =================
    // Only candidate tokens are inserted (store-then-verify); reference tokens
    // look up: a reference token absent from the candidate can neither be
    // counted (min(c, 0) = 0) nor start a matching n-gram.  Owners are
    // therefore always candidate positions, and the table holds <= clen keys.
    const int nrq = nq - ncq;
    for (int qi = tid; qi < ncq; qi += kThreads) {  // round 1: claim home slots (plain stores)
      const int p0 = 4 * qi;
      const uint32_t vm = clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u);
      T t[4];
      load4(p0, t);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (vm >> k & 1u) own[tok_hash32(t[k]) >> hshift] = static_cast<uint16_t>(p0 + k);
      *reinterpret_cast<uint4*>(cnt + p0) = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    TB_MARK(28);
    for (int qi = tid; qi < ncq; qi += kThreads) {  // round 2: verify
      const int p0 = 4 * qi;
      const uint32_t vm = clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u);
      T t[4];
      load4(p0, t);
      uint32_t hv[4], home[4];
      uint16_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        hv[k] = tok_hash32(t[k]);
        home[k] = hv[k] >> hshift;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = own[home[k]];
      uint32_t lm = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int pos = p0 + k;
        if ((vm >> k & 1u) && w[k] != pos) {
          if (tok[w[k]] == t[k]) {
            atomicAdd(&cnt[w[k]], 1u);
          } else {
            lm |= 1u << k;
            pair_retry_store(own, hv[k], 1, hshift, static_cast<uint16_t>(pos));
          }
        }
      }
      *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(home[0] | (home[1] << 16), home[2] | (home[3] << 16));
      for (; lm; lm &= lm - 1) ly[atomicAdd(&s_nlost, 1)] = static_cast<uint16_t>(p0 + __ffs(lm) - 1);
    }
    // the brevity penalty depends on the lengths only: the last warp (idle in the
    // candidate passes unless the candidate has > 7/8 * 4 * blockDim tokens)
    // computes it here, off the critical path of the epilogue
    if (tid == kThreads - 32) s_bp = brevity_penalty_fp64(s_len[0], s_len[1]);
    __syncthreads();
    TB_MARK(29);
    TB_NOTE(27, s_nlost);
    {
      // One pass: retry round 1 of the lost candidate positions (verify half,
      // plus the store half of round 2) together with the home-slot lookups of
      // every reference position.  A lookup is final when the home slot is
      // EMPTY (the token has no candidate occurrence: lost keys never have an
      // empty home) or holds the same token (home owners are fixed since
      // round 1); a home held by a different token is deferred until the
      // retry rounds have settled.  The store halves only fill EMPTY slots,
      // and a home read EMPTY here stays conclusive for that token.
      const int nl = s_nlost;
      uint16_t* const lost = ly;
      uint16_t* const defl = ly + roff;  // deferred reference positions (capacity: padded ref width)
      auto hash1 = [&](uint16_t q) { return tok_hash32(tok[q]); };
      auto eq1 = [&](uint16_t a, uint16_t b) { return tok[a] == tok[b]; };
      int left = 0;
      for (int i = tid; i < nl; i += kThreads) {
        const uint16_t pos = lost[i];
        const uint32_t h = hash1(pos);
        const uint32_t cs = rehash(h, 1, hshift);
        const uint16_t w = own[cs];
        if (w == pos || eq1(pos, w)) {
          if (w != pos) atomicAdd(&cnt[w], 1u);
          id1[pos] = static_cast<uint16_t>(cs);
          lost[i] = 0xffffu;
        } else {
          left = 1;
          pair_retry_store(own, h, 2, hshift, pos);
        }
      }
      for (int q0 = 0; q0 < nrq; q0 += kThreads) {  // reference lookups (home slots)
        const int qi = q0 + tid;
        const int p0 = roff + 4 * qi;
        uint32_t fm = 0;  // found: live at order 1
        if (qi < nrq) {
        const uint32_t vm = roff + rlen - p0 >= 4 ? 0xfu : ((1u << (roff + rlen - p0)) - 1u);
        T t[4];
        load4(p0, t);
        uint32_t v[4];
        uint16_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = tok_hash32(t[k]) >> hshift;
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = (vm >> k & 1u) ? own[v[k]] : static_cast<uint16_t>(0xffffu);
        T to[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) to[k] = o[k] != 0xffffu ? tok[o[k]] : t[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (o[k] != 0xffffu && to[k] != t[k]) {  // home held by another token: later
            defl[atomicAdd(&s_ndef, 1)] = static_cast<uint16_t>(p0 + k);
            o[k] = 0xffffu;
          }
          if (o[k] == 0xffffu) {
            v[k] = 0xffffu;
          } else {
            atomicAdd(&cnt[o[k]], 1u << 16);
            fm |= 1u << k;
          }
        }
        const uint2 vv = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
        *reinterpret_cast<uint2*>(id1 + p0) = vv;  // 0xffff: token absent from the candidate
        *reinterpret_cast<uint2*>(idn + p0) = vv;
        }
        warp_append_quad(lx + roff, &s_nr, fm, [&](int k) { return p0 + k; }, lane);
      }
      if (__syncthreads_or(left))
        pair_resolve_lost(own, cnt, lost, nl, id1, mask, hshift, roff, tid, hash1, eq1, 2);
      TB_MARK(3);
      const int nd = s_ndef;
      for (int i0 = 0; i0 < nd; i0 += kThreads) {  // deferred lookups: the full chain
        const int i = i0 + tid;
        bool f = false;
        int pos = 0;
        if (i < nd) {
          pos = defl[i];
          const T t = tok[pos];
          uint16_t o;
          const int sl = pair_find_retry(own, tok, t, tok_hash32(t), hshift, mask, &o);
          if (sl >= 0) {
            atomicAdd(&cnt[o], 1u << 16);
            id1[pos] = static_cast<uint16_t>(sl);
            idn[pos] = static_cast<uint16_t>(sl);
            f = true;
          }
        }
        warp_append(lx + roff, &s_nr, f, pos, lane);
      }
    }
    __syncthreads();
    TB_MARK(26);
    {  // candidate liveness + clipped count (added once per slot by its owner)
      unsigned int hits = 0;
      for (int q0 = 0; q0 < ncq; q0 += kThreads) {
        const int qi = q0 + tid;
        const int p0 = 4 * qi;
        uint32_t lm = 0;
        if (qi < ncq) {
        const uint32_t vm = clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u);
        const uint2 s2 = *reinterpret_cast<const uint2*>(id1 + p0);
        const uint32_t s[4] = {s2.x & 0xffffu, s2.x >> 16, s2.y & 0xffffu, s2.y >> 16};
        uint32_t o[4], cw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = own[s[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) cw[k] = cnt[(vm >> k & 1u) ? o[k] : 0u];
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int pos = p0 + k;
          v[k] = 0xffffu;
          if (vm >> k & 1u) {
            const uint32_t c = (cw[k] & 0xffffu) + 1u;  // the owner counts itself
            const uint32_t x = cw[k] >> 16;
            if (o[k] == static_cast<uint32_t>(pos)) hits += c < x ? c : x;
            if (x != 0) {
              v[k] = s[k];
              lm |= 1u << k;
            }
          }
        }
        const uint2 vv = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
        *reinterpret_cast<uint2*>(id1 + p0) = vv;  // 0xffff: token unmatched, no n-gram can contain it
        *reinterpret_cast<uint2*>(idn + p0) = vv;
        }
        warp_append_quad(lx, &s_nc, lm, [&](int k) { return p0 + k; }, lane);
      }
      hits = __reduce_add_sync(kFull, hits);
      if (lane == 0 && hits) atomicAdd(&s_hits[0], hits);
    }
    __syncthreads();
    }
    TB_MARK(4);
    int nc = s_nc, nr = s_nr;

    // ================= orders n >= 2 =================
    // The live positions of order n-1 (list lin, nsurv entries; idn[pos]: id of
    // pos's (n-1)-gram, canonical within that order) form the keys of order n:
    // (idn[pos] << 16 | id1[pos + n - 1]).  While more than 32 stay live, one
    // table pass per order over the LIST (not all positions): candidate keys
    // claim, candidate entries verify and reference entries look up (like order
    // 1), then the live pass adds the clipped counts, appends the survivors to
    // the other list and clears the table for the next order.  Owners, counts
    // and ids are list indices (kc[i], cnt[i]).  With at most 32 live, warp 0
    // finishes the remaining orders with match.any (no table, no barriers).
    uint16_t* lin = lx;
    uint16_t* lout = ly;
    int n = 2;
    bool cleared = false;  // own[] still holds order 1's table (or the filter bitmaps)
    while (__builtin_expect(n <= N && nc > 0 && nc + nr > 32, 0)) {
      // entry quads: candidate entries [0, nc) then reference entries [roff, roff + nr)
      const int mcq = (nc + 3) >> 2;
      const int mq = mcq + ((nr + 3) >> 2);
      auto equad = [&](int qi, int& i0) -> uint32_t {
        int left;
        if (qi < mcq) {
          i0 = 4 * qi;
          left = nc - i0;
        } else {
          i0 = roff + 4 * (qi - mcq);
          left = nr - (i0 - roff);
        }
        return left >= 4 ? 0xfu : ((1u << left) - 1u);
      };
      auto lpos = [&](int i0, int (&pos)[4]) {
        const uint2 l2 = *reinterpret_cast<const uint2*>(lin + i0);
        pos[0] = l2.x & 0xffffu;
        pos[1] = l2.x >> 16;
        pos[2] = l2.y & 0xffffu;
        pos[3] = l2.y >> 16;
      };
      if (!cleared)
        for (uint32_t s = tid; s < cap / 8; s += kThreads)
          reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
      for (int qi = tid; qi < mq; qi += kThreads) {  // keys (~0: dead), counts, candidate claims
        int i0;
        const uint32_t vm = equad(qi, i0);
        int pos[4];
        lpos(i0, pos);
        const int end = i0 < roff ? clen : roff + rlen;
        uint32_t key[4];
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          key[k] = ~0u;
          const int q = pos[k] + n - 1;
          if ((vm >> k & 1u) && q < end) {
            const uint16_t l = id1[q];
            if (l != 0xffffu) key[k] = (static_cast<uint32_t>(idn[pos[k]]) << 16) | l;
          }
        }
        *reinterpret_cast<uint4*>(kc + i0) = make_uint4(key[0], key[1], key[2], key[3]);
        if (i0 < roff) {
          *reinterpret_cast<uint4*>(cnt + i0) = make_uint4(0, 0, 0, 0);
          if (cleared) {
  #pragma unroll
            for (int k = 0; k < 4; ++k)
              if (key[k] != ~0u) own[(key[k] * 0x9E3779B1u) >> hshift] = static_cast<uint16_t>(i0 + k);
          }
        }
      }
      if (tid == 0) {
        s_nlost = 0;
        s_ndef = 0;
      }
      __syncthreads();
      if (!cleared) {
        for (int qi = tid; qi < mcq; qi += kThreads) {
          const int i0 = 4 * qi;
          const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
          const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
  #pragma unroll
          for (int k = 0; k < 4; ++k)
            if (key[k] != ~0u) own[(key[k] * 0x9E3779B1u) >> hshift] = static_cast<uint16_t>(i0 + k);
        }
        __syncthreads();
      }
      if (tid == 0) {  // every thread has read them (barrier above)
        s_nc = 0;
        s_nr = 0;
      }
      uint16_t* const defl = lout + roff;  // deferred reference entries (lost candidates from 0)
      for (int qi = tid; qi < mq; qi += kThreads) {  // verify (candidates) / home lookups (references)
        int i0;
        equad(qi, i0);
        int pos[4];
        lpos(i0, pos);
        const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
        const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
        uint16_t w[4];
  #pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = key[k] != ~0u ? own[(key[k] * 0x9E3779B1u) >> hshift] : 0xffffu;
        uint32_t kw[4];
  #pragma unroll
        for (int k = 0; k < 4; ++k) kw[k] = w[k] != 0xffffu ? kc[w[k]] : ~0u;
        if (i0 < roff) {
  #pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (key[k] == ~0u) continue;
            const int i = i0 + k;
            if (w[k] == i) {
              idn[pos[k]] = static_cast<uint16_t>(i);
            } else if (kw[k] == key[k]) {
              atomicAdd(&cnt[w[k]], 1u);
              idn[pos[k]] = w[k];
            } else {
              lout[atomicAdd(&s_nlost, 1)] = static_cast<uint16_t>(i);
              pair_retry_store(own, key[k] * 0x9E3779B1u, 1, hshift, static_cast<uint16_t>(i));
            }
          }
        } else {
  #pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (key[k] == ~0u) continue;
            const int i = i0 + k;
            if (w[k] == 0xffffu) {  // empty home: no candidate n-gram has this key
              kc[i] = ~0u;
            } else if (kw[k] == key[k]) {
              atomicAdd(&cnt[w[k]], 1u << 16);
              idn[pos[k]] = w[k];
            } else {
              defl[atomicAdd(&s_ndef, 1)] = static_cast<uint16_t>(i);
            }
          }
        }
      }
      __syncthreads();
      if (s_nlost) list_resolve_lost(own, cnt, kc, lout, s_nlost, lin, idn, mask, hshift, tid);
      if (s_ndef) {
        const int nd = s_ndef;
        for (int j = tid; j < nd; j += kThreads) {
          const uint16_t i = defl[j];
          const uint32_t key = kc[i];
          uint16_t w;
          if (pair_find_retry(own, kc, key, key * 0x9E3779B1u, hshift, mask, &w) >= 0) {
            atomicAdd(&cnt[w], 1u << 16);
            idn[lin[i]] = w;
          } else {
            kc[i] = ~0u;
          }
        }
        __syncthreads();
      }
      // live: clipped counts (owners), survivors to lout, the table cleared
      if (n < N)
        for (uint32_t s = tid; s < cap / 8; s += kThreads)
          reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
      unsigned int hits = 0;
      for (int q0 = 0; q0 < mq; q0 += kThreads) {
        const int qi = q0 + tid;
        int i0 = 0;
        uint32_t lm = 0;
        int pos[4] = {0, 0, 0, 0};
        if (qi < mq) {
          equad(qi, i0);
          lpos(i0, pos);
          const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
          const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
          uint32_t w[4], cw[4];
  #pragma unroll
          for (int k = 0; k < 4; ++k) w[k] = key[k] != ~0u ? idn[pos[k]] : 0u;
  #pragma unroll
          for (int k = 0; k < 4; ++k) cw[k] = key[k] != ~0u ? cnt[w[k]] : 0u;
  #pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (key[k] == ~0u) continue;
            const uint32_t c = (cw[k] & 0xffffu) + 1u;  // owners are candidate entries
            const uint32_t x = cw[k] >> 16;
            if (w[k] == static_cast<uint32_t>(i0 + k)) hits += c < x ? c : x;
            if (i0 >= roff || x != 0) lm |= 1u << k;
          }
        }
        // the quads of a warp can straddle the two parts: one append per part
        const bool cside = qi < mcq;
        warp_append_quad(lout, &s_nc, cside ? lm : 0u, [&](int k) { return pos[k]; }, lane);
        warp_append_quad(lout + roff, &s_nr, cside ? 0u : lm, [&](int k) { return pos[k]; }, lane);
      }
      hits = __reduce_add_sync(kFull, hits);
      if (lane == 0 && hits) atomicAdd(&s_hits[n - 1], hits);
      cleared = true;
      __syncthreads();
      nc = s_nc;
      nr = s_nr;
      uint16_t* const t = lin;
      lin = lout;
      lout = t;
      TB_MARK(3 + 4 * (n - 1) + 3);
      ++n;
    }
    if (nc > 0 && n <= N) {
      // Few survivors: warp 0 finishes the remaining orders with match.any on the
      // keys.  An n-gram's id for the next order is the lowest lane holding it.
      if (tid < 32) {
        int pos = lane < nc ? lin[lane] : (lane < nc + nr ? lin[roff + lane - nc] : -1);
        uint32_t pid = pos >= 0 ? idn[pos] : 0u;
        for (int m = n; m <= N; ++m) {
          bool valid = pos >= 0;
          uint32_t key = 0;
          if (valid) {
            const int end = pos < roff ? clen : roff + rlen;
            const int q = pos + m - 1;
            valid = q < end && id1[q] != 0xffffu;
            if (valid) key = (pid << 16) | id1[q];
          }
          const unsigned peers = __match_any_sync(kFull, valid ? key : 0xffffffffu - lane);
          const unsigned cm = __ballot_sync(kFull, valid && pos < roff);
          const unsigned rm = __ballot_sync(kFull, valid && pos >= roff);
          const unsigned c = __popc(peers & cm), x = __popc(peers & rm);
          const int leader = __ffs(peers) - 1;
          unsigned h = (valid && lane == leader) ? (c < x ? c : x) : 0u;
          h = __reduce_add_sync(kFull, h);
          if (lane == 0) s_hits[m - 1] += h;
          const bool ok = valid && (pos < roff ? x > 0 : c > 0);
          if (!__any_sync(kFull, ok && pos < roff)) break;
          pos = ok ? pos : -1;
          pid = static_cast<uint32_t>(leader);
        }
        __syncwarp();
      }
    }

    TB_MARK(24);
    // ---- epilogue (warp 0)
    if (tid < 32) {
      const int64_t c = s_len[0];
      const int64_t num = lane < N ? static_cast<int64_t>(s_hits[lane]) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      if (lane < N) {
        if (p.num) p.num[b * N + lane] = num;
        if (p.den) p.den[b * N + lane] = den;
      }
      const int64_t r = s_len[1];
      if (lane == 0) {
        if (p.cand_len_out) p.cand_len_out[b] = c;
        if (p.eff_ref) p.eff_ref[b] = r;
      }
      if (p.scores || p.precisions || p.bp)
        warp_epilogue(num, den, c, r, N, p.smoothing, p.eps, p.k, lane < N ? p.weights[lane] : 0.0,
                      p.precisions ? p.precisions + b * N : nullptr, p.bp ? p.bp + b : nullptr,
                      p.scores ? p.scores + b : nullptr, s_bp);
      if (corpus) {
        if (lane < N) {
          s_tot[lane] += static_cast<unsigned long long>(num);
          s_tot[N + lane] += static_cast<unsigned long long>(den);
        }
        if (lane == 0) {
          s_tot[2 * N] += static_cast<unsigned long long>(c);
          s_tot[2 * N + 1] += static_cast<unsigned long long>(r);
        }
      }
    }
    if (!dbuf && b + gridDim.x < p.batch) {
      __syncthreads();
      issue_stage(b + gridDim.x, 0);
    }
    if (dbuf) {
      cur ^= 1;
      __syncthreads();  // s_len / s_hits of this group are read before the next group resets them
    }
    TB_MARK(30);
  }
  finish_cta(p, s_tot, s_flags, s_last);
  TB_MARK(31);
}

// --------------------------------------------------------------------------
// Multi-reference kernel (2 <= R <= kMultiMaxRefs): the single-reference
// design (candidate insert, reference lookups, retry rounds, quads) with one
// u16 count per (reference, candidate owner) so that the clip is
// min(cand, max_r ref_r) (bleu.py:148-157, oracle.py:36-37).  Every order,
// including the pruned orders >= 2 when more than 32 positions stay live, runs
// the same passes on its keys: order 1 on the tokens, order n on the packed
// (prefix slot, last-token slot) keys.  All references are looked up in one
// pass, so the number of barrier phases does not grow with R.
//
// Positions: candidate [0, cand_pad), reference r at cand_pad + ref_off[r]
// (rows padded to 4).  cnt[o]: candidate count of owner o (owner excluded);
// rc[r][o]: occurrences in reference r of the key owned by candidate position o.
// --------------------------------------------------------------------------

template <typename T>
__global__ void __launch_bounds__(kMultiThreads, 2)
    bleu_multi_kernel(const __grid_constant__ StatsParams p) {
  constexpr int NT = kMultiThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int s_hits[TB_MAX_ORDER];
  __shared__ int64_t s_len[kMultiMaxRefs + 1];
  __shared__ int64_t s_stage_len[kMultiMaxRefs + 1];
  __shared__ unsigned long long s_tot[2 * TB_MAX_ORDER + 2];
  __shared__ int s_last, s_flags;
  __shared__ int s_nlost, s_nc, s_nr, s_ndef;  // s_nc / s_nr: live candidate / reference entries
  __shared__ int s_qbase[kMultiMaxRefs + 2];  // first flattened reference quad of each reference (+ total)
  __shared__ uint32_t s_skey[kSmallSet];   // small-set path: their keys at the current order
  __shared__ uint8_t s_sside[kSmallSet];   // small-set path: 0 = candidate, 1 + r = reference r
  __shared__ int64_t s_effref;             // effective reference length of the current group
  __shared__ double s_bp;                  // and its brevity penalty

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int R = p.num_refs;
  const int N = p.max_order;
  const int cap_log2 = p.cap_log2;
  const uint32_t cap = 1u << cap_log2;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  const int cpad = p.cand_pad;

  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  T* tok = reinterpret_cast<T*>(smem + 16);
  uint32_t* kc = reinterpret_cast<uint32_t*>(smem + 16);           // aliases tok (orders >= 2)
  uint16_t* id1 = reinterpret_cast<uint16_t*>(smem + p.off_id1);   // order-1 slot; 0xffff: token unmatched
  uint16_t* idn = reinterpret_cast<uint16_t*>(smem + p.off_idn);   // order-n slot; 0xffff: n-gram unmatched
  uint16_t* own = reinterpret_cast<uint16_t*>(smem + p.off_ent);   // slot -> owner (candidate) position
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + p.off_mref);  // candidate owner -> candidate count
  uint32_t* rc = reinterpret_cast<uint32_t*>(smem + p.off_kc);     // (ref, candidate owner) -> u16 count, 2 per word
  // two position lists of ptot entries (as in the pair kernel): the live
  // positions of an order (candidates from 0, references from cpad) and the
  // lost (from 0) / deferred (from cpad) entries of the current order
  const int ptot = cpad + p.ref_off[R];
  uint16_t* const lx = reinterpret_cast<uint16_t*>(smem + p.off_lists);
  uint16_t* const ly = lx + ptot;
  uint16_t* const lost = ly;
  uint16_t* const defl = ly + cpad;
  const uint32_t hshift = 32 - cap_log2;
  const uint32_t mask = cap - 1;

  auto issue_stage = [&](int64_t b) {
    if (tid == 0) issue_rows<T>(p, b, R + 1, tok, mbar, s_stage_len, &s_flags);
  };

  if (tid < 2 * N + 2) s_tot[tid] = 0;
  if (tid == 0) {
    s_flags = 0;
    mbar_init(mbar, 1);
  }
  griddep_wait_and_release();
  if (static_cast<int64_t>(blockIdx.x) < p.batch) issue_stage(blockIdx.x);
  __syncthreads();
  TB_MARK(0);
  uint32_t phase = 0;

  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    if (p.prefix_only) {
      __syncthreads();  // s_stage_len of this group, written by thread 0 in issue_rows
      if (tid <= R) s_len[tid] = s_stage_len[tid];
    } else if (tid <= R) {
      const int64_t len = tid == 0 ? p.cand_len[b] : p.refs[tid - 1].len[b];
      const int64_t width = row_width(p, tid);
      int64_t l = len;
      if (len < 0 || len > width) {
        atomicOr(&s_flags, TB_FLAG_BAD_LENGTH);
        l = len < 0 ? 0 : width;
      }
      s_len[tid] = l;
    }
    if (tid < N) s_hits[tid] = 0;
    copy_row_tails<T>(p, b, R + 1, tok, s_stage_len, tid, NT);  // tails / unaligned rows
    mbar_wait(mbar, phase);
    phase ^= 1;
    __syncthreads();
    TB_MARK(2);
    if (tid == 0) {
      int q = 0;
      for (int r = 0; r < R; ++r) {
        s_qbase[r] = q;
        q += static_cast<int>((s_len[r + 1] + 3) >> 2);
      }
      s_qbase[R] = q;
    }

    const int clen = static_cast<int>(s_len[0]);
    const int ncq = (clen + 3) >> 2;
    auto cand_mask = [&](int p0) -> uint32_t { return clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u); };
    // flattened reference quad -> (reference, first position, valid mask)
    auto ref_quad = [&](int qi, int& r, int& p0) -> uint32_t {
      r = 0;
      while (r + 1 < R && qi >= s_qbase[r + 1]) ++r;
      const int j = 4 * (qi - s_qbase[r]);
      p0 = cpad + p.ref_off[r] + j;
      const int left = static_cast<int>(s_len[r + 1]) - j;
      return left >= 4 ? 0xfu : ((1u << left) - 1u);
    };
    auto ref_of = [&](int pos) -> int {  // reference index of a reference position
      int r = 0;  // independent compares against the row starts (no dependent chain)
#pragma unroll
      for (int j = 1; j < kMultiMaxRefs; ++j) r += (j < R && pos >= cpad + p.ref_off[j]) ? 1 : 0;
      return r;
    };
    auto row_end = [&](int pos) -> int {  // one past the last valid position of pos's row
      if (pos < cpad) return clen;
      const int r = ref_of(pos);
      return cpad + p.ref_off[r] + static_cast<int>(s_len[r + 1]);
    };
    auto rc_add = [&](int r, uint32_t o) {
      const uint32_t i = static_cast<uint32_t>(r * cpad) + o;
      atomicAdd(&rc[i >> 1], 1u << (16 * (i & 1u)));
    };
    auto rc_max = [&](uint32_t o) -> uint32_t {
      uint32_t x = 0;
      for (int r = 0; r < R; ++r) {
        const uint32_t i = static_cast<uint32_t>(r * cpad) + o;
        const uint32_t v = (rc[i >> 1] >> (16 * (i & 1u))) & 0xffffu;
        x = v > x ? v : x;
      }
      return x;
    };
    __syncthreads();  // s_qbase
    const int nrq = s_qbase[R];

    // Order 1 on the tokens (K = token type): ids -> slot or 0xffff; the live
    // positions go to the list lx (s_nc / s_nr entries).  All threads call it.
    auto count_order1 = [&](auto* keys, uint16_t* ids, uint16_t* ids2) {
      using K = typename std::remove_const<typename std::remove_pointer<decltype(keys)>::type>::type;
      auto load_keys = [&](int p0, K (&k)[4]) {
        if constexpr (sizeof(K) == 4) {
          const uint4 v = *reinterpret_cast<const uint4*>(keys + p0);
          k[0] = static_cast<K>(v.x);
          k[1] = static_cast<K>(v.y);
          k[2] = static_cast<K>(v.z);
          k[3] = static_cast<K>(v.w);
        } else {
          const longlong2 u = *reinterpret_cast<const longlong2*>(keys + p0);
          const longlong2 v = *reinterpret_cast<const longlong2*>(keys + p0 + 2);
          k[0] = u.x;
          k[1] = u.y;
          k[2] = v.x;
          k[3] = v.y;
        }
      };
      // table, candidate counts and per-reference counts start empty
      for (uint32_t s = tid; s < cap / 8; s += NT) reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
      for (int i = tid; i < (R * cpad + 7) / 8; i += NT) reinterpret_cast<uint4*>(rc)[i] = make_uint4(0, 0, 0, 0);
      if (tid == 0) {
        s_nlost = 0;
        s_ndef = 0;
        s_nc = 0;
        s_nr = 0;
      }
      __syncthreads();
      for (int qi = tid; qi < ncq; qi += NT) {  // claims (plain stores)
        const int p0 = 4 * qi;
        K k[4];
        load_keys(p0, k);
        const uint32_t vm = cand_mask(p0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (vm >> j & 1u) own[tok_hash32(k[j]) >> hshift] = static_cast<uint16_t>(p0 + j);
        *reinterpret_cast<uint4*>(cnt + p0) = make_uint4(0, 0, 0, 0);
      }
      __syncthreads();
      TB_MARK(28);
      for (int qi = tid; qi < ncq; qi += NT) {  // verify
        const int p0 = 4 * qi;
        K k[4];
        load_keys(p0, k);
        const uint32_t vm = cand_mask(p0);
        uint32_t hv[4], home[4];
        uint16_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          hv[j] = tok_hash32(k[j]);
          home[j] = hv[j] >> hshift;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = (vm >> j & 1u) ? own[home[j]] : static_cast<uint16_t>(p0 + j);
        uint32_t lm = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pos = p0 + j;
          if (w[j] != pos) {
            if (keys[w[j]] == k[j]) {
              atomicAdd(&cnt[w[j]], 1u);
            } else {
              lm |= 1u << j;
              pair_retry_store(own, hv[j], 1, hshift, static_cast<uint16_t>(pos));
            }
          }
        }
        *reinterpret_cast<uint2*>(ids + p0) = make_uint2(home[0] | (home[1] << 16), home[2] | (home[3] << 16));
        for (; lm; lm &= lm - 1) lost[atomicAdd(&s_nlost, 1)] = static_cast<uint16_t>(p0 + __ffs(lm) - 1);
      }
      if (tid == NT - 32) {  // lengths only: the last warp, off the epilogue's critical path
        const int64_t r = closest_ref_len(s_len[0], &s_len[1], R);
        s_effref = r;
        s_bp = brevity_penalty_fp64(s_len[0], r);
      }
      __syncthreads();
      TB_MARK(29);
      const int nl = s_nlost;
      auto hashk = [&](uint16_t q) { return tok_hash32(keys[q]); };
      auto eqk = [&](uint16_t a, uint16_t c) { return keys[a] == keys[c]; };
      int left = 0;
      for (int i = tid; i < nl; i += NT) {  // retry round 1 (verify half) ...
        const uint16_t pos = lost[i];
        const uint32_t h = hashk(pos);
        const uint32_t cs = rehash(h, 1, hshift);
        const uint16_t w = own[cs];
        if (w == pos || eqk(pos, w)) {
          if (w != pos) atomicAdd(&cnt[w], 1u);
          ids[pos] = static_cast<uint16_t>(cs);
          lost[i] = 0xffffu;
        } else {
          left = 1;
          pair_retry_store(own, h, 2, hshift, pos);
        }
      }
      for (int q0 = 0; q0 < nrq; q0 += NT) {  // ... with the home-slot lookups of all references
        const int qi = q0 + tid;
        int r = 0, p0 = 0;
        uint32_t fm = 0;  // found: live
        if (qi < nrq) {
        const uint32_t vm0 = ref_quad(qi, r, p0);
        K k[4];
        load_keys(p0, k);
        const uint32_t vm = vm0;
        uint32_t v[4];
        uint16_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = tok_hash32(k[j]) >> hshift;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = (vm >> j & 1u) ? own[v[j]] : static_cast<uint16_t>(0xffffu);
        K ko[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ko[j] = o[j] != 0xffffu ? keys[o[j]] : k[j];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (o[j] != 0xffffu && ko[j] != k[j]) {  // home held by another key: after the retries
            defl[atomicAdd(&s_ndef, 1)] = static_cast<uint16_t>(p0 + j);
            o[j] = 0xffffu;
          }
          if (o[j] == 0xffffu) {
            v[j] = 0xffffu;
          } else {
            rc_add(r, o[j]);
            fm |= 1u << j;
          }
        }
        const uint2 vv = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
        *reinterpret_cast<uint2*>(ids + p0) = vv;
        if (ids2) *reinterpret_cast<uint2*>(ids2 + p0) = vv;
        }
        warp_append_quad(lx + cpad, &s_nr, fm, [&](int j) { return p0 + j; }, lane);
      }
      if (__syncthreads_or(left))
        pair_resolve_lost<NT>(own, cnt, lost, nl, ids, mask, hshift, cpad, tid, hashk, eqk, 2);
      TB_MARK(3);
      const int nd = s_ndef;
      for (int i0 = 0; i0 < nd; i0 += NT) {  // deferred lookups: the full chain
        const int i = i0 + tid;
        bool f = false;
        int pos = 0;
        if (i < nd) {
          pos = defl[i];
          const K key = keys[pos];
          uint16_t o;
          const int sl = pair_find_retry(own, keys, key, tok_hash32(key), hshift, mask, &o);
          if (sl >= 0) {
            rc_add(ref_of(pos), o);
            ids[pos] = static_cast<uint16_t>(sl);
            if (ids2) ids2[pos] = static_cast<uint16_t>(sl);
            f = true;
          }
        }
        warp_append(lx + cpad, &s_nr, f, pos, lane);
      }
      __syncthreads();
      TB_MARK(26);
      unsigned int hits = 0;
      for (int q0 = 0; q0 < ncq; q0 += NT) {  // candidate liveness + clipped count
        const int qi = q0 + tid;
        const int p0 = 4 * qi;
        uint32_t lm = 0;
        if (qi < ncq) {
        K k[4];
        load_keys(p0, k);
        const uint32_t vm = cand_mask(p0);
        const uint2 s2 = *reinterpret_cast<const uint2*>(ids + p0);
        const uint32_t s[4] = {s2.x & 0xffffu, s2.x >> 16, s2.y & 0xffffu, s2.y >> 16};
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pos = p0 + j;
          v[j] = 0xffffu;
          if (vm >> j & 1u) {
            const uint32_t o = own[s[j]];
            const uint32_t x = rc_max(o);
            if (o == static_cast<uint32_t>(pos)) {
              const uint32_t c = (cnt[o] & 0xffffu) + 1u;  // the owner counts itself
              hits += c < x ? c : x;
            }
            if (x != 0) {
              v[j] = s[j];
              lm |= 1u << j;
            }
          }
        }
        const uint2 vv = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
        *reinterpret_cast<uint2*>(ids + p0) = vv;
        if (ids2) *reinterpret_cast<uint2*>(ids2 + p0) = vv;
        }
        warp_append_quad(lx, &s_nc, lm, [&](int j) { return p0 + j; }, lane);
      }
      hits = __reduce_add_sync(kFull, hits);
      if (lane == 0 && hits) atomicAdd(&s_hits[0], hits);
      __syncthreads();
    };

    // ================= order 1: tokens =================
    count_order1(static_cast<const T*>(tok), id1, idn);
    TB_MARK(4);
    int nc = s_nc, nr = s_nr;

    // ================= orders n >= 2 =================
    // While more than kSmallSet positions stay live: one table round per order
    // over the live LISTS, in quads of entries (the pair kernel's rounds, with
    // the per-reference counts rc[r][owner] and the clip min(cand, max_r ref)).
    // Owners, counts and the next prefix ids are list indices.
    uint16_t* lin = lx;
    uint16_t* lout = ly;
    int n = 2;
    bool cleared = false;  // own[] still holds order 1's table
    while (__builtin_expect(n <= N && nc > 0 && nc + nr > kSmallSet, 0)) {
      const int mcq = (nc + 3) >> 2;
      const int mq = mcq + ((nr + 3) >> 2);
      auto equad = [&](int qi, int& i0) -> uint32_t {
        int left;
        if (qi < mcq) {
          i0 = 4 * qi;
          left = nc - i0;
        } else {
          i0 = cpad + 4 * (qi - mcq);
          left = nr - (i0 - cpad);
        }
        return left >= 4 ? 0xfu : ((1u << left) - 1u);
      };
      auto lpos = [&](int i0, int (&pos)[4]) {
        const uint2 l2 = *reinterpret_cast<const uint2*>(lin + i0);
        pos[0] = l2.x & 0xffffu;
        pos[1] = l2.x >> 16;
        pos[2] = l2.y & 0xffffu;
        pos[3] = l2.y >> 16;
      };
      if (!cleared)
        for (uint32_t s = tid; s < cap / 8; s += NT) reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
      for (int qi = tid; qi < mq; qi += NT) {  // keys (~0: dead), counts, candidate claims
        int i0;
        const uint32_t vm = equad(qi, i0);
        int pos[4];
        lpos(i0, pos);
        uint32_t key[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          key[j] = ~0u;
          if (vm >> j & 1u) {
            const int q = pos[j] + n - 1;
            if (q < row_end(pos[j])) {
              const uint16_t l = id1[q];
              if (l != 0xffffu) key[j] = (static_cast<uint32_t>(idn[pos[j]]) << 16) | l;
            }
          }
        }
        *reinterpret_cast<uint4*>(kc + i0) = make_uint4(key[0], key[1], key[2], key[3]);
        if (i0 < cpad) {
          *reinterpret_cast<uint4*>(cnt + i0) = make_uint4(0, 0, 0, 0);
          for (int r = 0; r < R; ++r)  // rc[r][i0 .. i0 + 3]: 4 u16, 8-byte aligned (cpad % 4 == 0)
            *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(rc) + r * cpad + i0) = make_uint2(0, 0);
          if (cleared) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (key[j] != ~0u) own[(key[j] * 0x9E3779B1u) >> hshift] = static_cast<uint16_t>(i0 + j);
          }
        }
      }
      if (tid == 0) {
        s_nlost = 0;
        s_ndef = 0;
      }
      __syncthreads();
      if (!cleared) {
        for (int qi = tid; qi < mcq; qi += NT) {
          const int i0 = 4 * qi;
          const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
          const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (key[j] != ~0u) own[(key[j] * 0x9E3779B1u) >> hshift] = static_cast<uint16_t>(i0 + j);
        }
        __syncthreads();
      }
      if (tid == 0) {  // every thread has read them (barrier above)
        s_nc = 0;
        s_nr = 0;
      }
      uint16_t* const ldef = lout + cpad;  // deferred reference entries (lost candidates from 0)
      for (int qi = tid; qi < mq; qi += NT) {  // verify (candidates) / home lookups (references)
        int i0;
        equad(qi, i0);
        int pos[4];
        lpos(i0, pos);
        const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
        const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
        uint16_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = key[j] != ~0u ? own[(key[j] * 0x9E3779B1u) >> hshift] : 0xffffu;
        uint32_t kw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) kw[j] = w[j] != 0xffffu ? kc[w[j]] : ~0u;
        if (i0 < cpad) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (key[j] == ~0u) continue;
            const int i = i0 + j;
            if (w[j] == i) {
              idn[pos[j]] = static_cast<uint16_t>(i);
            } else if (kw[j] == key[j]) {
              atomicAdd(&cnt[w[j]], 1u);
              idn[pos[j]] = w[j];
            } else {
              lout[atomicAdd(&s_nlost, 1)] = static_cast<uint16_t>(i);
              pair_retry_store(own, key[j] * 0x9E3779B1u, 1, hshift, static_cast<uint16_t>(i));
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (key[j] == ~0u) continue;
            const int i = i0 + j;
            if (w[j] == 0xffffu) {  // empty home: no candidate n-gram has this key
              kc[i] = ~0u;
            } else if (kw[j] == key[j]) {
              rc_add(ref_of(pos[j]), w[j]);
              idn[pos[j]] = w[j];
            } else {
              ldef[atomicAdd(&s_ndef, 1)] = static_cast<uint16_t>(i);
            }
          }
        }
      }
      __syncthreads();
      if (s_nlost) list_resolve_lost<NT>(own, cnt, kc, lout, s_nlost, lin, idn, mask, hshift, tid);
      if (s_ndef) {
        const int nd = s_ndef;
        for (int j = tid; j < nd; j += NT) {
          const uint16_t i = ldef[j];
          const uint32_t key = kc[i];
          uint16_t w;
          if (pair_find_retry(own, kc, key, key * 0x9E3779B1u, hshift, mask, &w) >= 0) {
            rc_add(ref_of(lin[i]), w);
            idn[lin[i]] = w;
          } else {
            kc[i] = ~0u;
          }
        }
        __syncthreads();
      }
      // live: clipped counts (owners), survivors to lout, the table cleared
      if (n < N)
        for (uint32_t s = tid; s < cap / 8; s += NT) reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
      unsigned int hits = 0;
      for (int q0 = 0; q0 < mq; q0 += NT) {
        const int qi = q0 + tid;
        int i0 = 0;
        uint32_t lm = 0;
        int pos[4] = {0, 0, 0, 0};
        if (qi < mq) {
          equad(qi, i0);
          lpos(i0, pos);
          const uint4 k4 = *reinterpret_cast<const uint4*>(kc + i0);
          const uint32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (key[j] == ~0u) continue;
            if (i0 >= cpad) {
              lm |= 1u << j;
              continue;
            }
            const uint32_t w = idn[pos[j]];
            const uint32_t x = rc_max(w);
            if (w == static_cast<uint32_t>(i0 + j)) {
              const uint32_t c = (cnt[w] & 0xffffu) + 1u;  // owners are candidate entries
              hits += c < x ? c : x;
            }
            if (x != 0) lm |= 1u << j;
          }
        }
        const bool cside = qi < mcq;
        warp_append_quad(lout, &s_nc, cside ? lm : 0u, [&](int j) { return pos[j]; }, lane);
        warp_append_quad(lout + cpad, &s_nr, cside ? 0u : lm, [&](int j) { return pos[j]; }, lane);
      }
      hits = __reduce_add_sync(kFull, hits);
      if (lane == 0 && hits) atomicAdd(&s_hits[n - 1], hits);
      cleared = true;
      __syncthreads();
      nc = s_nc;
      nr = s_nr;
      uint16_t* const t = lin;
      lin = lout;
      lout = t;
      ++n;
    }
    if (n <= N && nc > 0) {
      // <= kSmallSet live positions: the remaining orders by direct comparison
      // of their keys (S^2 / blockDim compares per thread, two barriers per
      // order, no table).  An n-gram's id for the next order is the lowest
      // index holding it.
      const int S = nc + nr;
      int pos = -1, side = 0, end = 0;
      uint32_t pid = 0;
      if (tid < S) {
        pos = tid < nc ? lin[tid] : lin[cpad + tid - nc];
        side = pos < cpad ? 0 : 1 + ref_of(pos);
        end = row_end(pos);
        pid = idn[pos];
        s_sside[tid] = static_cast<uint8_t>(side);
      }
      for (int m = n; m <= N; ++m) {
        bool valid = pos >= 0;
        uint32_t key = 0xffffffffu - static_cast<uint32_t>(tid);  // unique for invalid entries
        if (valid) {
          const int q = pos + m - 1;
          valid = q < end && id1[q] != 0xffffu;
          if (valid) key = (pid << 16) | id1[q];
        }
        if (tid < S) s_skey[tid] = key;
        __syncthreads();
        bool ok = false;
        int leader = tid;
        if (valid) {
          unsigned c = 0;
          unsigned xr[kMultiMaxRefs] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int j = 0; j < S; ++j) {
            if (s_skey[j] != key) continue;
            leader = j < leader ? j : leader;
            const int sj = s_sside[j];
            if (sj == 0) {
              ++c;
            } else {
#pragma unroll
              for (int r = 0; r < kMultiMaxRefs; ++r) xr[r] += (sj == r + 1) ? 1u : 0u;
            }
          }
          unsigned x = 0;
#pragma unroll
          for (int r = 0; r < kMultiMaxRefs; ++r) x = xr[r] > x ? xr[r] : x;
          if (leader == tid) {
            const unsigned h = c < x ? c : x;
            if (h) atomicAdd(&s_hits[m - 1], h);
          }
          ok = side == 0 ? x > 0 : c > 0;
        }
        if (!__syncthreads_or(ok && side == 0)) break;  // also: every key read before the next order
        pos = ok ? pos : -1;
        pid = static_cast<uint32_t>(leader);
      }
    }
    __syncthreads();
    TB_MARK(24);

    // ---- epilogue (warp 0)
    if (tid < 32) {
      const int64_t c = s_len[0];
      const int64_t num = lane < N ? static_cast<int64_t>(s_hits[lane]) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      if (lane < N) {
        if (p.num) p.num[b * N + lane] = num;
        if (p.den) p.den[b * N + lane] = den;
      }
      const int64_t r = s_effref;
      if (lane == 0) {
        if (p.cand_len_out) p.cand_len_out[b] = c;
        if (p.eff_ref) p.eff_ref[b] = r;
      }
      if (p.scores || p.precisions || p.bp)
        warp_epilogue(num, den, c, r, N, p.smoothing, p.eps, p.k, lane < N ? p.weights[lane] : 0.0,
                      p.precisions ? p.precisions + b * N : nullptr, p.bp ? p.bp + b : nullptr,
                      p.scores ? p.scores + b : nullptr, s_bp);
      if (corpus) {
        if (lane < N) {
          s_tot[lane] += static_cast<unsigned long long>(num);
          s_tot[N + lane] += static_cast<unsigned long long>(den);
        }
        if (lane == 0) {
          s_tot[2 * N] += static_cast<unsigned long long>(c);
          s_tot[2 * N + 1] += static_cast<unsigned long long>(r);
        }
      }
    }
    if (b + gridDim.x < p.batch) {
      __syncthreads();
      issue_stage(b + gridDim.x);
    }
    TB_MARK(30);
  }
  finish_cta(p, s_tot, s_flags, s_last);
  TB_MARK(31);
}

// --------------------------------------------------------------------------
// Stand-alone epilogue / totals / validation kernels.
// --------------------------------------------------------------------------
struct EpiParams {
  int smoothing;
  double eps;
  double k;
  double weights[TB_MAX_ORDER];
};

__global__ void bleu_scores_kernel(const int64_t* __restrict__ num, const int64_t* __restrict__ den,
                                   const int64_t* __restrict__ cand_len,
                                   const int64_t* __restrict__ eff_ref, int64_t batch, int N,
                                   const __grid_constant__ EpiParams e, double* scores,
                                   double* precisions, double* bp) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < batch;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bleu_epilogue(num + b * N, den + b * N, cand_len[b], eff_ref[b], N, e.smoothing, e.eps, e.k,
                  e.weights, precisions ? precisions + b * N : nullptr, bp ? bp + b : nullptr,
                  scores ? scores + b : nullptr);
  }
}

// one CTA per output column: [num_0..N-1 | den_0..N-1 | cand_len | eff_ref]
__global__ void bleu_totals_kernel(const int64_t* __restrict__ num, const int64_t* __restrict__ den,
                                   const int64_t* __restrict__ cand_len,
                                   const int64_t* __restrict__ eff_ref, int64_t batch, int N,
                                   int64_t* totals) {
  __shared__ long long s_part[32];
  const int col = blockIdx.x;
  long long acc = 0;
  for (int64_t b = threadIdx.x; b < batch; b += blockDim.x) {
    if (col < N)
      acc += num[b * N + col];
    else if (col < 2 * N)
      acc += den[b * N + (col - N)];
    else if (col == 2 * N)
      acc += cand_len[b];
    else
      acc += eff_ref[b];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += s_part[w];
    totals[col] = t;
  }
}

// B == 0: no flags; corpus totals zero, epilogue of zeros (bleu.py:295-305 on empty stats)
__global__ void bleu_empty_corpus_kernel(int N, const __grid_constant__ EpiParams e, int64_t* totals,
                                         double* corpus, int32_t* err) {
  if (threadIdx.x != 0) return;
  *err = 0;
  int64_t z[TB_MAX_ORDER];
  for (int n = 0; n < N; ++n) z[n] = 0;
  if (totals)
    for (int i = 0; i < 2 * N + 2; ++i) totals[i] = 0;
  if (corpus) bleu_epilogue(z, z, 0, 0, N, e.smoothing, e.eps, e.k, e.weights, corpus + 2, corpus + 1, corpus);
}

template <typename T>
__global__ void validate_batch_kernel(const T* __restrict__ ids, int64_t ld, int64_t width,
                                      const int64_t* __restrict__ lengths, int64_t batch,
                                      int32_t* err) {
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    int64_t len = lengths[b];
    if (len < 0 || len > width) {
      if (threadIdx.x == 0) atomicOr(err, TB_FLAG_BAD_LENGTH);
      len = len < 0 ? 0 : width;
    }
    const T* row = ids + b * ld;
    bool neg = false;
    for (int64_t j = threadIdx.x; j < len; j += blockDim.x) neg |= row[j] < 0;
    if (__any_sync(kFull, neg) && (threadIdx.x & 31) == 0) atomicOr(err, TB_FLAG_NEGATIVE_ID);
  }
}

// --------------------------------------------------------------------------
// Device properties (cached per device).
// --------------------------------------------------------------------------
struct DevInfo {
  int sms = 0;
  int smem_optin = 0;
  bool ok = false;
};
DevInfo g_dev[64];

int dev_info(DevInfo** out) {
  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return TB_ERR_UNSUPPORTED;
  DevInfo& d = g_dev[dev];
  if (!d.ok) {
    TB_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    TB_CUDA(cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    d.ok = true;
  }
  *out = &d;
  return TB_OK;
}

// --------------------------------------------------------------------------
// Shape planning shared by the workspace query and the launch.
// --------------------------------------------------------------------------
struct Plan {
  bool smem_mode = false;
  bool pair = false;   // single-reference kernel
  bool multi = false;  // multi-reference kernel
  int cap_log2 = 0;
  int filter_log2 = 0;
  int cand_pad = 0;
  int ref_off[TB_MAX_REFS + 1] = {0};
  int off_id1 = 0, off_idn = 0, off_live = 0, off_ent = 0, off_mref = 0, off_kc = 0, off_lists = 0, off_seg = 0;
  int off_tok2 = 0;
  size_t smem_bytes = 0;   // dynamic smem (smem mode)
  size_t gtab_stride = 0;  // per-CTA table bytes (global mode)
  int64_t grid = 0;
  size_t acc_bytes = 0;
  size_t ws_bytes = 0;
};

constexpr size_t kStaticSmemReserve = 2048;  // static __shared__ of the stats kernels (upper bound)
constexpr int64_t kGlobalGridCap = 2 * 148;
// fixed-size completion region at the start of the workspace, independent of N
constexpr size_t kAccBytes = ((kAccCopies * (2 * TB_MAX_ORDER + 2) * 8 + 256) + 255) / 256 * 256;

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int cap_log2_for(int64_t want, int min_log2) {
  int c = min_log2;
  while ((int64_t(1) << c) < want) ++c;
  return c;
}

int make_plan(int64_t batch, int R, int64_t cand_width, const int64_t* ref_widths, int token_bytes,
              int N, int smem_optin, int sms, Plan* pl) {
  (void)N;
  int64_t ref_total = 0, max_rw = 0;
  for (int r = 0; r < R; ++r) {
    ref_total += ref_widths[r];
    if (ref_widths[r] > max_rw) max_rw = ref_widths[r];
  }
  const int64_t elems16 = 16 / token_bytes;
  pl->acc_bytes = kAccBytes;

  // ---- single reference: joint-insert kernel
  pl->cand_pad = static_cast<int>(round_up(cand_width, elems16));
  if (R == 1) {
    const int64_t cpad4 = round_up(cand_width, 4);  // quads of positions never straddle the two rows
    const int64_t rpad = round_up(ref_widths[0], 4);
    const int64_t ptot = cpad4 + rpad;
    auto pair_layout = [&](int log2, int64_t* offs) {
      const int64_t c = int64_t(1) << log2;
      int64_t o = round_up(16 + ptot * (token_bytes > 4 ? token_bytes : 4), 16);
      offs[0] = o;                       // id1
      o = round_up(o + ptot * 2, 16);
      offs[1] = o;                       // idn
      o = round_up(o + ptot * 2, 16);
      offs[2] = o;                       // own (u16 per slot)
      o = round_up(o + c * 2, 16);
      offs[3] = o;                       // cnt (u32 per candidate position / entry)
      o = round_up(o + cpad4 * 4, 16);
      offs[4] = o;                       // two position lists (u16 per position each)
      o = round_up(o + ptot * 4, 16);
      offs[5] = o;
      return o;
    };
    // only candidate keys are inserted (every order).  Table load factor <= 1/8
    // of the candidate width, else <= 1/4, at kPairCtasPerSm CTAs per SM, else
    // the same at 3 CTAs per SM, else <= 1/2.
    auto fits = [&](int64_t t, int ctas) {
      return t + static_cast<int64_t>(kStaticSmemReserve) <= smem_optin / ctas;
    };
    int64_t offs[6];
    int lg = -1;
    for (int ctas = kPairCtasPerSm; ctas >= 3 && lg < 0; --ctas)
      for (int l = cap_log2_for(8 * cpad4, 6); l >= 6 && (int64_t(1) << l) >= 4 * cpad4; --l)
        if (fits(pair_layout(l, offs), ctas)) {
          lg = l;
          break;
        }
    if (lg < 0) lg = cap_log2_for(2 * cpad4, 6);
    const int64_t total = pair_layout(lg, offs);
    if (lg <= 16 && ptot <= 16384 && total + static_cast<int64_t>(kStaticSmemReserve) <= smem_optin) {
      pl->smem_mode = true;
      pl->pair = true;
      pl->cand_pad = static_cast<int>(cpad4);
      pl->cap_log2 = lg;
      // the order-1 filter's two bitmaps span the table and the count array
      // (adjacent; neither is in use while filtering)
      {
        const int64_t words = ((int64_t(1) << lg) * 2 + cpad4 * 4) / 8;  // per side
        int fl = 0;
        while ((int64_t(2) << fl) <= words) ++fl;
        pl->filter_log2 = fl;
      }
      pl->ref_off[0] = 0;
      pl->ref_off[1] = static_cast<int>(rpad);
      pl->off_id1 = static_cast<int>(offs[0]);
      pl->off_idn = static_cast<int>(offs[1]);
      pl->off_ent = static_cast<int>(offs[2]);
      pl->off_mref = static_cast<int>(offs[3]);
      pl->off_lists = static_cast<int>(offs[4]);
      pl->smem_bytes = static_cast<size_t>(total);
      // CTAs that process several groups prefetch the next group's rows into a
      // second token buffer while they work on the current one — when that
      // buffer still fits kPairCtasPerSm CTAs per SM
      const int64_t tok2 = round_up(ptot * (token_bytes > 4 ? token_bytes : 4), 16);
      int ctas = static_cast<int>(smem_optin / (total + static_cast<int64_t>(kStaticSmemReserve)));
      ctas = ctas < kPairCtasPerSm ? ctas : kPairCtasPerSm;
      if (ctas >= 1 && batch > static_cast<int64_t>(ctas) * sms && fits(total + tok2, ctas)) {
        pl->off_tok2 = static_cast<int>(total);
        pl->smem_bytes = static_cast<size_t>(total + tok2);
      }
      pl->ws_bytes = pl->acc_bytes;
      return TB_OK;
    }
  }

  // ---- multi-reference kernel layout (2 <= R <= kMultiMaxRefs)
  if (R >= 2 && R <= kMultiMaxRefs) {
    const int64_t cpad4 = round_up(cand_width, 4);
    int64_t roff[TB_MAX_REFS + 1];
    int64_t o = 0;
    for (int r = 0; r < R; ++r) {
      roff[r] = o;
      o += round_up(ref_widths[r], 4);
    }
    roff[R] = o;
    const int64_t ptot = cpad4 + o;
    auto multi_layout = [&](int log2, int64_t* offs) {
      const int64_t c = int64_t(1) << log2;
      int64_t q = round_up(16 + ptot * (token_bytes > 4 ? token_bytes : 4), 16);
      offs[0] = q;                          // id1
      q = round_up(q + ptot * 2, 16);
      offs[1] = q;                          // idn
      q = round_up(q + ptot * 2, 16);
      offs[2] = q;                          // own (u16 per slot)
      q = round_up(q + c * 2, 16);
      offs[3] = q;                          // cnt (u32 per candidate position)
      q = round_up(q + cpad4 * 4, 16);
      offs[4] = q;                          // rc (u16 per reference x candidate position)
      q = round_up(q + R * cpad4 * 2, 16);
      offs[5] = q;                          // two position lists (u16 per position each)
      q = round_up(q + ptot * 4, 16);
      return q;
    };
    // table load <= 1/8 of the candidate positions while two CTAs fit per SM
    int lg = cap_log2_for(8 * cpad4, 6);
    int64_t offs[6];
    int64_t total = multi_layout(lg, offs);
    while (total + static_cast<int64_t>(kStaticSmemReserve) > smem_optin / 2 && (int64_t(1) << (lg - 1)) >= 2 * cpad4) {
      --lg;
      total = multi_layout(lg, offs);
    }
    if (lg <= 15 && ptot < 65535 && total + static_cast<int64_t>(kStaticSmemReserve) <= smem_optin) {
      pl->smem_mode = true;
      pl->multi = true;
      pl->cand_pad = static_cast<int>(cpad4);
      pl->cap_log2 = lg;
      for (int r = 0; r <= R; ++r) pl->ref_off[r] = static_cast<int>(roff[r]);
      pl->off_id1 = static_cast<int>(offs[0]);
      pl->off_idn = static_cast<int>(offs[1]);
      pl->off_ent = static_cast<int>(offs[2]);
      pl->off_mref = static_cast<int>(offs[3]);
      pl->off_kc = static_cast<int>(offs[4]);
      pl->off_lists = static_cast<int>(offs[5]);
      pl->smem_bytes = static_cast<size_t>(total);
      pl->ws_bytes = pl->acc_bytes;
      return TB_OK;
    }
  }

  // ---- shared-memory (pruned progressive) layout
  int64_t off = 0;
  for (int r = 0; r < R; ++r) {
    pl->ref_off[r] = static_cast<int>(off);
    off += round_up(ref_widths[r], elems16);
  }
  pl->ref_off[R] = static_cast<int>(off);
  const int64_t ptot = pl->cand_pad + off;  // positions (candidate + references, padded)
  auto layout = [&](int log2, int64_t* offs) {
    const int64_t c = int64_t(1) << log2;
    int64_t o = round_up(16 + ptot * token_bytes, 16);
    offs[0] = o;                              // id1
    o = round_up(o + ptot * 2, 16);
    offs[1] = o;                              // idn
    o = round_up(o + ptot * 2, 16);
    offs[2] = o;                              // live
    o = round_up(o + ptot, 16);
    offs[3] = o;                              // ent (u32) + reference counts (u16)
    o = round_up(o + c * 6, 16);
    offs[4] = o;                              // mref
    if (R > 1) o = round_up(o + c * 2, 16);
    offs[5] = o;                              // kc (u32 per candidate position)
    o = round_up(o + static_cast<int64_t>(pl->cand_pad) * 4, 16);
    offs[6] = o;                              // lists: lc, ins (cand_pad each), lr[2] (ref_off[R] each)
    o = round_up(o + (2 * pl->cand_pad + 2 * off) * 2, 16);
    return o;
  };
  int64_t offs[7];
  // load factor <= 1/4 when four CTAs still fit per SM, else <= 1/2
  int sm_log2 = cap_log2_for(4 * cand_width, 6);
  if (sm_log2 > 16) sm_log2 = 16;
  int64_t total = layout(sm_log2, offs);
  if (total + static_cast<int64_t>(kStaticSmemReserve) > smem_optin / 4 && sm_log2 > 6) {
    --sm_log2;
    total = layout(sm_log2, offs);
  }
  const bool fits = cand_width <= 32768 && max_rw <= 65535 && ptot <= 65535 && (int64_t(1) << sm_log2) >= 2 * cand_width &&
                    total + static_cast<int64_t>(kStaticSmemReserve) <= smem_optin;
  if (fits) {
    pl->smem_mode = true;
    pl->cap_log2 = sm_log2;
    pl->off_id1 = static_cast<int>(offs[0]);
    pl->off_idn = static_cast<int>(offs[1]);
    pl->off_live = static_cast<int>(offs[2]);
    pl->off_ent = static_cast<int>(offs[3]);
    pl->off_mref = static_cast<int>(offs[4]);
    pl->off_kc = static_cast<int>(offs[5]);
    pl->off_lists = static_cast<int>(offs[6]);
    pl->smem_bytes = static_cast<size_t>(total);
    pl->gtab_stride = 0;
    pl->ws_bytes = pl->acc_bytes;
    return TB_OK;
  }

  // ---- global-memory fallback (very wide rows): position-keyed table of all reference n-grams
  const int64_t max_w = cand_width > max_rw ? cand_width : max_rw;
  if (max_w >= (int64_t(1) << kGlobalKeyShift)) return TB_ERR_UNSUPPORTED;
  const int g_log2 = cap_log2_for(2 * ref_total < 32 ? 32 : 2 * ref_total, 5);
  if (g_log2 > 30) return TB_ERR_UNSUPPORTED;
  pl->smem_mode = false;
  pl->cap_log2 = g_log2;
  pl->smem_bytes = 16;
  pl->gtab_stride = static_cast<size_t>(round_up((int64_t(1) << g_log2) * (8 + 4), 256));
  const int64_t cap_grid = sms > 0 ? 2 * sms : kGlobalGridCap;
  pl->grid = batch < cap_grid ? batch : cap_grid;
  if (pl->grid < 1) pl->grid = 1;
  pl->ws_bytes = pl->acc_bytes + static_cast<size_t>(pl->grid) * pl->gtab_stride;
  return TB_OK;
}

template <typename K>
int launch_kernel(K kern, const StatsParams& prm, const Plan& pl, int sms, bool persistent_fill,
                  size_t* attr_set, cudaStream_t stream, int threads = kThreads) {
  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  if (pl.smem_bytes > 48 * 1024 && attr_set[dev & 63] < pl.smem_bytes) {
    TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(pl.smem_bytes)));
    attr_set[dev & 63] = pl.smem_bytes;
  }
  int64_t grid = pl.grid;
  if (persistent_fill) {
    // occupancy per (device, dynamic smem) of this kernel instantiation, cached:
    // the query costs microseconds on every launch otherwise
    static thread_local struct { int dev; size_t smem; int occ; } cache[8] = {};
    static thread_local int next = 0;
    int occ = 0;
    for (auto& e : cache)
      if (e.occ > 0 && e.dev == dev && e.smem == pl.smem_bytes) occ = e.occ;
    if (occ == 0) {
      TB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, pl.smem_bytes));
      if (occ < 1) occ = 1;
      cache[next] = {dev, pl.smem_bytes, occ};
      next = (next + 1) & 7;
    }
    const int64_t resident = static_cast<int64_t>(occ) * sms;
    grid = prm.batch < resident ? prm.batch : resident;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = pl.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TB_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

template <typename T>
int launch_stats(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream) {
  if (pl.pair) {
    static size_t attr_set[64] = {0};
    return launch_kernel(bleu_pair_kernel<T>, prm, pl, sms, true, attr_set, stream);
  }
  if (pl.multi) {
    static size_t attr_set[64] = {0};
    return launch_kernel(bleu_multi_kernel<T>, prm, pl, sms, true, attr_set, stream, kMultiThreads);
  }
  if (pl.smem_mode) {
    static size_t attr_set[64] = {0};
    return launch_kernel(bleu_group_kernel<T>, prm, pl, sms, true, attr_set, stream);
  }
  static size_t attr_set[64] = {0};
  return launch_kernel(bleu_stats_kernel<T, false>, prm, pl, sms, false, attr_set, stream);
}

void fill_epi(EpiParams* e, int N, int smoothing, double eps, double k, const double* weights) {
  e->smoothing = smoothing;
  e->eps = eps;
  e->k = k;
  for (int n = 0; n < TB_MAX_ORDER; ++n) e->weights[n] = n < N ? weights[n] : 0.0;
}

int check_epi(int N, int smoothing, double eps, double k, const double* weights) {
  if (N < 1) return TB_ERR_INVALID_ARG;
  if (N > TB_MAX_ORDER) return TB_ERR_UNSUPPORTED;
  if (smoothing < TB_SMOOTH_NONE || smoothing > TB_SMOOTH_EXP) return TB_ERR_INVALID_ARG;
  if (!(eps > 0) || !(k > 0)) return TB_ERR_INVALID_ARG;
  if (!weights) return TB_ERR_INVALID_ARG;
  for (int n = 0; n < N; ++n)
    if (!(weights[n] >= 0)) return TB_ERR_INVALID_ARG;
  return TB_OK;
}

}  // namespace

// ==========================================================================
// Segment kernels for the plugin surface live in plugin.cu; C ABI below.
// ==========================================================================
// The launch behind tb_bleu_stats / tb_bleu_host.
static int stats_impl(int32_t token_bytes, const void* cand_ids, int64_t cand_ld, int64_t cand_width,
                  const int64_t* cand_len, int32_t num_refs, const void* const* ref_ids,
                  const int64_t* ref_ld, const int64_t* ref_width, const int64_t* const* ref_len,
                  int64_t batch, int32_t max_order, int32_t smoothing, double eps, double k,
                  const double* weights, int64_t* num_out, int64_t* den_out, int64_t* cand_len_out,
                  int64_t* eff_ref_out, double* scores_out, double* precisions_out, double* bp_out,
                  int64_t* totals_out, double* corpus_out, int32_t* err_flag, void* workspace,
                  size_t workspace_bytes, void* stream_, int prefix_only, int err_store) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (token_bytes != 4 && token_bytes != 8) return TB_ERR_INVALID_ARG;
  if (num_refs < 1) return TB_ERR_INVALID_ARG;
  if (num_refs > TB_MAX_REFS) return TB_ERR_UNSUPPORTED;
  if (batch < 0 || cand_width < 0 || cand_ld < cand_width) return TB_ERR_INVALID_ARG;
  int rc = check_epi(max_order, smoothing, eps, k, weights);
  if (rc != TB_OK) return rc;
  if (!ref_ids || !ref_ld || !ref_width || !ref_len || !err_flag) return TB_ERR_INVALID_ARG;
  for (int r = 0; r < num_refs; ++r)
    if (ref_width[r] < 0 || ref_ld[r] < ref_width[r]) return TB_ERR_INVALID_ARG;
  if (batch == 0) {
    EpiParams e;
    fill_epi(&e, max_order, smoothing, eps, k, weights);
    bleu_empty_corpus_kernel<<<1, 32, 0, stream>>>(max_order, e, totals_out, corpus_out, err_flag);
    TB_CUDA(cudaGetLastError());
    return TB_OK;
  }
  if ((!cand_ids && cand_width > 0) || !cand_len) return TB_ERR_INVALID_ARG;

  DevInfo* d = nullptr;
  rc = dev_info(&d);
  if (rc != TB_OK) return rc;
  Plan pl;
  rc = make_plan(batch, num_refs, cand_width, ref_width, token_bytes, max_order, d->smem_optin, d->sms, &pl);
  if (rc != TB_OK) return rc;
  if (workspace_bytes < pl.ws_bytes || (pl.ws_bytes && !workspace)) return TB_ERR_WORKSPACE;

  StatsParams prm;
  memset(&prm, 0, sizeof(prm));
  prm.cand_ids = cand_ids;
  prm.cand_ld = cand_ld;
  prm.cand_width = cand_width;
  prm.cand_len = cand_len;
  for (int r = 0; r < num_refs; ++r) {
    prm.refs[r].ids = ref_ids[r];
    prm.refs[r].ld = ref_ld[r];
    prm.refs[r].width = ref_width[r];
    prm.refs[r].len = ref_len[r];
    if (!ref_len[r] || (!ref_ids[r] && ref_width[r] > 0)) return TB_ERR_INVALID_ARG;
  }
  prm.num_refs = num_refs;
  prm.max_order = max_order;
  prm.batch = batch;
  prm.smoothing = smoothing;
  prm.eps = eps;
  prm.k = k;
  for (int n = 0; n < TB_MAX_ORDER; ++n) prm.weights[n] = n < max_order ? weights[n] : 0.0;
  prm.num = num_out;
  prm.den = den_out;
  prm.cand_len_out = cand_len_out;
  prm.eff_ref = eff_ref_out;
  prm.scores = scores_out;
  prm.precisions = precisions_out;
  prm.bp = bp_out;
  prm.totals = totals_out;
  prm.corpus = corpus_out;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  prm.acc = reinterpret_cast<unsigned long long*>(ws);
  prm.done = reinterpret_cast<unsigned int*>(ws + pl.acc_bytes - 256);
  prm.ws_flag = reinterpret_cast<int*>(ws + pl.acc_bytes - 256 + 4);
  prm.err = err_flag;
  prm.cap_log2 = pl.cap_log2;
  prm.filter_log2 = pl.filter_log2;
  prm.cand_pad = pl.cand_pad;
  for (int r = 0; r <= num_refs; ++r) prm.ref_off[r] = pl.ref_off[r];
  prm.off_id1 = pl.off_id1;
  prm.off_idn = pl.off_idn;
  prm.off_live = pl.off_live;
  prm.off_ent = pl.off_ent;
  prm.off_mref = pl.off_mref;
  prm.off_kc = pl.off_kc;
  prm.off_lists = pl.off_lists;
  prm.off_seg = pl.off_seg;
  prm.off_tok2 = pl.off_tok2;
  prm.gtab = pl.smem_mode ? nullptr : ws + pl.acc_bytes;
  prm.gtab_stride = pl.gtab_stride;
  prm.prefix_only = prefix_only && pl.smem_mode;
  prm.err_store = err_store;

  if (token_bytes == 4) return launch_stats<int32_t>(prm, pl, d->sms, stream);
  return launch_stats<int64_t>(prm, pl, d->sms, stream);
}


// --------------------------------------------------------------------------
// Host-buffer mode (tb_bleu_host): per-thread, per-device cached buffers.
// --------------------------------------------------------------------------
namespace {

struct HostCtx {
  void* ws = nullptr;            // device workspace, zero-filled (kernel contract)
  size_t ws_bytes = 0;
  unsigned char* pin = nullptr;  // pinned, mapped staging: lengths in, results out
  unsigned char* pin_dev = nullptr;
  size_t pin_bytes = 0;
  unsigned char* dstage = nullptr;  // device staging for rows the kernel cannot read in place
  size_t dstage_bytes = 0;
  unsigned char* rows = nullptr;   // pinned, mapped: valid prefixes of pageable rows
  unsigned char* rows_dev = nullptr;
  size_t rows_bytes = 0;
};
thread_local HostCtx g_host[64];

int grow_device(void** buf, size_t* have, size_t want, bool zero) {
  if (*have >= want && *buf) return TB_OK;
  if (*buf) TB_CUDA(cudaFree(*buf));
  *buf = nullptr;
  *have = 0;
  const size_t sz = want < (size_t(1) << 16) ? (size_t(1) << 16) : want + want / 4;
  TB_CUDA(cudaMalloc(buf, sz));
  if (zero) TB_CUDA(cudaMemset(*buf, 0, sz));
  *have = sz;
  return TB_OK;
}

int grow_pinned(HostCtx& c, size_t want) {
  if (c.pin_bytes >= want && c.pin) return TB_OK;
  if (c.pin) TB_CUDA(cudaFreeHost(c.pin));
  c.pin = nullptr;
  c.pin_bytes = 0;
  const size_t sz = want < (size_t(1) << 16) ? (size_t(1) << 16) : want + want / 4;
  void* h = nullptr;
  TB_CUDA(cudaHostAlloc(&h, sz, cudaHostAllocMapped | cudaHostAllocPortable));
  void* d = nullptr;
  TB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
  c.pin = static_cast<unsigned char*>(h);
  c.pin_dev = static_cast<unsigned char*>(d);
  c.pin_bytes = sz;
  return TB_OK;
}

int grow_pinned_rows(HostCtx& c, size_t want) {
  if (c.rows_bytes >= want && c.rows) return TB_OK;
  if (c.rows) TB_CUDA(cudaFreeHost(c.rows));
  c.rows = nullptr;
  c.rows_bytes = 0;
  const size_t sz = want < (size_t(1) << 20) ? (size_t(1) << 20) : want + want / 4;
  void* h = nullptr;
  TB_CUDA(cudaHostAlloc(&h, sz, cudaHostAllocMapped | cudaHostAllocPortable));
  void* dv = nullptr;
  TB_CUDA(cudaHostGetDevicePointer(&dv, h, 0));
  c.rows = static_cast<unsigned char*>(h);
  c.rows_dev = static_cast<unsigned char*>(dv);
  c.rows_bytes = sz;
  return TB_OK;
}

// A small persistent pool of host threads for the pageable-row staging copy
// (the caller works too).  Jobs are serialised; run(n, f) calls f(i) for
// every i in [0, n) exactly once and returns when all are done.  Work items
// are claimed by CAS on a counter tagged with the job number, so a worker that
// is late for one job can never claim (or skip) an item of the next one.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  template <typename F>
  void run(int n, F f) {
    std::lock_guard<std::mutex> job_lock(job_);
    std::function<void(int)> fn(f);
    uint32_t g;
    {
      std::lock_guard<std::mutex> l(m_);
      g = ++gen_;
      fn_ = &fn;
      n_ = n;
      left_.store(n);
      next_.store(static_cast<uint64_t>(g) << 32);
      gen_pub_.store(g);
    }
    cv_.notify_all();
    work(g, &fn, n);
    while (left_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
  }

 private:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = std::max(0, std::min(7, static_cast<int>(hw / 2) - 1));
    for (int i = 0; i < nt; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
    }
    stop_flag_.store(true);
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  // claim items of job g only (never touches another job's counter)
  void work(uint32_t g, std::function<void(int)>* fn, int n) {
    uint64_t v = next_.load();
    while (true) {
      if (static_cast<uint32_t>(v >> 32) != g || static_cast<int>(v & 0xffffffffu) >= n) return;
      if (!next_.compare_exchange_weak(v, v + 1)) continue;
      (*fn)(static_cast<int>(v & 0xffffffffu));
      left_.fetch_sub(1, std::memory_order_release);
      v = next_.load();
    }
  }
  void loop() {
    uint32_t seen = 0;
    while (true) {
      // spin briefly for the next job (calls usually come back to back; a
      // condition-variable wake-up costs tens of microseconds), then sleep
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_pub_.load() == seen && !stop_flag_.load() &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(300)) {
      }
      uint32_t g;
      std::function<void(int)>* fn;
      int n;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        g = seen = gen_;
        fn = fn_;
        n = n_;
      }
      work(g, fn, n);
    }
  }
  std::vector<std::thread> threads_;
  std::mutex job_, m_;
  std::condition_variable cv_;
  // the current job (written under m_)
  uint32_t gen_ = 0;
  std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  bool stop_ = false;
  std::atomic<uint32_t> gen_pub_{0};
  std::atomic<bool> stop_flag_{false};
  std::atomic<uint64_t> next_{0};
  std::atomic<int> left_{0};
};

// Copy the clamped valid prefixes of rows [b0, b1) of every set to dst[s]
// (row stride dst_lds[s] elements of `ob` bytes; int64 -> int32 when ob == 4
// < token_bytes) on the host thread pool.  Returns the OR of the bits of the
// narrowed IDs above bit 30 (non-zero: some ID does not fit int32).
uint64_t copy_rows(int token_bytes, int ob, int nsets, const void* const* ids, const int64_t* lds,
                   const int64_t* widths, const int64_t* const* lens, int64_t b0, int64_t b1,
                   unsigned char* const* dst, const int64_t* dst_lds) {
  constexpr int64_t kRowsPerItem = 16;
  const int64_t per_set = (b1 - b0 + kRowsPerItem - 1) / kRowsPerItem;
  std::atomic<uint64_t> high{0};
  CopyPool::get().run(static_cast<int>(per_set * nsets), [&](int item) {
    const int s = static_cast<int>(item / per_set);
    const int64_t r0 = b0 + (item % per_set) * kRowsPerItem;
    const int64_t r1 = std::min(b1, r0 + kRowsPerItem);
    uint64_t hi = 0;
    for (int64_t b = r0; b < r1; ++b) {
      int64_t n = lens[s][b];
      n = n < 0 ? 0 : (n > widths[s] ? widths[s] : n);  // the kernel's clamp (it flags the row)
      unsigned char* o = dst[s] + static_cast<size_t>((b - b0) * dst_lds[s]) * ob;
      if (token_bytes == 8 && ob == 4) {
        const int64_t* src = static_cast<const int64_t*>(ids[s]) + b * lds[s];
        int32_t* o32 = reinterpret_cast<int32_t*>(o);
        for (int64_t j = 0; j < n; ++j) {
          const int64_t v = src[j];
          hi |= static_cast<uint64_t>(v) >> 31;
          o32[j] = static_cast<int32_t>(v);
        }
      } else if (n > 0) {
        memcpy(o, static_cast<const unsigned char*>(ids[s]) + static_cast<size_t>(b * lds[s]) * token_bytes,
               static_cast<size_t>(n) * token_bytes);
      }
    }
    if (hi) high.fetch_or(hi, std::memory_order_relaxed);
  });
  return high.load();
}

// Valid prefixes of pageable token rows -> pinned, mapped memory the kernel
// reads over PCIe (instead of DMA-ing whole rows through the driver's bounce
// buffer).  int64 rows are narrowed to int32 when every valid ID fits (the
// common case: vocabulary IDs), halving the PCIe bytes; an ID >= 2^31 makes
// the copy redo in int64.  Rows are written at a 16-byte-aligned stride; only
// the clamped valid prefix of each row is written (the kernel reads no more).
// Returns the token bytes of the staged rows (0: not staged).
int stage_pageable_rows(HostCtx& c, int token_bytes, int nsets, const void* const* ids, const int64_t* lds,
                        const int64_t* widths, const int64_t* const* lens, int64_t B, const void** out_ids,
                        int64_t* out_lds, int* rc_out) {
  *rc_out = TB_OK;
  // the outputs may alias the inputs: keep the source pointers and strides
  const void* src_ids[TB_MAX_REFS + 1];
  int64_t src_lds[TB_MAX_REFS + 1];
  for (int s = 0; s < nsets; ++s) {
    src_ids[s] = ids[s];
    src_lds[s] = lds[s];
  }
  constexpr int64_t kRowsPerItem = 16;
  const int64_t items_per_set = (B + kRowsPerItem - 1) / kRowsPerItem;
  auto layout = [&](int ob, size_t* offs) {
    size_t o = 0;
    for (int s = 0; s < nsets; ++s) {
      offs[s] = o;
      const int64_t ld = (widths[s] * ob + 15) / 16 * 16 / ob;
      out_lds[s] = ld > 0 ? ld : 16 / ob;
      o += static_cast<size_t>(B * out_lds[s] * ob + 15) / 16 * 16;
    }
    return o;
  };
  size_t offs[TB_MAX_REFS + 1];
  for (int pass = 0; pass < 2; ++pass) {
    const int ob = (pass == 0 && token_bytes == 8) ? 4 : token_bytes;
    if (pass == 1 && ob == token_bytes && token_bytes == 4) break;
    const size_t total = layout(ob, offs);
    const int rc = grow_pinned_rows(c, total);
    if (rc != TB_OK) {
      *rc_out = rc;
      return 0;
    }
    std::atomic<uint64_t> high{0};
    CopyPool::get().run(static_cast<int>(items_per_set * nsets), [&](int item) {
      const int s = static_cast<int>(item / items_per_set);
      const int64_t b0 = (item % items_per_set) * kRowsPerItem;
      const int64_t b1 = std::min(B, b0 + kRowsPerItem);
      unsigned char* dst = c.rows + offs[s];
      uint64_t hi = 0;
      for (int64_t b = b0; b < b1; ++b) {
        int64_t n = lens[s][b];
        n = n < 0 ? 0 : (n > widths[s] ? widths[s] : n);  // the kernel's clamp (it flags the row)
        if (token_bytes == 8 && ob == 4) {
          const int64_t* src = static_cast<const int64_t*>(src_ids[s]) + b * src_lds[s];
          int32_t* o = reinterpret_cast<int32_t*>(dst) + b * out_lds[s];
          for (int64_t j = 0; j < n; ++j) {
            const int64_t v = src[j];
            hi |= static_cast<uint64_t>(v) >> 31;
            o[j] = static_cast<int32_t>(v);
          }
        } else if (n > 0) {
          memcpy(dst + static_cast<size_t>(b * out_lds[s]) * ob,
                 static_cast<const unsigned char*>(src_ids[s]) + static_cast<size_t>(b * src_lds[s]) * token_bytes,
                 static_cast<size_t>(n) * token_bytes);
        }
      }
      if (hi) high.fetch_or(hi, std::memory_order_relaxed);
    });
    if (ob == token_bytes || high.load() == 0) {
      for (int s = 0; s < nsets; ++s) out_ids[s] = c.rows + offs[s];
      return ob;
    }
  }
  return 0;
}

enum Where { kDeviceMem = 0, kPinnedHost = 1, kPageableHost = 2 };

// Where does `p` live, and what address does the device use for it?
Where classify(const void* p, const void** dev_view) {
  *dev_view = p;
  if (!p) return kDeviceMem;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return kPageableHost;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return kDeviceMem;
  if (a.type == cudaMemoryTypeHost && a.devicePointer) {
    *dev_view = a.devicePointer;
    return kPinnedHost;
  }
  return kPageableHost;
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

extern "C" {

const char* tb_version(void) { return TB_VERSION_STRING; }

const char* tb_strerror(int code) {
  switch (code) {
    case TB_OK: return "ok";
    case TB_ERR_INVALID_ARG: return "invalid argument";
    case TB_ERR_CAPACITY: return "capacity exceeded (index space overflows int64)";
    case TB_ERR_CUDA: return "CUDA error";
    case TB_ERR_UNSUPPORTED: return "unsupported by the device path";
    case TB_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

const char* tb_last_cuda_error(void) { return g_last_cuda_error; }

#ifdef TB_PHASES
int tb_debug_phase_buffer(void* buf) {
  TB_CUDA(cudaMemcpyToSymbol(g_tb_phases, &buf, sizeof(buf)));
  return TB_OK;
}
#endif

size_t tb_bleu_workspace_bytes(int64_t batch, int32_t num_refs, int64_t cand_width,
                               const int64_t* ref_widths, int32_t token_bytes, int32_t max_order) {
  if (num_refs < 1 || num_refs > TB_MAX_REFS || max_order < 1 || max_order > TB_MAX_ORDER) return 0;
  if (token_bytes != 4 && token_bytes != 8) return 0;
  DevInfo* d = nullptr;
  int smem_optin = 227 * 1024, sms = 148;
  if (dev_info(&d) == TB_OK) {
    smem_optin = d->smem_optin;
    sms = d->sms;
  }
  Plan pl;
  if (make_plan(batch, num_refs, cand_width, ref_widths, token_bytes, max_order, smem_optin, sms, &pl) != TB_OK)
    return 0;
  return pl.ws_bytes;
}

int tb_bleu_stats(int32_t token_bytes, const void* cand_ids, int64_t cand_ld, int64_t cand_width,
                  const int64_t* cand_len, int32_t num_refs, const void* const* ref_ids,
                  const int64_t* ref_ld, const int64_t* ref_width, const int64_t* const* ref_len,
                  int64_t batch, int32_t max_order, int32_t smoothing, double eps, double k,
                  const double* weights, int64_t* num_out, int64_t* den_out, int64_t* cand_len_out,
                  int64_t* eff_ref_out, double* scores_out, double* precisions_out, double* bp_out,
                  int64_t* totals_out, double* corpus_out, int32_t* err_flag, void* workspace,
                  size_t workspace_bytes, void* stream) {
  return stats_impl(token_bytes, cand_ids, cand_ld, cand_width, cand_len, num_refs, ref_ids, ref_ld, ref_width,
                    ref_len, batch, max_order, smoothing, eps, k, weights, num_out, den_out, cand_len_out,
                    eff_ref_out, scores_out, precisions_out, bp_out, totals_out, corpus_out, err_flag, workspace,
                    workspace_bytes, stream, 0, 0);
}

// Pageable rows, per-sentence outputs, B >= 2 * kPipeRows: the batch runs in
// chunks of rows — the host threads stage chunk i + 1 (valid prefixes, int64
// narrowed to int32 when its IDs fit) while the kernel reads chunk i over
// PCIe — one launch per chunk on `stream`, one synchronisation at the end.
constexpr int64_t kPipeRows = 512;
constexpr int kPipeMaxChunks = 8;
int host_pipelined(HostCtx& c, int token_bytes, int R, const void* const* ids, const int64_t* lds,
                   const int64_t* widths, const int64_t* const* lens, int64_t B, int N, int smoothing, double eps,
                   double k, const double* weights, int64_t* num_out, int64_t* den_out, int64_t* cand_len_out,
                   int64_t* eff_ref_out, double* scores_out, double* precisions_out, double* bp_out,
                   int32_t* flags_out, cudaStream_t stream) {
  const int nsets = R + 1;
  int nchunks = static_cast<int>(B / kPipeRows);
  nchunks = nchunks < kPipeMaxChunks ? nchunks : kPipeMaxChunks;
  const int64_t rows_per = (B + nchunks - 1) / nchunks;
  // pinned staging: [err word per chunk | outputs | pageable lengths]
  struct Out { void* user; size_t bytes; size_t off; int64_t per_row; };
  Out outs[7] = {{num_out, size_t(B * N) * 8, 0, N},  {den_out, size_t(B * N) * 8, 0, N},
                 {cand_len_out, size_t(B) * 8, 0, 1}, {eff_ref_out, size_t(B) * 8, 0, 1},
                 {scores_out, size_t(B) * 8, 0, 1},   {precisions_out, size_t(B * N) * 8, 0, N},
                 {bp_out, size_t(B) * 8, 0, 1}};
  size_t off = 256;  // kPipeMaxChunks err words
  for (auto& o : outs)
    if (o.user) {
      o.off = off;
      off = align_up(off + o.bytes);
    }
  const void* v = nullptr;
  size_t len_off[TB_MAX_REFS + 1];
  const int64_t* len_dev[TB_MAX_REFS + 1];
  for (int s = 0; s < nsets; ++s) {
    len_dev[s] = nullptr;
    len_off[s] = 0;
    if (classify(lens[s], &v) == kPageableHost) {
      len_off[s] = off;
      off = align_up(off + size_t(B) * 8);
    } else {
      len_dev[s] = static_cast<const int64_t*>(v);  // pinned: its device view
    }
  }
  int rc = grow_pinned(c, off);
  if (rc != TB_OK) return rc;
  for (int s = 0; s < nsets; ++s)
    if (!len_dev[s]) {
      memcpy(c.pin + len_off[s], lens[s], size_t(B) * 8);
      len_dev[s] = reinterpret_cast<const int64_t*>(c.pin_dev + len_off[s]);
    }
  // rows: one region per (chunk, set), sized for int64 rows
  int64_t ld4[TB_MAX_REFS + 1], ld8[TB_MAX_REFS + 1];
  size_t region[TB_MAX_REFS + 1], chunk_bytes = 0;
  for (int s = 0; s < nsets; ++s) {
    ld4[s] = widths[s] > 0 ? (widths[s] + 3) / 4 * 4 : 4;
    ld8[s] = widths[s] > 0 ? (widths[s] + 1) / 2 * 2 : 2;
    const size_t a = size_t(rows_per * ld4[s]) * 4, b8 = size_t(rows_per * ld8[s]) * 8;
    region[s] = align_up(a > b8 ? a : b8);
    chunk_bytes += region[s];
  }
  rc = grow_pinned_rows(c, chunk_bytes * nchunks);
  if (rc != TB_OK) return rc;
  rc = grow_device(&c.ws, &c.ws_bytes, kAccBytes, true);  // the shared-memory plans need the completion region only
  if (rc != TB_OK) return rc;
  int32_t* err_host = reinterpret_cast<int32_t*>(c.pin);
  for (int i = 0; i < nchunks; ++i) err_host[i] = 0;
  auto P = [&](int i, int64_t b0) -> void* {
    return outs[i].user ? c.pin_dev + outs[i].off + size_t(b0 * outs[i].per_row) * 8 : nullptr;
  };
  for (int ci = 0; ci < nchunks; ++ci) {
    const int64_t b0 = ci * rows_per;
    const int64_t b1 = b0 + rows_per < B ? b0 + rows_per : B;
    if (b1 <= b0) break;
    unsigned char* dst[TB_MAX_REFS + 1];
    const void* dev_ids[TB_MAX_REFS + 1];
    size_t o = chunk_bytes * ci;
    for (int s = 0; s < nsets; ++s) {
      dst[s] = c.rows + o;
      dev_ids[s] = c.rows_dev + o;
      o += region[s];
    }
    int ob = token_bytes == 8 ? 4 : token_bytes;
    const int64_t* dlds = ob == 4 ? ld4 : ld8;
    if (copy_rows(token_bytes, ob, nsets, ids, lds, widths, lens, b0, b1, dst, dlds) != 0) {
      ob = 8;  // an ID >= 2^31 in this chunk: stage it as int64
      dlds = ld8;
      copy_rows(token_bytes, ob, nsets, ids, lds, widths, lens, b0, b1, dst, dlds);
    }
    const int64_t* lchunk[TB_MAX_REFS + 1];
    for (int s = 0; s < nsets; ++s) lchunk[s] = len_dev[s] + b0;
    rc = stats_impl(ob, dev_ids[0], dlds[0], widths[0], lchunk[0], R, dev_ids + 1, dlds + 1, widths + 1, lchunk + 1,
                    b1 - b0, N, smoothing, eps, k, weights, static_cast<int64_t*>(P(0, b0)),
                    static_cast<int64_t*>(P(1, b0)), static_cast<int64_t*>(P(2, b0)),
                    static_cast<int64_t*>(P(3, b0)), static_cast<double*>(P(4, b0)),
                    static_cast<double*>(P(5, b0)), static_cast<double*>(P(6, b0)), nullptr, nullptr,
                    reinterpret_cast<int32_t*>(c.pin_dev) + ci, c.ws, c.ws_bytes, stream, 1, 1);
    if (rc != TB_OK) return rc;
  }
  TB_CUDA(cudaStreamSynchronize(stream));
  for (auto& ou : outs)
    if (ou.user && ou.bytes) memcpy(ou.user, c.pin + ou.off, ou.bytes);
  int32_t flags = 0;
  for (int i = 0; i < nchunks; ++i) flags |= reinterpret_cast<volatile int32_t*>(err_host)[i];
  *flags_out = flags;
  return TB_OK;
}

int tb_bleu_host(int32_t token_bytes, const void* cand_ids, int64_t cand_ld, int64_t cand_width,
                 const int64_t* cand_len, int32_t num_refs, const void* const* ref_ids,
                 const int64_t* ref_ld, const int64_t* ref_width, const int64_t* const* ref_len,
                 int64_t batch, int32_t max_order, int32_t smoothing, double eps, double k,
                 const double* weights, int64_t* num_out, int64_t* den_out, int64_t* cand_len_out,
                 int64_t* eff_ref_out, double* scores_out, double* precisions_out, double* bp_out,
                 int64_t* totals_out, double* corpus_out, int32_t* flags_out, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (token_bytes != 4 && token_bytes != 8) return TB_ERR_INVALID_ARG;
  if (num_refs < 1) return TB_ERR_INVALID_ARG;
  if (num_refs > TB_MAX_REFS) return TB_ERR_UNSUPPORTED;
  if (batch < 0 || cand_width < 0 || cand_ld < cand_width || !flags_out) return TB_ERR_INVALID_ARG;
  if (!ref_ids || !ref_ld || !ref_width || !ref_len) return TB_ERR_INVALID_ARG;
  int rc = check_epi(max_order, smoothing, eps, k, weights);
  if (rc != TB_OK) return rc;
  for (int r = 0; r < num_refs; ++r) {
    if (ref_width[r] < 0 || ref_ld[r] < ref_width[r]) return TB_ERR_INVALID_ARG;
    if (batch > 0 && (!ref_len[r] || (!ref_ids[r] && ref_width[r] > 0))) return TB_ERR_INVALID_ARG;
  }
  if (batch > 0 && ((!cand_ids && cand_width > 0) || !cand_len)) return TB_ERR_INVALID_ARG;
  const int R = num_refs, N = max_order;

  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return TB_ERR_UNSUPPORTED;
  HostCtx& c = g_host[dev];
  DevInfo* d = nullptr;
  rc = dev_info(&d);
  if (rc != TB_OK) return rc;
  const int64_t B = batch;
  const void* ids_in[TB_MAX_REFS + 1];
  const int64_t* len_in[TB_MAX_REFS + 1];
  int64_t lds[TB_MAX_REFS + 1], widths[TB_MAX_REFS + 1];
  ids_in[0] = cand_ids;
  len_in[0] = cand_len;
  lds[0] = cand_ld;
  widths[0] = cand_width;
  for (int r = 0; r < R; ++r) {
    ids_in[r + 1] = ref_ids[r];
    len_in[r + 1] = ref_len[r];
    lds[r + 1] = ref_ld[r];
    widths[r + 1] = ref_width[r];
  }
  // Pageable token rows (e.g. numpy arrays): copy their valid prefixes into
  // pinned memory with the host thread pool — narrowed to int32 when every ID
  // fits — for the kernel to read over PCIe, when the shared-memory kernels
  // take the rows (they stage valid prefixes).  Otherwise the rows are DMA'd
  // whole below.
  // (Pinned rows are read in place: staging pinned int64 rows to narrow them
  // lost on cold data — the copy reads 8 bytes per token from DRAM.)
  if (B > 0) {
    bool pageable = true;
    for (int s = 0; s <= R && pageable; ++s) {
      const void* v = nullptr;
      if (classify(len_in[s], &v) == kDeviceMem) pageable = false;
      if (widths[s] > 0 && classify(ids_in[s], &v) != kPageableHost) pageable = false;
    }
    Plan probe, probe8;
    const bool corpus_mode = totals_out != nullptr || corpus_out != nullptr;
    if (pageable && !corpus_mode && B >= 2 * kPipeRows &&
        make_plan(kPipeRows, R, cand_width, ref_width, 4, N, d->smem_optin, d->sms, &probe) == TB_OK &&
        probe.smem_mode &&
        make_plan(kPipeRows, R, cand_width, ref_width, 8, N, d->smem_optin, d->sms, &probe8) == TB_OK &&
        probe8.smem_mode)
      return host_pipelined(c, token_bytes, R, ids_in, lds, widths, len_in, B, N, smoothing, eps, k, weights,
                            num_out, den_out, cand_len_out, eff_ref_out, scores_out, precisions_out, bp_out,
                            flags_out, stream);
    if (pageable && make_plan(B, R, cand_width, ref_width, 4, N, d->smem_optin, d->sms, &probe) == TB_OK &&
        probe.smem_mode) {
      int src = TB_OK;
      const int tb = stage_pageable_rows(c, token_bytes, R + 1, ids_in, lds, widths, len_in, B, ids_in, lds, &src);
      if (src != TB_OK) return src;
      if (tb) token_bytes = tb;
    }
  }
  Plan pl;
  if (batch > 0) {
    rc = make_plan(batch, R, cand_width, ref_width, token_bytes, N, d->smem_optin, d->sms, &pl);
    if (rc != TB_OK) return rc;
  }
  rc = grow_device(&c.ws, &c.ws_bytes, pl.ws_bytes > kAccBytes ? pl.ws_bytes : kAccBytes, true);
  if (rc != TB_OK) return rc;

  // ---- pinned staging layout: [err | outputs | pageable lengths]
  struct Out { void* user; size_t bytes; size_t off; };
  Out outs[9] = {{num_out, size_t(B * N) * 8, 0},   {den_out, size_t(B * N) * 8, 0},
                 {cand_len_out, size_t(B) * 8, 0},  {eff_ref_out, size_t(B) * 8, 0},
                 {scores_out, size_t(B) * 8, 0},    {precisions_out, size_t(B * N) * 8, 0},
                 {bp_out, size_t(B) * 8, 0},        {totals_out, size_t(2 * N + 2) * 8, 0},
                 {corpus_out, size_t(N + 2) * 8, 0}};
  size_t off = 256;  // err word
  for (auto& o : outs)
    if (o.user) {
      o.off = off;
      off = align_up(off + o.bytes);
    }
  const void* ids_dev[TB_MAX_REFS + 1];
  const int64_t* len_dev[TB_MAX_REFS + 1];
  Where len_where[TB_MAX_REFS + 1];
  size_t len_off[TB_MAX_REFS + 1];
  bool need_stage[TB_MAX_REFS + 1];
  size_t stage_off[TB_MAX_REFS + 1];
  size_t stage_total = 0;
  bool zero_copy = false;
  for (int s = 0; s <= R; ++s) {
    const void* v = nullptr;
    len_where[s] = B > 0 ? classify(len_in[s], &v) : kDeviceMem;
    len_dev[s] = static_cast<const int64_t*>(v);
    len_off[s] = 0;
    if (len_where[s] == kPageableHost) {
      len_off[s] = off;
      off = align_up(off + size_t(B) * 8);
    }
    need_stage[s] = false;
    stage_off[s] = 0;
    ids_dev[s] = ids_in[s];
    if (B == 0 || widths[s] == 0) continue;
    const void* iv = nullptr;
    const Where w = classify(ids_in[s], &iv);
    if (w == kDeviceMem) continue;
    if (w == kPinnedHost && pl.smem_mode) {  // the kernel reads the valid prefixes over PCIe
      ids_dev[s] = iv;
      zero_copy = true;
      continue;
    }
    need_stage[s] = true;
    stage_off[s] = stage_total;
    stage_total = align_up(stage_total + size_t((B - 1) * lds[s] + widths[s]) * token_bytes);
  }
  rc = grow_pinned(c, off);
  if (rc != TB_OK) return rc;
  if (stage_total) {
    rc = grow_device(reinterpret_cast<void**>(&c.dstage), &c.dstage_bytes, stage_total, false);
    if (rc != TB_OK) return rc;
  }
  for (int s = 0; s <= R; ++s) {
    if (len_where[s] == kPageableHost) {
      memcpy(c.pin + len_off[s], len_in[s], size_t(B) * 8);
      len_dev[s] = reinterpret_cast<const int64_t*>(c.pin_dev + len_off[s]);
    }
    if (need_stage[s]) {
      const size_t bytes = size_t((B - 1) * lds[s] + widths[s]) * token_bytes;
      TB_CUDA(cudaMemcpyAsync(c.dstage + stage_off[s], ids_in[s], bytes, cudaMemcpyHostToDevice, stream));
      ids_dev[s] = c.dstage + stage_off[s];
    }
  }
  auto P = [&](int i) -> void* { return outs[i].user ? c.pin_dev + outs[i].off : nullptr; };
  int32_t* err_host = reinterpret_cast<int32_t*>(c.pin);
  *err_host = 0;
  rc = stats_impl(token_bytes, ids_dev[0], lds[0], cand_width, len_dev[0], R, ids_dev + 1, lds + 1, ref_width,
                  len_dev + 1, B, N, smoothing, eps, k, weights, static_cast<int64_t*>(P(0)),
                  static_cast<int64_t*>(P(1)), static_cast<int64_t*>(P(2)), static_cast<int64_t*>(P(3)),
                  static_cast<double*>(P(4)), static_cast<double*>(P(5)), static_cast<double*>(P(6)),
                  static_cast<int64_t*>(P(7)), static_cast<double*>(P(8)), reinterpret_cast<int32_t*>(c.pin_dev),
                  c.ws, c.ws_bytes, stream, zero_copy ? 1 : 0, 1);
  if (rc != TB_OK) return rc;
  TB_CUDA(cudaStreamSynchronize(stream));
  for (auto& o : outs)
    if (o.user && o.bytes) memcpy(o.user, c.pin + o.off, o.bytes);
  *flags_out = *reinterpret_cast<volatile int32_t*>(err_host);
  return TB_OK;
}

int tb_bleu_scores(const int64_t* num, const int64_t* den, const int64_t* cand_len,
                   const int64_t* eff_ref, int64_t batch, int32_t max_order, int32_t smoothing,
                   double eps, double k, const double* weights, double* scores_out,
                   double* precisions_out, double* bp_out, void* stream) {
  int rc = check_epi(max_order, smoothing, eps, k, weights);
  if (rc != TB_OK) return rc;
  if (batch < 0) return TB_ERR_INVALID_ARG;
  if (batch == 0) return TB_OK;
  if (!num || !den || !cand_len || !eff_ref) return TB_ERR_INVALID_ARG;
  EpiParams e;
  fill_epi(&e, max_order, smoothing, eps, k, weights);
  const int threads = 128;
  int64_t blocks = (batch + threads - 1) / threads;
  if (blocks > 65535) blocks = 65535;
  bleu_scores_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      num, den, cand_len, eff_ref, batch, max_order, e, scores_out, precisions_out, bp_out);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_bleu_totals(const int64_t* num, const int64_t* den, const int64_t* cand_len,
                   const int64_t* eff_ref, int64_t batch, int32_t max_order, int64_t* totals_out,
                   void* stream) {
  if (max_order < 1) return TB_ERR_INVALID_ARG;
  if (max_order > TB_MAX_ORDER) return TB_ERR_UNSUPPORTED;
  if (batch < 0 || !totals_out) return TB_ERR_INVALID_ARG;
  if (batch > 0 && (!num || !den || !cand_len || !eff_ref)) return TB_ERR_INVALID_ARG;
  bleu_totals_kernel<<<2 * max_order + 2, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      num, den, cand_len, eff_ref, batch, max_order, totals_out);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_validate_batch(int32_t token_bytes, const void* ids, int64_t ld, int64_t width,
                      const int64_t* lengths, int64_t batch, int32_t* err_flag, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (token_bytes != 4 && token_bytes != 8) return TB_ERR_INVALID_ARG;
  if (batch < 0 || width < 0 || ld < width || !err_flag) return TB_ERR_INVALID_ARG;
  if (batch == 0) return TB_OK;
  if (!lengths || (!ids && width > 0)) return TB_ERR_INVALID_ARG;
  int64_t grid = batch < 4096 ? batch : 4096;
  if (token_bytes == 4)
    validate_batch_kernel<int32_t><<<static_cast<unsigned>(grid), 256, 0, stream>>>(
        static_cast<const int32_t*>(ids), ld, width, lengths, batch, err_flag);
  else
    validate_batch_kernel<int64_t><<<static_cast<unsigned>(grid), 256, 0, stream>>>(
        static_cast<const int64_t*>(ids), ld, width, lengths, batch, err_flag);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

}  // extern "C"
