// tb_runtime.cu — shape planning, launches, the host-buffer path (pinned /
// pageable staging, copy pool) and the C ABI of include/tensorbleu.h.
// (see tb_common.cuh for the source layout)

#include "tb_launch.cuh"

namespace tbk {

thread_local char g_last_cuda_error[256] = "";

int cuda_fail(cudaError_t e) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
  return TB_ERR_CUDA;
}

}  // namespace tbk

namespace {

// --------------------------------------------------------------------------
// Stand-alone epilogue / totals / validation kernels.
// --------------------------------------------------------------------------

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

// Any max_order, weights in device memory; R = double (fp64, numpy's
// operation order as bleu_epilogue: explicit round-to-nearest operations, no
// FMA contraction) or float (the fp32 epilogue: the same operations in single
// precision, outputs float).  One thread per sentence.
__device__ __forceinline__ double r_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double r_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double r_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double r_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double r_log(double a) { return log(a); }
__device__ __forceinline__ double r_exp(double a) { return exp(a); }
__device__ __forceinline__ float r_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float r_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float r_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float r_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float r_log(float a) { return logf(a); }
__device__ __forceinline__ float r_exp(float a) { return expf(a); }

template <typename R>
__global__ void bleu_scores_any_kernel(const int64_t* __restrict__ num, const int64_t* __restrict__ den,
                                       const int64_t* __restrict__ cand_len, const int64_t* __restrict__ eff_ref,
                                       int64_t batch, int N, int smoothing, double eps, double kk,
                                       const double* __restrict__ w, R* scores, R* precisions, R* bp_out) {
  const R eps_r = static_cast<R>(eps), k_r = static_cast<R>(kk);
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < batch;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // _bp_vector, bleu.py:256-261: 0 for an empty candidate, 1 if c > r, else exp(1 - r/c)
    const R cd = static_cast<R>(cand_len[b]);
    const R rd = static_cast<R>(eff_ref[b]);
    R bp = cd > rd ? R(1) : r_exp(r_sub(R(1), r_div(rd, cd > R(0) ? cd : R(1))));
    if (!(cd > R(0))) bp = R(0);
    R counter = 1, s = 0;
    bool ok = true;
    for (int n = 0; n < N; ++n) {
      const int64_t nn = num[b * N + n], dn = den[b * N + n];
      const R nd = static_cast<R>(nn), dd = static_cast<R>(dn);
      const bool has_den = dn > 0;
      R pn = (has_den && nn != 0) ? r_div(nd, dd) : R(0);      // bleu.py:222
      const bool zero_num = has_den && nn == 0;                 // bleu.py:223
      if (smoothing == TB_SMOOTH_FLOOR) {
        if (zero_num) pn = r_div(eps_r, dd);                    // bleu.py:228
      } else if (smoothing == TB_SMOOTH_ADD_K) {
        if (n >= 1 && has_den) pn = r_div(r_add(nd, k_r), r_add(dd, k_r));  // bleu.py:230-232
      } else if (smoothing == TB_SMOOTH_EXP) {
        if (zero_num) {                                         // bleu.py:234-238, exact 2^counter
          pn = r_div(R(1), r_mul(static_cast<R>(ldexp(1.0, static_cast<int>(counter))), dd));
          counter = r_add(counter, R(1));
        }
      }
      if (precisions) precisions[b * N + n] = pn;
      const R wn = static_cast<R>(w[n]);
      if (wn > R(0)) {                                          // bleu.py:242-253, sequential sum
        if (pn > R(0))
          s = r_add(s, r_mul(r_log(pn), wn));
        else
          ok = false;
      }
    }
    R score = ok ? r_mul(bp, r_exp(s)) : R(0);
    score = score < R(0) ? R(0) : (score > R(1) ? R(1) : score);
    if (bp_out) bp_out[b] = bp;
    if (scores) scores[b] = score;
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


int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int cap_log2_for(int64_t want, int min_log2) {
  int c = min_log2;
  while ((int64_t(1) << c) < want) ++c;
  return c;
}

// The warp-per-group kernel goes first when the rows are narrow enough; the
// CTA-per-group plan already made scores the groups it lists (a count and B
// int32 group indices after the completion region).  TB_NO_SPARSE=1 turns it
// off (A/B measurements).
void use_sparse(Plan* pl, int64_t batch, int R, int64_t cand_width, const int64_t* ref_widths, int token_bytes,
                int smem_optin) {
  static const bool off = [] {
    const char* e = getenv("TB_NO_SPARSE");
    return e && e[0] == '1';
  }();
  static const bool force = [] {
    const char* e = getenv("TB_FORCE_SPARSE");
    return e && e[0] == '1';
  }();
  if (off || R > kSparseMaxRefs || cand_width > kSparseMaxWidth || batch > INT32_MAX) return;
  // Measured on B200: the filter kernel wins for long rows in
  // many waves (c5 2048-token rows: 263 -> 194 us); for <= 1024-token rows the
  // hash-table kernel alone is as fast or faster (c4 37.6 vs 41.5 us with the
  // list handoff; c2 7.5 vs 13.5 us), so it keeps them.  TB_FORCE_SPARSE=1
  // takes the filter kernel for every shape (tests, A/B runs).
  if (!force && (cand_width <= 1024 || batch < 8 * 148)) return;
  // one group slot (tb_kernel_sparse.cu launch_sparse) must fit with room to spare
  int64_t fc = 4096;  // Fc bytes: >= 16 per candidate position (tb_kernel_sparse.cu launch_sparse)
  while (fc < 16 * cand_width) fc *= 2;
  int64_t slot = fc + 2048 + 128 * token_bytes + 512 + 896 + 1024;
  for (int s = 0; s <= R; ++s) {
    const int64_t w = s == 0 ? cand_width : ref_widths[s - 1];
    if (w > kSparseMaxWidth) return;
    slot += (w * token_bytes + 16 + 15) / 16 * 16;
  }
  if (slot > smem_optin - 8192) return;
  pl->sparse = true;
  pl->list_off = pl->acc_bytes;
  pl->ws_bytes = pl->acc_bytes + static_cast<size_t>(round_up(16 + 4 * batch, 256));
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
      use_sparse(pl, batch, R, cand_width, ref_widths, token_bytes, smem_optin);
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
    while (total + static_cast<int64_t>(kMultiStaticReserve) > smem_optin / 2 && (int64_t(1) << (lg - 1)) >= 2 * cpad4) {
      --lg;
      total = multi_layout(lg, offs);
    }
    if (lg <= 15 && ptot < 65535 && total + static_cast<int64_t>(kMultiStaticReserve) <= smem_optin) {
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
      use_sparse(pl, batch, R, cand_width, ref_widths, token_bytes, smem_optin);
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

int launch_stats(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes) {
  if (pl.sparse) {  // warp per group; then the listed dense groups, CTA per group
    const int rc = launch_sparse(prm, sms, stream, token_bytes);
    if (rc != TB_OK) return rc;
    // TB_DEBUG_NO_DENSE=1: timing experiments only (results are wrong if a group was listed)
    static const bool no_dense = [] {
      const char* e = getenv("TB_DEBUG_NO_DENSE");
      return e && e[0] == '1';
    }();
    if (no_dense) return TB_OK;
  }
  if (pl.pair) return launch_pair(prm, pl, sms, stream, token_bytes);
  if (pl.multi) return launch_multi(prm, pl, sms, stream, token_bytes);
  if (pl.smem_mode) return launch_group(prm, pl, sms, stream, token_bytes);
  return launch_global(prm, pl, sms, stream, token_bytes);
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
  {  // full-width bulk copies take every row whole when bases, pitches and widths are 16-byte multiples
    auto whole = [&](const void* base, int64_t ld, int64_t width) {
      return (reinterpret_cast<uintptr_t>(base) & 15) == 0 && ((ld * token_bytes) & 15) == 0 &&
             ((width * token_bytes) & 15) == 0;
    };
    bool nt = !prm.prefix_only && whole(cand_ids, cand_ld, cand_width);
    for (int r = 0; r < num_refs && nt; ++r) nt = whole(ref_ids[r], ref_ld[r], ref_width[r]);
    prm.no_tails = nt ? 1 : 0;
  }
  if (pl.sparse) {
    prm.gcount = reinterpret_cast<unsigned int*>(ws + pl.list_off);
    prm.glist = reinterpret_cast<int*>(ws + pl.list_off + 16);
  }

  return launch_stats(prm, pl, d->sms, stream, token_bytes);
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
// Host-call contexts: a per-device pool shared by all calling threads (a
// call takes one for its duration and gives it back), so concurrent calls
// get separate buffers and threads that exit leave nothing behind.
struct HostPool {
  std::mutex m;
  std::vector<HostCtx*> free_list;
};
HostPool g_host_pool[64];

struct HostLease {  // RAII: a context of device `dev` for one call
  int dev;
  HostCtx* c;
  explicit HostLease(int d) : dev(d), c(nullptr) {
    std::lock_guard<std::mutex> l(g_host_pool[dev].m);
    auto& fl = g_host_pool[dev].free_list;
    if (!fl.empty()) {
      c = fl.back();
      fl.pop_back();
    }
    if (!c) c = new HostCtx();
  }
  ~HostLease() {
    std::lock_guard<std::mutex> l(g_host_pool[dev].m);
    g_host_pool[dev].free_list.push_back(c);
  }
};

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
  // TB_COPY_THREADS: worker threads (default min(7, cores/2 - 1));
  // TB_COPY_SPIN_US: how long an idle worker spins for the next job before it
  // sleeps (default 200 us; calls usually come back to back)
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    int nt = std::max(0, std::min(7, static_cast<int>(hw / 2) - 1));
    if (const char* e = getenv("TB_COPY_THREADS")) nt = std::max(0, std::min(64, atoi(e)));
    if (const char* e = getenv("TB_COPY_SPIN_US")) spin_us_ = std::max(0, atoi(e));
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
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(spin_us_)) {
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#else
        std::this_thread::yield();
#endif
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
  int spin_us_ = 200;
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
  int rc = set_phases_pair(buf);
  if (rc == TB_OK) rc = set_phases_multi(buf);
  if (rc == TB_OK) rc = set_phases_group(buf);
  return rc;
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
  StreamDeviceGuard device_guard(stream);
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
  {  // the shared-memory plans need the completion region (+ the dense-group list)
    size_t want = kAccBytes;
    DevInfo* d = nullptr;
    rc = dev_info(&d);
    if (rc != TB_OK) return rc;
    for (int tbytes = 4; tbytes <= 8; tbytes += 4) {
      Plan cp;
      if (make_plan(rows_per, R, widths[0], widths + 1, tbytes, N, d->smem_optin, d->sms, &cp) == TB_OK &&
          cp.ws_bytes > want)
        want = cp.ws_bytes;
    }
    rc = grow_device(&c.ws, &c.ws_bytes, want, true);
    if (rc != TB_OK) return rc;
  }
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
  StreamDeviceGuard device_guard(stream_);
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
  HostLease lease(dev);
  HostCtx& c = *lease.c;
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
  StreamDeviceGuard device_guard(stream);
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
  StreamDeviceGuard device_guard(stream);
  if (max_order < 1) return TB_ERR_INVALID_ARG;  // any order: one CTA per output column
  if (batch < 0 || !totals_out) return TB_ERR_INVALID_ARG;
  if (batch > 0 && (!num || !den || !cand_len || !eff_ref)) return TB_ERR_INVALID_ARG;
  bleu_totals_kernel<<<2 * max_order + 2, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      num, den, cand_len, eff_ref, batch, max_order, totals_out);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_bleu_scores_any(const int64_t* num, const int64_t* den, const int64_t* cand_len, const int64_t* eff_ref,
                       int64_t batch, int32_t max_order, int32_t smoothing, double eps, double k,
                       const double* weights_dev, int32_t fp32, void* scores_out, void* precisions_out, void* bp_out,
                       void* stream) {
  StreamDeviceGuard device_guard(stream);
  if (max_order < 1 || smoothing < TB_SMOOTH_NONE || smoothing > TB_SMOOTH_EXP || !(eps > 0) || !(k > 0))
    return TB_ERR_INVALID_ARG;
  if (batch < 0) return TB_ERR_INVALID_ARG;
  if (batch == 0) return TB_OK;
  if (!num || !den || !cand_len || !eff_ref || !weights_dev) return TB_ERR_INVALID_ARG;
  const int threads = 128;
  int64_t blocks = (batch + threads - 1) / threads;
  if (blocks > 65535) blocks = 65535;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fp32)
    bleu_scores_any_kernel<float><<<static_cast<unsigned>(blocks), threads, 0, st>>>(
        num, den, cand_len, eff_ref, batch, max_order, smoothing, eps, k, weights_dev,
        static_cast<float*>(scores_out), static_cast<float*>(precisions_out), static_cast<float*>(bp_out));
  else
    bleu_scores_any_kernel<double><<<static_cast<unsigned>(blocks), threads, 0, st>>>(
        num, den, cand_len, eff_ref, batch, max_order, smoothing, eps, k, weights_dev,
        static_cast<double*>(scores_out), static_cast<double*>(precisions_out), static_cast<double*>(bp_out));
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_validate_host(int32_t token_bytes, const void* ids, int64_t ld, int64_t width, const int64_t* lengths,
                     int64_t batch) {
  if (token_bytes != 4 && token_bytes != 8) return -TB_ERR_INVALID_ARG;
  if (batch < 0 || width < 0 || ld < width) return -TB_ERR_INVALID_ARG;
  if (batch == 0) return 0;
  if (!lengths || (!ids && width > 0)) return -TB_ERR_INVALID_ARG;
  for (int64_t b = 0; b < batch; ++b)  // batch.py:30-31, checked first
    if (lengths[b] < 0 || lengths[b] > width) return TB_FLAG_BAD_LENGTH;
  // batch.py:32-34: the OR of the valid IDs of a block of rows has its sign
  // bit set iff one of them is negative
  auto rows_negative = [&](int64_t r0, int64_t r1) -> bool {
    if (token_bytes == 8) {
      const int64_t* p = static_cast<const int64_t*>(ids);
      for (int64_t b = r0; b < r1; ++b) {
        const int64_t* row = p + b * ld;
        int64_t acc = 0;
        for (int64_t j = 0; j < lengths[b]; ++j) acc |= row[j];
        if (acc < 0) return true;
      }
    } else {
      const int32_t* p = static_cast<const int32_t*>(ids);
      for (int64_t b = r0; b < r1; ++b) {
        const int32_t* row = p + b * ld;
        int32_t acc = 0;
        for (int64_t j = 0; j < lengths[b]; ++j) acc |= row[j];
        if (acc < 0) return true;
      }
    }
    return false;
  };
  int64_t tokens = 0;
  for (int64_t b = 0; b < batch; ++b) tokens += lengths[b];
  if (tokens < (int64_t(1) << 16)) return rows_negative(0, batch) ? TB_FLAG_NEGATIVE_ID : 0;
  constexpr int64_t kRows = 32;
  const int64_t items = (batch + kRows - 1) / kRows;
  std::atomic<int> neg{0};
  CopyPool::get().run(static_cast<int>(items), [&](int item) {
    if (neg.load(std::memory_order_relaxed)) return;
    const int64_t r0 = item * kRows;
    if (rows_negative(r0, std::min(batch, r0 + kRows))) neg.store(1, std::memory_order_relaxed);
  });
  return neg.load() ? TB_FLAG_NEGATIVE_ID : 0;
}

int tb_validate_batch(int32_t token_bytes, const void* ids, int64_t ld, int64_t width,
                      const int64_t* lengths, int64_t batch, int32_t* err_flag, void* stream_) {
  StreamDeviceGuard device_guard(stream_);
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
