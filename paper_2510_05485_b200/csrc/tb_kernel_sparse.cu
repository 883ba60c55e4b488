// tb_kernel_sparse.cu — filter kernel: one CTA per sentence group (1 <= R <= kSparseMaxRefs).
// (see tb_common.cuh for the source layout, DESIGN.md §3.0 for the design)
//
// A CTA of NT threads (128 or 256) scores one sentence group (candidate i and
// its R references) at a time, grid-striding over the batch; the rows of the
// group after the current one are staged into the other half of a double
// buffer by bulk copies (TMA engine) while the current one is counted, so a
// CTA rarely waits for memory.  Per group:
//   1. the candidate's tokens set one bit each in Fc, a 2^17..2^18-bit filter
//      (>= 128 bits per candidate position: ~0.6% false positives);
//   2. every reference token is tested against Fc; the survivors (the tokens
//      that may occur in the candidate) are listed and set a bit in Fs;
//   3. the candidate's tokens are tested against Fs; survivors listed.
//   A token occurring on both sides is listed from both sides (no false
//   negatives), and an n-gram present on both sides has all its tokens listed,
//   so the list holds everything that can contribute to a clipped count.
//   4. warp 0 sorts the S listed elements by (row, position) and counts
//      exactly: S <= 32 with match.any per order (element e in lane e; the
//      order-n key is (id of the (n-1)-gram at e, id of the token at e+n-1),
//      an id being the lowest lane holding the key; the (n-1)-grams at e and
//      e+1 must both have matched — exact pruning); 32 < S <= kSparseMax with
//      a tiny hash table per order.  Both clip as the reference does:
//      Σ_key min(candidate count, max_r reference_r count).
//   5. the fp64 epilogue (lane n = order n).
// Every token costs a handful of instructions per pass (one multiply, one
// shift for the word, one funnel shift for the bit, one shared-memory access).
// A group with more than kSparseMax survivors (related text) is appended to
// the dense list in the workspace and scored by the CTA-per-group hash-table
// kernel that follows in the same stream (pair / multi kernel in list mode);
// that kernel also finishes the corpus totals and the error flags.

#include "tb_launch.cuh"

#include <algorithm>

namespace {

constexpr int kFsWords = 512;    // Fs: 16384 bits

// Filters: word from the top bits of h = tok_hash32(t), bit from its low five
// bits; bit_of(s) = 1 << (s & 31) in one funnel shift.

// Four tokens of a row at positions q..q+3 (q multiple of 4, q < len).  Vector
// loads when the row is 16-byte aligned and q+4 <= width (the row's padding is
// readable memory); otherwise positions >= len read as 0.  Callers mask
// positions >= len where it matters.
template <typename T>
__device__ __forceinline__ void load_quad(const T* row, int q, int len, int width, bool vec, T (&t)[4]) {
  if (vec && q + 4 <= width) {
    if constexpr (sizeof(T) == 4) {
      const int4 v = __ldg(reinterpret_cast<const int4*>(row + q));
      t[0] = v.x;
      t[1] = v.y;
      t[2] = v.z;
      t[3] = v.w;
    } else {
      const longlong2 u = __ldg(reinterpret_cast<const longlong2*>(row + q));
      const longlong2 v = __ldg(reinterpret_cast<const longlong2*>(row + q + 2));
      t[0] = u.x;
      t[1] = u.y;
      t[2] = v.x;
      t[3] = v.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = q + k < len ? __ldg(row + q + k) : T(0);
  }
}

template <typename T>
__device__ __forceinline__ void store_quad(T* dst, const T (&t)[4]) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<int4*>(dst) = make_int4(t[0], t[1], t[2], t[3]);
  } else {
    reinterpret_cast<longlong2*>(dst)[0] = make_longlong2(t[0], t[1]);
    reinterpret_cast<longlong2*>(dst)[1] = make_longlong2(t[2], t[3]);
  }
}
template <typename T>
__device__ __forceinline__ void lds_quad(const T* src, T (&t)[4]) {
  if constexpr (sizeof(T) == 4) {
    const int4 v = *reinterpret_cast<const int4*>(src);
    t[0] = v.x;
    t[1] = v.y;
    t[2] = v.z;
    t[3] = v.w;
  } else {
    const longlong2 u = reinterpret_cast<const longlong2*>(src)[0];
    const longlong2 v = reinterpret_cast<const longlong2*>(src)[1];
    t[0] = u.x;
    t[1] = u.y;
    t[2] = v.x;
    t[3] = v.y;
  }
}


template <typename T, int NT>
__global__ void __launch_bounds__(NT, (sizeof(T) == 4 ? 1024 : 768) / NT)
    bleu_sparse_kernel(const __grid_constant__ StatsParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t s_mbar[2];
  __shared__ int s_cnt[2];         // reference / candidate elements listed
  __shared__ int s_len[3][16];     // clamped lengths of the groups in flight (3 buffers)
  __shared__ unsigned long long s_tot[2 * TB_MAX_ORDER + 2];
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  uint32_t* const fc = reinterpret_cast<uint32_t*>(smem + p.sp_off_fc);
  uint32_t* const fs = reinterpret_cast<uint32_t*>(smem + p.sp_off_fs);
  T* const etok = reinterpret_cast<T*>(smem + p.sp_off_tok);
  uint32_t* const eps = reinterpret_cast<uint32_t*>(smem + p.sp_off_ps);  // (row << 16) | position
  unsigned char* const aux = smem + p.sp_off_aux;
  const int nbuf = p.sp_nbuf;  // 1 or 2 row buffers
  T* const rows0 = reinterpret_cast<T*>(smem + p.sp_off_rows);

  const int N = p.max_order;
  const int R = p.num_refs;
  const bool corpus = p.totals != nullptr || p.corpus != nullptr;
  const uint32_t fc_quads = (1u << p.filter_log2) / 4;
  const uint32_t wshift = 32 - p.filter_log2;
  constexpr int kStager = NT / 32 - 1;  // the last warp stages rows
  const bool stager = (tid >> 5) == kStager;
  int flags = 0;

  if (tid == 0) {
    mbar_init(&s_mbar[0], 1);
    mbar_init(&s_mbar[1], 1);
  }
  griddep_wait_and_release();
  const int64_t stride = gridDim.x;

  // The stager warp reads a group's lengths (lane s: row s) one group ahead
  // and lane s issues one bulk copy of row s's valid prefix rounded up to 16
  // bytes (in bounds: the row pitch is a multiple of 16 bytes — rows without
  // that, flagged off in sp_tma_mask, are copied by the whole CTA with plain
  // loads after the wait).
  int64_t nlen = 0;
  auto load_len = [&](int64_t g) {
    nlen = 0;
    if (g < p.batch && lane <= R) nlen = lane == 0 ? p.cand_len[g] : p.refs[lane - 1].len[g];
  };
  auto stage = [&](int64_t g, int buf, int lbuf) {
    int64_t l = nlen;
    uint32_t bytes = 0;
    if (lane <= R) {
      const int64_t w = row_width(p, lane);
      if (l < 0 || l > w) {
        flags |= TB_FLAG_BAD_LENGTH;
        l = l < 0 ? 0 : w;
      }
      s_len[lbuf][lane] = static_cast<int>(l);
      if (p.sp_tma_mask >> lane & 1)
        bytes = static_cast<uint32_t>((l * static_cast<int64_t>(sizeof(T)) + 15) & ~int64_t(15));
    }
    const uint32_t total = __reduce_add_sync(kFull, bytes);
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&s_mbar[buf], total);
    }
    __syncwarp();
    if (bytes)
      bulk_g2s(rows0 + buf * p.sp_buf_elems + p.sp_row_off[lane], row_src<T>(p, lane, g), bytes, &s_mbar[buf]);
  };

  const int64_t b0 = blockIdx.x;
  if (stager) load_len(b0);
  __syncthreads();  // the mbarriers are initialised before the first copy arrives on them
  if (stager) {
    if (b0 < p.batch) stage(b0, 0, 0);
    load_len(b0 + stride);
    if (nbuf == 2) {
      if (b0 + stride < p.batch) stage(b0 + stride, 1, 1);
      load_len(b0 + 2 * stride);
    }
  }
  uint32_t phases = 0;

  int it = 0;
  for (int64_t b = b0; b < p.batch; b += stride, ++it) {
    const int cur = nbuf == 2 ? (it & 1) : 0;
    const int lb = it % 3;
    T* const rows = rows0 + cur * p.sp_buf_elems;
    if (tid == 0) {
      s_cnt[0] = 0;
      s_cnt[1] = 0;
    }
    for (uint32_t i = tid; i < fc_quads; i += NT) reinterpret_cast<uint4*>(fc)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < kFsWords / 4; i += NT) reinterpret_cast<uint4*>(fs)[i] = make_uint4(0, 0, 0, 0);
    mbar_wait(&s_mbar[cur], (phases >> cur) & 1u);
    phases ^= 1u << cur;
    if (p.sp_tma_mask != (1u << (R + 1)) - 1u) {  // rows the bulk copies could not take
      __syncthreads();
      for (int s_ = 0; s_ <= R; ++s_)
        if (!(p.sp_tma_mask >> s_ & 1)) {
          const T* src = row_src<T>(p, s_, b);
          T* dst = rows + p.sp_row_off[s_];
          const int n = s_len[lb][s_];
          for (int j = tid; j < n; j += NT) dst[j] = src[j];
        }
    }
    __syncthreads();
    const int mylen = lane <= R ? s_len[lb][lane] : 0;  // this group's lengths, lane s: row s
    const int clen = __shfl_sync(kFull, mylen, 0);
    const T* const crow = rows;
    const int ncq = (clen + 3) >> 2;

    // ---- 1. the candidate's tokens into Fc (a last partial quad's padding may
    // be marked too: extra bits only add false positives)
#pragma unroll 2
    for (int qi = tid; qi < ncq; qi += NT) {
      T t[4];
      lds_quad(crow + 4 * qi, t);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t h = tok_hash32(t[k]);
        atomicOr(&fc[h >> wshift], bit_of(h));
      }
    }
    __syncthreads();

    // ---- 2. reference tokens against Fc, 3. candidate tokens against Fs.  A
    // thread's quads are qi = tid, tid + NT, ...; the survivor bits of 8 of
    // them (4 per quad) collect in `sm` and are listed together: survivors
    // are rare, so the listing code seldom runs.
    auto flush = [&](uint32_t sm, int qb, int* counter, int base_slot, uint32_t side, const T* row,
                     bool mark) -> bool {
      int at = base_slot + atomicAdd(counter, __popc(sm));
      for (; sm; sm &= sm - 1) {
        const int bit = __ffs(sm) - 1;
        const int pos = 4 * (qb + (bit >> 2) * NT) + (bit & 3);
        const T tk = row[pos];
        if (at < kSparseMax) {
          etok[at] = tk;
          eps[at] = (side << 16) | static_cast<uint32_t>(pos);
        }
        ++at;
        if (mark) {
          const uint32_t h = tok_hash32(tk);
          atomicOr(&fs[h >> 23], bit_of(h >> 13));
        }
      }
      return at <= kSparseMax;
    };
    auto scan_row = [&](const T* row, int len, const uint32_t* filt, uint32_t fshift, uint32_t bshift,
                        int* counter, int base_slot, uint32_t side, bool mark) {
      const int nq = (len + 3) >> 2;
      uint32_t sm = 0;
      int j = 0, qb = tid;
#pragma unroll 2
      for (int qi = tid; qi < nq; qi += NT) {
        T t[4];
        lds_quad(row + 4 * qi, t);
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t h = tok_hash32(t[k]);
          m |= (filt[h >> fshift] & bit_of(h >> bshift)) ? (1u << k) : 0u;
        }
        if (4 * qi + 4 > len) m &= (1u << (len - 4 * qi)) - 1u;
        sm |= m << (4 * j);
        if (++j == 8) {
          // a group over the list's capacity goes to the hash-table kernel: stop early
          if (sm && !flush(sm, qb, counter, base_slot, side, row, mark)) return;
          sm = 0;
          j = 0;
          qb = qi + NT;
        }
      }
      if (sm) flush(sm, qb, counter, base_slot, side, row, mark);
    };
    for (int r = 0; r < R; ++r)
      scan_row(rows + p.sp_row_off[r + 1], __shfl_sync(kFull, mylen, r + 1), fc, wshift, 0, &s_cnt[0], 0,
               static_cast<uint32_t>(r + 1), true);
    __syncthreads();
    const int Sr = s_cnt[0];
    if (Sr > 0 && Sr <= kSparseMax) scan_row(crow, clen, fs, 23, 13, &s_cnt[1], Sr, 0u, false);
    __syncthreads();  // every thread is done with the rows: the buffer takes a later group
    const int S = Sr > kSparseMax ? Sr : Sr + s_cnt[1];
    if (stager) {
      const int64_t g = b + nbuf * stride;
      if (g < p.batch) stage(g, cur, (it + nbuf) % 3);
      load_len(g + stride);  // in flight while this group finishes
    }
    if (S > kSparseMax) {  // related text: the hash-table kernel takes this group
      if (tid == 0) p.glist[atomicAdd(p.gcount, 1u)] = static_cast<int>(b);
      continue;  // no shared state of this group is read after this point
    }

    // ---- 4. exact clipped counts (warp 0; lane n-1 holds order n), 5. epilogue
    if (tid < 32) {
      const unsigned int hits =
          S > 0 ? exact_counts<T>(etok, eps, reinterpret_cast<uint32_t*>(aux), aux + 4 * kSparseMax,
                                  aux + 5 * kSparseMax, aux + 6 * kSparseMax, reinterpret_cast<uint16_t*>(fc),
                                  fc + kTinySlots / 2, S, R, N, lane)
                : 0u;
      const int64_t c = clen;
      int64_t rbest = __shfl_sync(kFull, mylen, 1);
      for (int r = 2; r <= R; ++r) {  // closest reference length, ties -> shorter (bleu.py:108-114)
        const int64_t v = __shfl_sync(kFull, mylen, r);
        const int64_t d = v > c ? v - c : c - v;
        const int64_t bd = rbest > c ? rbest - c : c - rbest;
        if (d < bd || (d == bd && v < rbest)) rbest = v;
      }
      const int64_t num = lane < N ? static_cast<int64_t>(hits) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      if (lane < N) {
        if (p.num) p.num[b * N + lane] = num;
        if (p.den) p.den[b * N + lane] = den;
      }
      if (lane == 0) {
        if (p.cand_len_out) p.cand_len_out[b] = c;
        if (p.eff_ref) p.eff_ref[b] = rbest;
      }
      if (p.scores || p.precisions || p.bp)
        warp_epilogue(num, den, c, rbest, N, p.smoothing, p.eps, p.k, lane < N ? p.weights[lane] : 0.0,
                      p.precisions ? p.precisions + b * N : nullptr, p.bp ? p.bp + b : nullptr,
                      p.scores ? p.scores + b : nullptr);
      if (corpus) {  // this group's sums into one of the replicated accumulators;
        // fire-and-forget reductions (the launch's last CTA adds them up)
        const int nt = 2 * N + 2;
        unsigned long long* acc = p.acc + (b % kAccCopies) * nt;
        if (lane < N) {
          if (num) atomicAdd(&acc[lane], static_cast<unsigned long long>(num));
          if (den) atomicAdd(&acc[N + lane], static_cast<unsigned long long>(den));
        }
        if (lane == 0) {
          if (c) atomicAdd(&acc[2 * N], static_cast<unsigned long long>(c));
          if (rbest) atomicAdd(&acc[2 * N + 1], static_cast<unsigned long long>(rbest));
        }
      }
    }
    // the next group's clears wait for warp 0 (the tiny table aliases Fc):
    // the barrier after the clears and the wait orders them
    __syncthreads();
  }

  // ---- flags; corpus: the last CTA finishes the launch unless groups were
  // listed (then the hash-table kernel that follows does)
  flags = __reduce_or_sync(kFull, flags);
  if (!corpus) {  // per-sentence: straight into the caller's flag word
    if (lane == 0 && flags) {
      if (p.err_store)
        *reinterpret_cast<volatile int*>(p.err) = flags;  // mapped host memory; the only bit is BAD_LENGTH
      else
        atomicOr(p.err, flags);
    }
    return;
  }
  if (lane == 0 && flags) atomicOr(p.ws_flag, flags);
  __syncthreads();
  if (tid == 0) s_last = arrive_last(p, gridDim.x) ? 1 : 0;
  __syncthreads();
  if (!s_last) return;
  if (*reinterpret_cast<volatile unsigned int*>(p.gcount) == 0)
    finalize_launch(p, s_tot);
  else if (tid == 0)
    *p.done = 0;  // the hash-table kernel counts its own arrivals
}

}  // namespace

namespace tbk {

// Shared-memory layout, CTA size, row double-buffering and grid of the filter
// kernel (fills prm.sp_* and prm.filter_log2 of the copy it launches with).
int launch_sparse(const StatsParams& prm_in, int sms, cudaStream_t stream, int token_bytes) {
  StatsParams prm = prm_in;
  const int R = prm.num_refs;
  const int64_t cw = prm.cand_width;
  int fl2 = 10;  // Fc words: >= 128 bits per candidate position, >= 4 KiB
  while ((int64_t(1) << fl2) < 4 * cw) ++fl2;
  prm.filter_log2 = fl2;
  auto r16 = [](int64_t v) { return static_cast<int>((v + 15) / 16 * 16); };
  int o = 0;
  prm.sp_off_fc = o;
  o += 4 << fl2;
  prm.sp_off_fs = o;
  o += 4 * kFsWords;
  prm.sp_off_tok = o;
  o = r16(o + kSparseMax * token_bytes);
  prm.sp_off_ps = o;
  o += 4 * kSparseMax;
  prm.sp_off_aux = o;
  o = r16(o + 7 * kSparseMax);
  prm.sp_off_rows = o;
  int buf = 0;
  prm.sp_tma_mask = 0;
  for (int s = 0; s <= R; ++s) {
    prm.sp_row_off[s] = buf / token_bytes;
    const int64_t w = s == 0 ? cw : prm.refs[s - 1].width;
    buf += r16(w * token_bytes + 16);  // + the round-up of a prefix
    const void* base = s == 0 ? prm.cand_ids : prm.refs[s - 1].ids;
    const int64_t ld = s == 0 ? prm.cand_ld : prm.refs[s - 1].ld;
    if ((reinterpret_cast<uintptr_t>(base) & 15) == 0 && ((ld * token_bytes) & 15) == 0) prm.sp_tma_mask |= 1u << s;
  }
  prm.sp_buf_elems = buf / token_bytes;
  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  int smem_sm = 0;
  TB_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  // most warps per SM (registers: 64 per thread for int32 tokens), then two
  // row buffers, then 256 threads; a single wave of groups takes 256 threads
  const int64_t B = prm.batch;
  const int reg_threads = token_bytes == 4 ? 1024 : 768;
  int best_nt = 0, best_nbuf = 0, best_warps = -1;
  for (int nt : {256, 128})
    for (int nb : {2, 1}) {
      const int64_t bytes = o + static_cast<int64_t>(nb) * buf + 1024;
      const int ctas = static_cast<int>(std::min<int64_t>((smem_sm - 1024) / bytes, reg_threads / nt));
      int warps = ctas * nt / 32;
      if (ctas < 1) continue;
      if (B <= static_cast<int64_t>(sms) * ctas && nt == 256) warps += 64;  // single wave: short latency
      if (warps > best_warps) {
        best_warps = warps;
        best_nt = nt;
        best_nbuf = nb;
      }
    }
  if (best_nt == 0) return TB_ERR_UNSUPPORTED;
  prm.sp_nbuf = best_nbuf;
  const int threads = best_nt;
  const size_t smem = static_cast<size_t>(o) + static_cast<size_t>(best_nbuf) * buf;

  using K = void (*)(StatsParams);
  K kern;
  if (token_bytes == 4)
    kern = threads == 256 ? bleu_sparse_kernel<int32_t, 256> : bleu_sparse_kernel<int32_t, 128>;
  else
    kern = threads == 256 ? bleu_sparse_kernel<int64_t, 256> : bleu_sparse_kernel<int64_t, 128>;
  static thread_local struct { const void* k; int dev; size_t smem; int occ; } cache[16] = {};
  static thread_local int next = 0;
  int occ = 0;
  for (auto& e : cache)
    if (e.occ > 0 && e.k == reinterpret_cast<const void*>(kern) && e.dev == dev && e.smem == smem) occ = e.occ;
  // the dynamic shared-memory opt-in of each kernel only ever grows (a smaller
  // value set for one shape would refuse a larger cached shape later)
  static size_t attr_max[4][64] = {};
  size_t& amax = attr_max[(token_bytes == 4 ? 0 : 2) + (threads == 256 ? 0 : 1)][dev & 63];
  if (smem > amax) {
    TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    amax = smem;
  }
  if (occ == 0) {
    // one shared-memory carveout for every stats kernel: back-to-back launches
    // of different kernels then need no L1/shared reconfiguration
    TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    TB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    if (occ < 1) occ = 1;
    cache[next] = {reinterpret_cast<const void*>(kern), dev, smem, occ};
    next = (next + 1) & 15;
  }
  int64_t grid = B;
  if (grid > static_cast<int64_t>(occ) * sms) grid = static_cast<int64_t>(occ) * sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // plain stream order: with programmatic serialization its early-launched
  // CTAs slowed the hash-table kernel of the previous launch (c5, related
  // text: 1206 -> 1282 us per step, measured)
  cfg.numAttrs = pdl_mode() == 3 ? 1 : 0;
  TB_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

}  // namespace tbk
