// tb_kernel_group.cu — reference-at-a-time kernel (R > 8) and the global-memory kernel (very wide rows)
// (see tb_common.cuh for the source layout, DESIGN.md §3 for the design)

#include "tb_launch.cuh"

namespace {

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
    if (!p.no_tails) copy_row_tails<T>(p, b, R + 1, tok, s_stage_len, tid, kThreads);  // tails / unaligned rows
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

}  // namespace

namespace tbk {

int launch_group(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes) {
  static size_t attr_set[2][64] = {};
  if (token_bytes == 4)
    return launch_kernel(bleu_group_kernel<int32_t>, prm, pl, sms, true, attr_set[0], stream);
  return launch_kernel(bleu_group_kernel<int64_t>, prm, pl, sms, true, attr_set[1], stream);
}

int launch_global(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes) {
  static size_t attr_set[2][64] = {};
  if (token_bytes == 4)
    return launch_kernel(bleu_stats_kernel<int32_t, false>, prm, pl, sms, false, attr_set[0], stream);
  return launch_kernel(bleu_stats_kernel<int64_t, false>, prm, pl, sms, false, attr_set[1], stream);
}

#ifdef TB_PHASES
int set_phases_group(void* buf) { return set_phase_buffer_here(buf); }
#endif

}  // namespace tbk
