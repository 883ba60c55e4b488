// tb_kernel_multi.cu — multi-reference kernel (2 <= R <= 8)
// (see tb_common.cuh for the source layout, DESIGN.md §3 for the design)

#include "tb_launch.cuh"

namespace {


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

template <typename T, bool kList>
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
  __shared__ uint16_t s_flist[kSmallSet];  // order-1 filter survivors (positions)
  __shared__ T s_ftok[kSmallSet];          // and their tokens
  __shared__ int s_nf;

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
  // list mode: the dense groups listed by the warp-per-group kernel before this one
  const int64_t nb = kList ? static_cast<int64_t>(*reinterpret_cast<volatile unsigned int*>(p.gcount)) : p.batch;
  auto group_at = [&](int64_t i) -> int64_t { return kList ? static_cast<int64_t>(p.glist[i]) : i; };
  if (static_cast<int64_t>(blockIdx.x) < nb) issue_stage(group_at(blockIdx.x));
  __syncthreads();
  TB_MARK(0);
  uint32_t phase = 0;
  // The order-1 filter (below) is tried until a group of this CTA needs the
  // hash passes (related text; listed groups are known to), and only when
  // every CTA has two or more groups: with one group per CTA a group of
  // related text pays the whole failed filter (c3 related 43.9 -> 47.6 us,
  // against c3 uniform 15.1 -> 12.3 us); with more, one failure per CTA.
  bool try_filter = !kList && nb >= 2 * static_cast<int64_t>(gridDim.x);
  // Fc: a blocked two-bit Bloom filter of the candidate tokens in the first
  // half of the table region (2^fl words), Fs: the reference survivors' filter
  // after it (2^tl <= 256 words)
  const int fl = cap_log2 - 2;
  const uint32_t tl = fl < 8 ? fl : 8;

  for (int64_t gi = blockIdx.x; gi < nb; gi += gridDim.x) {
    const int64_t b = group_at(gi);
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
    if (tid == 0) {
      s_nf = 0;
      s_nc = 0;
      s_nr = 0;
    }
    if (!p.no_tails) copy_row_tails<T>(p, b, R + 1, tok, s_stage_len, tid, NT);  // tails / unaligned rows
    if (try_filter)
      for (uint32_t s = tid; s < ((1u << fl) + (1u << tl)) / 4; s += NT)
        reinterpret_cast<uint4*>(own)[s] = make_uint4(0, 0, 0, 0);
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

    // ================= order 1: filter =================
    // Unrelated text: three Bloom passes — candidate tokens into Fc, every
    // reference's tokens tested against Fc (survivors listed and marked in
    // Fs), candidate tokens tested against Fs — leave the few positions whose
    // token may occur on the other side.  When at most kSmallSet do, the block
    // matches them exactly (per-reference counts, clip min(c, max_r x_r)),
    // gives each live position its order-1 id (the lowest list index holding
    // its token) and the small-set path below finishes orders >= 2: no table.
    bool filtered = false;
    if (try_filter) {
      uint32_t* const fc = reinterpret_cast<uint32_t*>(own);
      uint32_t* const fsm = fc + (1u << fl);
      const uint32_t wshift = 32 - fl, bs1 = wshift - 5, bs2 = wshift - 10;
      auto fmask = [bs1, bs2](uint32_t h) { return bit_of(h >> bs1) | bit_of(h >> bs2); };
      auto smask = [tl](uint32_t h) { return bit_of(h >> (27 - tl)) | bit_of(h >> (22 - tl)); };
      auto load4 = [&](int p0, T (&t)[4]) {
        if constexpr (sizeof(T) == 4) {
          const int4 v = *reinterpret_cast<const int4*>(tok + p0);
          t[0] = v.x;
          t[1] = v.y;
          t[2] = v.z;
          t[3] = v.w;
        } else {
          const longlong2 u = *reinterpret_cast<const longlong2*>(tok + p0);
          const longlong2 v = *reinterpret_cast<const longlong2*>(tok + p0 + 2);
          t[0] = u.x;
          t[1] = u.y;
          t[2] = v.x;
          t[3] = v.y;
        }
      };
      auto list_survivors = [&](uint32_t pm, int p0, int side, bool mark) {
        // once the list has overflowed (related text) the filter has failed:
        // nothing more to list or mark (s_nf only grows)
        if (pm == 0 || *reinterpret_cast<volatile int*>(&s_nf) > kSmallSet) return;
        for (; pm; pm &= pm - 1) {
          const int pos = p0 + __ffs(pm) - 1;
          const int j = atomicAdd(&s_nf, 1);
          const T tk = tok[pos];
          if (j < kSmallSet) {
            s_flist[j] = static_cast<uint16_t>(pos);
            s_ftok[j] = tk;
            s_sside[j] = static_cast<uint8_t>(side);  // 0 = candidate, 1 + r = reference r
          }
          if (mark) {
            const uint32_t h = tok_hash32(tk);
            atomicOr(&fsm[h >> (32 - tl)], smask(h));
          }
        }
      };
      for (int qi = tid; qi < ncq; qi += NT) {  // candidate tokens into Fc (branch-free)
        const int p0 = 4 * qi;
        const uint32_t vm = cand_mask(p0);
        T t[4];
        load4(p0, t);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t h = tok_hash32(t[k]);
          atomicOr(&fc[h >> wshift], (vm >> k & 1u) ? fmask(h) : 0u);
        }
      }
      if (tid == NT - 32) {  // lengths only: the last warp
        const int64_t r = closest_ref_len(s_len[0], &s_len[1], R);
        s_effref = r;
        s_bp = brevity_penalty_fp64(s_len[0], r);
      }
      __syncthreads();
      TB_MARK(20);
      for (int qi = tid; qi < nrq; qi += NT) {  // reference tokens against Fc
        int r, p0;
        const uint32_t vm = ref_quad(qi, r, p0);
        T t[4];
        load4(p0, t);
        uint32_t pm = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t h = tok_hash32(t[k]);
          const uint32_t m = fmask(h);
          pm |= ((fc[h >> wshift] & m) == m ? 1u : 0u) << k;
        }
        *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);  // unmatched unless listed live
        *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
        list_survivors(pm & vm, p0, 1 + r, true);
      }
      __syncthreads();
      TB_MARK(21);
      TB_NOTE(25, s_nf);
      if (s_nf <= kSmallSet) {  // uniform
        for (int qi = tid; qi < ncq; qi += NT) {  // candidate tokens against Fs
          const int p0 = 4 * qi;
          const uint32_t vm = cand_mask(p0);
          T t[4];
          load4(p0, t);
          uint32_t pm = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t h = tok_hash32(t[k]);
            const uint32_t m = smask(h);
            pm |= ((fsm[h >> (32 - tl)] & m) == m ? 1u : 0u) << k;
          }
          *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);
          *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
          list_survivors(pm & vm, p0, 0, false);
        }
        __syncthreads();
      }
      TB_MARK(22);
      const int S = s_nf;
      TB_NOTE(27, S);
      if (S <= kSmallSet) {
        filtered = true;
        if (tid < S) {  // exact order 1 among the listed positions
          // branch-free scan of the list (every entry matches itself, so a
          // branch per match would run on every iteration): the reference
          // counts in eight 8-bit fields (<= kSmallSet = 128 each), the lowest
          // index holding the token as its id
          const int pos = s_flist[tid];
          const T tk = s_ftok[tid];
          const int side = s_sside[tid];
          unsigned c = 0;
          unsigned long long xr = 0;
          int leader = tid;
          for (int j = S - 1; j >= 0; --j) {
            const bool eq = s_ftok[j] == tk;
            const int sj = s_sside[j];
            leader = eq ? j : leader;
            c += (eq && sj == 0) ? 1u : 0u;
            xr += (eq && sj != 0) ? (1ull << (8 * (sj - 1))) : 0ull;
          }
          unsigned x = 0;
#pragma unroll
          for (int r = 0; r < kMultiMaxRefs; ++r) {
            const unsigned v = static_cast<unsigned>(xr >> (8 * r)) & 0xffu;
            x = v > x ? v : x;
          }
          if (leader == tid) {
            const unsigned h = c < x ? c : x;
            if (h) atomicAdd(&s_hits[0], h);
          }
          if (side == 0 ? x > 0 : c > 0) {
            id1[pos] = static_cast<uint16_t>(leader);
            idn[pos] = static_cast<uint16_t>(leader);
            if (side == 0) lx[atomicAdd(&s_nc, 1)] = static_cast<uint16_t>(pos);
            else lx[cpad + atomicAdd(&s_nr, 1)] = static_cast<uint16_t>(pos);
          }
        }
        __syncthreads();
      } else {
        try_filter = false;  // related text: the hash passes (uniform across the CTA)
      }
    }

    // ================= order 1: tokens =================
    if (!filtered) count_order1(static_cast<const T*>(tok), id1, idn);
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
          // branch-free (every entry matches itself): reference counts in
          // eight 8-bit fields (<= kSmallSet each)
          unsigned c = 0;
          unsigned long long xr = 0;
          for (int j = S - 1; j >= 0; --j) {
            const bool eq = s_skey[j] == key;
            const int sj = s_sside[j];
            leader = eq ? j : leader;
            c += (eq && sj == 0) ? 1u : 0u;
            xr += (eq && sj != 0) ? (1ull << (8 * (sj - 1))) : 0ull;
          }
          unsigned x = 0;
#pragma unroll
          for (int r = 0; r < kMultiMaxRefs; ++r) {
            const unsigned v = static_cast<unsigned>(xr >> (8 * r)) & 0xffu;
            x = v > x ? v : x;
          }
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

    // ---- epilogue: warp 0 the fp64 scores, warp 1 (in parallel) the integer outputs
    if (tid >= 32 && tid < 64) {
      const int64_t c = s_len[0];
      if (lane < N) {
        if (p.num) p.num[b * N + lane] = static_cast<int64_t>(s_hits[lane]);
        if (p.den) p.den[b * N + lane] = c - lane > 0 ? c - lane : 0;
      }
      if (lane == 0) {
        if (p.cand_len_out) p.cand_len_out[b] = c;
        if (p.eff_ref) p.eff_ref[b] = s_effref;
      }
    }
    if (tid < 32) {
      const int64_t c = s_len[0];
      const int64_t num = lane < N ? static_cast<int64_t>(s_hits[lane]) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      const int64_t r = s_effref;
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
    if (gi + gridDim.x < nb) {
      __syncthreads();
      issue_stage(group_at(gi + gridDim.x));
    }
    TB_MARK(30);
  }
  finish_cta<kList>(p, s_tot, s_flags, s_last, nb);
  TB_MARK(31);
}


}  // namespace

namespace tbk {

int launch_multi(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes) {
  static size_t attr_set[4][64] = {};
  const bool list = prm.glist != nullptr;
  if (token_bytes == 4)
    return list ? launch_kernel(bleu_multi_kernel<int32_t, true>, prm, pl, sms, true, attr_set[2], stream, kMultiThreads)
                : launch_kernel(bleu_multi_kernel<int32_t, false>, prm, pl, sms, true, attr_set[0], stream, kMultiThreads);
  return list ? launch_kernel(bleu_multi_kernel<int64_t, true>, prm, pl, sms, true, attr_set[3], stream, kMultiThreads)
              : launch_kernel(bleu_multi_kernel<int64_t, false>, prm, pl, sms, true, attr_set[1], stream, kMultiThreads);
}

#ifdef TB_PHASES
int set_phases_multi(void* buf) { return set_phase_buffer_here(buf); }
#endif

}  // namespace tbk
