// tb_kernel_pair.cu — single-reference kernel (R = 1), the headline path
// (see tb_common.cuh for the source layout, DESIGN.md §3.1 for the design)

#include "tb_launch.cuh"

namespace {


// --------------------------------------------------------------------------
// Single-reference kernel (R == 1, the headline configuration).
//
// Order 1: a blocked two-bit Bloom filter (in the table + count region)
// drops the tokens absent from the other side — two passes over both rows, or
// (kThree, rows of more quads than threads) three: candidate tokens into Fc,
// reference tokens against Fc, candidate tokens against the small filter of
// the reference survivors.  When <= kSmallSet positions survive (unrelated
// text) they are matched exactly without a table (<= 32: warp 0 with
// match.any, which also finishes orders >= 2 in its registers).  Otherwise
// only CANDIDATE tokens are inserted, store-then-verify:
//   claim:  every candidate position stores itself (u16) into its token's
//           home slot — plain stores, one wins;
//   verify: the winner owns the slot (its own occurrence is counted
//           implicitly); an equal token adds one to the owner's count word
// and orders >= 2 run table rounds over the live lists.
//
// 256 threads per CTA (4 CTAs per SM); kList: the groups listed by the filter
// kernel (tb_kernel_sparse.cu), which needed the hash passes.
template <typename T, int NT, bool kList, bool kThree>
__global__ void __launch_bounds__(NT, 1024 / NT)
    bleu_pair_kernel(const __grid_constant__ StatsParams p) {
  constexpr int kThreads = NT;
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
  // token buffer `buf` (computed from smem, not read from an array of pointers:
  // a pointer array lives in local memory and every token access through it
  // compiles to a generic LD/ST instead of LDS/STS)
  auto tok_buf = [&](int buf) { return reinterpret_cast<T*>(smem + (buf ? p.off_tok2 : 16)); };
  const bool dbuf = p.off_tok2 != 0;  // prefetch the next group into the other buffer
  int cur = 0;
  T* tok = tok_buf(0);
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
    if (tid == 0) issue_rows<T>(p, b, 2, tok_buf(buf), mbars + buf, s_stage_len, &s_flags);
  };

  if (tid < 2 * N + 2) s_tot[tid] = 0;
  if (tid == 0) {
    s_flags = 0;
    mbar_init(mbars, 1);
    if (dbuf) mbar_init(mbars + 1, 1);
  }
  griddep_wait_and_release();
  // list mode: the dense groups listed by the warp-per-group kernel before this one
  // (a template parameter: the runtime test cost the batch path 0.6 us at c4)
  const int64_t nb = kList ? static_cast<int64_t>(*reinterpret_cast<volatile unsigned int*>(p.gcount)) : p.batch;
  auto group_at = [&](int64_t i) -> int64_t { return kList ? static_cast<int64_t>(p.glist[i]) : i; };
  if (static_cast<int64_t>(blockIdx.x) < nb) issue_stage(group_at(blockIdx.x), 0);
  __syncthreads();
  TB_MARK(0);
  uint32_t phases = 0;  // bit i: parity of mbarrier i
  // off after a group of this CTA needed the hash passes (related text); listed
  // groups are known to need them
  bool try_filter = !kList;
  // Rows of more quads than threads filter in three passes (candidate tokens
  // into Fc, reference tokens against it, candidate tokens against the small
  // filter of the reference survivors): one loop iteration per thread and
  // pass instead of two over both rows.  Short rows keep the two passes.  A
  // template parameter: both paths in one kernel cost c2 0.1 us and c4 0.5 us.
  constexpr bool three_pass = kThree;

  for (int64_t gi = blockIdx.x; gi < nb; gi += gridDim.x) {
    const int64_t b = group_at(gi);
    tok = tok_buf(cur);
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
    if (!p.no_tails) copy_row_tails<T>(p, b, 2, tok, s_stage_len, tid, kThreads);  // tails / unaligned rows
    // the table region starts as the two filter bitmaps (zero; they extend over
    // the count array) or as the empty table
    if (try_filter) {
      // two-pass: both sides' bitmaps; three-pass: Fc and the small filter after it
      const uint32_t fwords = three_pass ? (1u << p.filter_log2) + (1u << min(p.filter_log2, 8))
                                         : 2u << p.filter_log2;
      for (uint32_t s = tid; s < fwords / 4; s += kThreads)
        reinterpret_cast<uint4*>(own)[s] = make_uint4(0, 0, 0, 0);
    } else {
      for (uint32_t s = tid; s < cap / 8; s += kThreads)
        reinterpret_cast<uint4*>(own)[s] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    mbar_wait(mbars + cur, (phases >> cur) & 1u);
    phases ^= 1u << cur;
    __syncthreads();
    // every thread is past the previous group: its buffer takes the next group
    if (dbuf && gi + gridDim.x < nb) issue_stage(group_at(gi + gridDim.x), cur ^ 1);
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
    // word; three-pass: the candidate side only, plus the small filter of the
    // reference survivors); a token not in the other side's filter cannot match (false
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
      // the two bits from the ten hash bits just below the word index (one
      // product per token: h's top bits pick the word)
      const uint32_t bs1 = wshift - 5, bs2 = wshift - 10;
      auto fmask = [bs1, bs2](uint32_t h) { return bit_of(h >> bs1) | bit_of(h >> bs2); };
      if (three_pass) {
        // Three passes: candidate tokens into Fc; reference tokens tested
        // against Fc — the survivors are listed and marked in a small filter Fs
        // (<= 256 words) — and candidate tokens tested against Fs only
        // while the list still fits (related text stops after the second).
        uint32_t* const fsm = bmr;  // Fs, in the (otherwise unused) reference half
        const uint32_t tl = p.filter_log2 < 8 ? p.filter_log2 : 8;  // Fs: 2^tl words
        auto smask = [tl](uint32_t h) { return bit_of(h >> (27 - tl)) | bit_of(h >> (22 - tl)); };
        for (int qi = tid; qi < ncq; qi += kThreads) {
          const int p0 = 4 * qi;
          const uint32_t vm = clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u);
          T t[4];
          load4(p0, t);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // branch-free: a position past the length ORs nothing
            const uint32_t h = tok_hash32(t[k]);
            atomicOr(&bmc[h >> wshift], (vm >> k & 1u) ? fmask(h) : 0u);
          }
        }
        __syncthreads();
        TB_MARK(20);
        const int nrq = nq - ncq;
        for (int qi = tid; qi < nrq; qi += kThreads) {
          const int p0 = roff + 4 * qi;
          const uint32_t vm = roff + rlen - p0 >= 4 ? 0xfu : ((1u << (roff + rlen - p0)) - 1u);
          T t[4];
          load4(p0, t);
          uint32_t pm = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t h = tok_hash32(t[k]);
            const uint32_t m = fmask(h);
            pm |= ((bmc[h >> wshift] & m) == m ? 1u : 0u) << k;
          }
          pm &= vm;
          *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);
          *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
          for (; pm; pm &= pm - 1) {
            const int k = __ffs(pm) - 1;
            const int j = atomicAdd(&s_nf, 1);
            if (j < kSmallSet) s_flist[j] = static_cast<uint16_t>(p0 + k);
            const uint32_t h = tok_hash32(tok[p0 + k]);
            atomicOr(&fsm[h >> (32 - tl)], smask(h));
          }
        }
        __syncthreads();
        if (s_nf <= kSmallSet) {  // uniform across the CTA
          for (int qi = tid; qi < ncq; qi += kThreads) {
            const int p0 = 4 * qi;
            const uint32_t vm = clen - p0 >= 4 ? 0xfu : ((1u << (clen - p0)) - 1u);
            T t[4];
            load4(p0, t);
            uint32_t pm = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t h = tok_hash32(t[k]);
              const uint32_t m = smask(h);
              pm |= ((fsm[h >> (32 - tl)] & m) == m ? 1u : 0u) << k;
            }
            pm &= vm;
            *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);
            *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
            for (; pm; pm &= pm - 1) {
              const int j = atomicAdd(&s_nf, 1);
              if (j < kSmallSet) s_flist[j] = static_cast<uint16_t>(p0 + __ffs(pm) - 1);
            }
          }
        }
      } else {
        for (int qi = tid; qi < nq; qi += kThreads) {
          int p0;
          const uint32_t vm = quad(qi, p0);
          T t[4];
          load4(p0, t);
          uint32_t* bm = p0 < roff ? bmc : bmr;
          // branch-free: a position past the row's length ORs nothing
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t h = tok_hash32(t[k]);
            atomicOr(&bm[h >> wshift], (vm >> k & 1u) ? fmask(h) : 0u);
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
          for (int k = 0; k < 4; ++k) {  // branch-free; positions past the length masked below
            const uint32_t h = tok_hash32(t[k]);
            const uint32_t m = fmask(h);
            pm |= ((bm[h >> wshift] & m) == m ? 1u : 0u) << k;
          }
          pm &= vm;
          // every valid position starts "unmatched" at order 1 (the exact match below
          // marks the matched ones)
          *reinterpret_cast<uint2*>(id1 + p0) = make_uint2(~0u, ~0u);
          *reinterpret_cast<uint2*>(idn + p0) = make_uint2(~0u, ~0u);
          // (an early exit once more survivors than the exact match takes were
          // listed — related text — saved 1.8 us at c2 related but cost 0.5 us
          // at c2 uniform: the loop stays branch-free)
          for (; pm; pm &= pm - 1) {
            const int j = atomicAdd(&s_nf, 1);
            if (j < kSmallSet) s_flist[j] = static_cast<uint16_t>(p0 + __ffs(pm) - 1);
          }

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
          if (lane == 0) {
            s_hits[0] = h;
            s_nc = 0;  // orders >= 2 are finished here: nothing left for the passes below
            s_nr = 0;
          }
          // orders 2..N of the same positions, still in this warp's registers
          // (no block barrier, no list round trip): an n-gram's id for the
          // next order is the lowest lane holding it
          __syncwarp();  // the live positions' order-1 ids
          int q0 = live ? pos : -1;
          uint32_t pid = static_cast<uint32_t>(leader);
          if (__any_sync(kFull, live && pos < roff))
            for (int m = 2; m <= N; ++m) {
              bool valid = q0 >= 0;
              uint32_t key = 0;
              if (valid) {
                const int end = q0 < roff ? clen : roff + rlen;
                const int q = q0 + m - 1;
                valid = q < end && id1[q] != 0xffffu;
                if (valid) key = (pid << 16) | id1[q];
              }
              const unsigned pm = __match_any_sync(kFull, valid ? key : 0xffffffffu - lane);
              const unsigned cn = __popc(pm & __ballot_sync(kFull, valid && q0 < roff));
              const unsigned xn = __popc(pm & __ballot_sync(kFull, valid && q0 >= roff));
              const int ld = __ffs(pm) - 1;
              unsigned hn = (valid && lane == ld) ? (cn < xn ? cn : xn) : 0u;
              hn = __reduce_add_sync(kFull, hn);
              if (lane == 0) s_hits[m - 1] = hn;
              const bool ok = valid && (q0 < roff ? xn > 0 : cn > 0);
              if (!__any_sync(kFull, ok && q0 < roff)) break;
              q0 = ok ? q0 : -1;
              pid = static_cast<uint32_t>(ld);
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
        pair_resolve_lost<NT>(own, cnt, lost, nl, id1, mask, hshift, roff, tid, hash1, eq1, 2);
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
        // predicated per entry (the branchy form spent a third of the related-text
        // instructions on control flow): a candidate owning its slot or a key
        // equal to its slot's records the slot id (+1 on the owner's count); a
        // reference key with an EMPTY home is dead; the rest — candidates lost to
        // a different key, references whose home holds another key — are rare
        // and handled after the loop.  (A live candidate key's home is never
        // empty: the claim pass stored into it.)
        const bool rside = i0 >= roff;
        uint32_t rare = 0;
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = i0 + k;
          const bool live = key[k] != ~0u;
          const bool self = !rside && w[k] == i;
          const bool hit = live && !self && kw[k] == key[k];
          const bool empty = live && rside && w[k] == 0xffffu;
          if (self || hit) idn[pos[k]] = static_cast<uint16_t>(w[k]);
          // (constant increments: one atomic with a per-lane operand made
          // vocab = 1 rows, every lane on one word, 12% slower)
          if (hit && !rside) atomicAdd(&cnt[w[k]], 1u);
          if (hit && rside) atomicAdd(&cnt[w[k]], 1u << 16);
          if (empty) kc[i] = ~0u;
          rare |= (live && !self && !hit && !empty ? 1u : 0u) << k;
        }
        for (; rare; rare &= rare - 1) {
          const int i = i0 + __ffs(rare) - 1;
          if (rside) {
            defl[atomicAdd(&s_ndef, 1)] = static_cast<uint16_t>(i);
          } else {
            lout[atomicAdd(&s_nlost, 1)] = static_cast<uint16_t>(i);
            pair_retry_store(own, kc[i] * 0x9E3779B1u, 1, hshift, static_cast<uint16_t>(i));
          }
        }
      }
      __syncthreads();
      if (s_nlost) list_resolve_lost<NT>(own, cnt, kc, lout, s_nlost, lin, idn, mask, hshift, tid);
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
          for (int k = 0; k < 4; ++k) {  // (predicated)
            const bool live = key[k] != ~0u;
            const uint32_t c = (cw[k] & 0xffffu) + 1u;  // owners are candidate entries
            const uint32_t x = cw[k] >> 16;
            hits += (live && w[k] == static_cast<uint32_t>(i0 + k)) ? (c < x ? c : x) : 0u;
            lm |= (live && (i0 >= roff || x != 0) ? 1u : 0u) << k;
          }
        }
        // the quads of (at most) one warp straddle the two parts: one append per part there
        const bool cside = qi < mcq;
        const unsigned cs = __ballot_sync(kFull, cside);
        if (cs != 0u) warp_append_quad(lout, &s_nc, cside ? lm : 0u, [&](int k) { return pos[k]; }, lane);
        if (cs != kFull) warp_append_quad(lout + roff, &s_nr, cside ? 0u : lm, [&](int k) { return pos[k]; }, lane);
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
    // ---- epilogue: warp 0 the fp64 scores, warp 1 (in parallel) the integer
    // outputs; warp 1 waits on a named barrier for warp 0, the last writer of
    // the counts (the orders >= 2 of few survivors)
    if (tid < 64) {
      asm volatile("bar.sync 1, 64;" ::: "memory");
      const int64_t c = s_len[0];
      const int64_t num = lane < N ? static_cast<int64_t>(s_hits[lane]) : 0;
      const int64_t den = (lane < N && c - lane > 0) ? c - lane : 0;
      const int64_t r = s_len[1];
      if (tid >= 32) {
        if (lane < N) {
          if (p.num) p.num[b * N + lane] = num;
          if (p.den) p.den[b * N + lane] = den;
        }
        if (lane == 0) {
          if (p.cand_len_out) p.cand_len_out[b] = c;
          if (p.eff_ref) p.eff_ref[b] = r;
        }
      } else {
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
    }
    if (!dbuf && gi + gridDim.x < nb) {
      __syncthreads();
      issue_stage(group_at(gi + gridDim.x), 0);
    }
    if (dbuf) {
      cur ^= 1;
      __syncthreads();  // s_len / s_hits of this group are read before the next group resets them
    }
    TB_MARK(30);
  }
  finish_cta<kList>(p, s_tot, s_flags, s_last, nb);
  TB_MARK(31);
}

}  // namespace

namespace tbk {

int launch_pair(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes) {
  static size_t attr_set[6][64] = {};
  // (512-thread CTAs, bleu_pair_kernel<T, 512, .>, measured no faster on single
  // waves of few groups: c1 5.48 vs 5.60 us; 256 everywhere)
  const bool list = prm.glist != nullptr;  // the groups listed by the filter kernel (no filter passes)
  // three-pass filter when the two rows hold more quads than a CTA has threads
  // (c2 7.06 -> 6.85 us, c4 33.8 -> 33.0; c1's 256-token rows 5.09 vs 5.45 two-pass)
  const bool three = (static_cast<int64_t>(prm.cand_pad) + prm.ref_off[1]) / 4 > 256;
  if (token_bytes == 4) {
    if (list) return launch_kernel(bleu_pair_kernel<int32_t, 256, true, false>, prm, pl, sms, true, attr_set[2], stream);
    return three ? launch_kernel(bleu_pair_kernel<int32_t, 256, false, true>, prm, pl, sms, true, attr_set[4], stream)
                 : launch_kernel(bleu_pair_kernel<int32_t, 256, false, false>, prm, pl, sms, true, attr_set[0], stream);
  }
  if (list) return launch_kernel(bleu_pair_kernel<int64_t, 256, true, false>, prm, pl, sms, true, attr_set[3], stream);
  return three ? launch_kernel(bleu_pair_kernel<int64_t, 256, false, true>, prm, pl, sms, true, attr_set[5], stream)
               : launch_kernel(bleu_pair_kernel<int64_t, 256, false, false>, prm, pl, sms, true, attr_set[1], stream);
}

#ifdef TB_PHASES
int set_phases_pair(void* buf) { return set_phase_buffer_here(buf); }
#endif

}  // namespace tbk
