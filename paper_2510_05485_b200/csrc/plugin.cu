// plugin.cu — device versions of the reference operator/plugin surface
// (pkg/src/batchbleu/_backend.py:45-54 -> _kernels.pyx / _py_kernels.py):
//
//   tb_unique_rows          batch-wide n-gram dictionary (global hash table,
//                           exact row compare, dense IDs in first-occurrence
//                           order via a device scan)
//   tb_segment_bincount     offset "batched bincount" (shared-memory histogram
//                           per segment, global atomics when U does not fit)
//   tb_clipped_numerators   fused candidate count + min-clip + row sum
//   tb_count_binary         max_reference_counts / clip_counts elementwise
//
// These serve the spec-level n-gram API (ngrams.py:63-141, 208-227) and the
// plugin functions; the fused sentence path lives in tensorbleu.cu.

#include "../../include/tensorbleu.h"
#include "tb_guard.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int64_t kTile = kScanThreads * kScanItems;

#define TB_CUDA(expr)                      \
  do {                                     \
    cudaError_t _e = (expr);               \
    if (_e != cudaSuccess) return TB_ERR_CUDA; \
  } while (0)

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int num_sms() {
  static int sms[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (!sms[dev & 63]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    sms[dev & 63] = v;
  }
  return sms[dev & 63];
}

int smem_optin() {
  static int val[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 48 * 1024;
  if (!val[dev & 63]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
      v = 48 * 1024;
    val[dev & 63] = v;
  }
  return val[dev & 63];
}

// --------------------------------------------------------------------------
// Block-wide exclusive scan of int64 values (256 threads x 8 items per tile).
// --------------------------------------------------------------------------
__device__ __forceinline__ long long warp_incl_scan(long long v) {
  const int lane = threadIdx.x & 31;
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// returns the exclusive prefix of `v` within the block, and the block total
__device__ __forceinline__ long long block_excl_scan(long long v, long long* total) {
  __shared__ long long s_warp[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long inc = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    const long long wi = warp_incl_scan(w);
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  const long long res = s_warp[warp] + inc - v;
  __syncthreads();
  return res;
}

// Values are produced by a functor so that flags need not be materialised.
struct SegLenValue {
  const int64_t* v;
  __device__ long long operator()(int64_t i) const { return v[i]; }
};
struct FirstOccValue {
  const int64_t* slot_of;  // (t,) slot of each row
  const int64_t* rep;      // (cap,) min row index per slot
  __device__ long long operator()(int64_t i) const { return rep[slot_of[i]] == i ? 1 : 0; }
};

template <class F>
__global__ void __launch_bounds__(kScanThreads) tile_sum_kernel(F f, int64_t n, int64_t* bsum) {
  const int64_t base = blockIdx.x * kTile + threadIdx.x * static_cast<int64_t>(kScanItems);
  long long s = 0;
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += f(base + i);
  __shared__ long long s_total;
  block_excl_scan(s, &s_total);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s_total;
}

// single CTA: exclusive scan of nb block sums in place; *total = sum
__global__ void __launch_bounds__(kScanThreads) scan_bsums_kernel(int64_t* bsum, int64_t nb, int64_t* total) {
  __shared__ long long s_total;
  long long carry = 0;
  for (int64_t base = 0; base < nb; base += kTile) {
    const int64_t i0 = base + threadIdx.x * static_cast<int64_t>(kScanItems);
    long long vals[kScanItems];
    long long s = 0;
    for (int i = 0; i < kScanItems; ++i) {
      vals[i] = (i0 + i < nb) ? bsum[i0 + i] : 0;
      s += vals[i];
    }
    long long ex = block_excl_scan(s, &s_total) + carry;
    for (int i = 0; i < kScanItems; ++i) {
      if (i0 + i < nb) bsum[i0 + i] = ex;
      ex += vals[i];
    }
    carry += s_total;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// exclusive prefix per element: out[i] = bsum_excl[tile] + prefix within tile
template <class F, class Sink>
__global__ void __launch_bounds__(kScanThreads)
    tile_scan_kernel(F f, int64_t n, const int64_t* bsum_excl, Sink sink) {
  __shared__ long long s_total;
  const int64_t base = blockIdx.x * kTile + threadIdx.x * static_cast<int64_t>(kScanItems);
  long long vals[kScanItems];
  long long s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    vals[i] = (base + i < n) ? f(base + i) : 0;
    s += vals[i];
  }
  long long ex = block_excl_scan(s, &s_total) + bsum_excl[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) sink(base + i, ex, vals[i]);
    ex += vals[i];
  }
}

struct OffsetSink {
  int64_t* out;
  __device__ void operator()(int64_t i, long long ex, long long) const { out[i] = ex; }
};

// --------------------------------------------------------------------------
// Valid n-gram windows (extract_ngrams + flatten_valid, ngrams.py:63-83):
// row i contributes max(len_i - n + 1, 0) windows, concatenated row-major.
// --------------------------------------------------------------------------
struct WindowCount {
  const int64_t* len;
  int64_t width;
  int n;
  __device__ long long operator()(int64_t i) const {
    int64_t l = len[i];
    l = l < 0 ? 0 : (l > width ? width : l);
    const int64_t c = l - n + 1;
    return c > 0 ? c : 0;
  }
};

// one warp per row: window j of row i -> out[(off_i + j) * n + c] = ids[i, j + c]
template <typename T>
__global__ void __launch_bounds__(256) windows_fill_kernel(const T* __restrict__ ids, int64_t ld, int64_t batch,
                                                           int n, WindowCount cnt, const int64_t* __restrict__ off,
                                                           int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < batch;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t c = cnt(i);
    const T* row = ids + i * ld;
    int64_t* dst = out + off[i] * n;
    // element e of this row's output block is column e % n of window e / n
    for (int64_t e = lane; e < c * n; e += 32) {
      const int64_t j = e / n, col = e - j * n;
      dst[e] = static_cast<int64_t>(row[j + col]);
    }
  }
}

// --------------------------------------------------------------------------
// Dictionary (unique_rows).
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t row_hash(const int64_t* row, int n) {
  uint64_t h = 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(n);
  for (int i = 0; i < n; ++i) {
    h ^= static_cast<uint64_t>(row[i]);
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  h *= 0x94D049BB133111EBull;
  h ^= h >> 29;
  return h;
}

__device__ __forceinline__ bool rows_equal(const int64_t* a, const int64_t* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

__global__ void dict_init_kernel(unsigned long long* keys, long long* rep, int64_t cap) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < cap;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    keys[s] = ~0ull;
    rep[s] = LLONG_MAX;
  }
}

__global__ void dict_insert_kernel(const int64_t* __restrict__ rows, int64_t t, int n,
                                   unsigned long long* keys, long long* rep, uint64_t mask,
                                   int64_t* slot_of) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < t;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t* row = rows + i * n;
    uint64_t s = row_hash(row, n) & mask;
    while (true) {
      unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&keys[s]);
      if (k == ~0ull) {
        k = atomicCAS(&keys[s], ~0ull, static_cast<unsigned long long>(i));
        if (k == ~0ull) break;
      }
      if (rows_equal(rows + static_cast<int64_t>(k) * n, row, n)) break;
      s = (s + 1) & mask;
    }
    slot_of[i] = static_cast<int64_t>(s);
    atomicMin(&rep[s], static_cast<long long>(i));
  }
}

struct DictSink {
  const int64_t* rows;
  int n;
  const int64_t* slot_of;
  int64_t* id_of_slot;
  int64_t* unique_out;
  __device__ void operator()(int64_t i, long long ex, long long v) const {
    if (!v) return;
    id_of_slot[slot_of[i]] = ex;
    for (int c = 0; c < n; ++c) unique_out[ex * n + c] = rows[i * n + c];
  }
};

__global__ void dict_finalize_kernel(int64_t* inverse, int64_t t, const int64_t* id_of_slot) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < t;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    inverse[i] = id_of_slot[inverse[i]];
}

// --------------------------------------------------------------------------
// Lexicographic order of the unique rows (the reference sorts rows
// lexicographically as signed int64, _kernels.pyx:20-30 / _py_kernels.py:24):
// an LSD radix sort of the U unique rows' indices — columns from last to first,
// 8-bit digits of the sign-flipped key from least to most significant, every
// pass stable — then the unique rows are gathered in that order and the
// inverse indices renumbered.  U is device-resident (no host round trip).
// --------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 4;
constexpr int kRadixTile = kRadixThreads * kRadixItems;
constexpr uint64_t kSignFlip = 0x8000000000000000ull;

__device__ __forceinline__ int64_t used_tiles(const int64_t* u) { return (*u + kRadixTile - 1) / kRadixTile; }

// keys[j] = column `col` of unique row perm[j] (perm = identity when init)
__global__ void lex_keys_kernel(const int64_t* __restrict__ uniq, int n, int col, int64_t* perm, bool init,
                                uint64_t* __restrict__ keys, const int64_t* __restrict__ num_unique) {
  const int64_t u = *num_unique;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < u;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (init) perm[j] = j;
    keys[j] = static_cast<uint64_t>(uniq[perm[j] * n + col]) ^ kSignFlip;
  }
}

// per tile: counts of each digit -> ghist[digit * ntiles + tile]
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint64_t* __restrict__ keys,
                                                                   const int64_t* __restrict__ num_unique,
                                                                   int shift, uint32_t* ghist, int64_t ntiles) {
  __shared__ uint32_t h[256];
  const int64_t tile = blockIdx.x;
  if (tile >= used_tiles(num_unique)) return;
  const int64_t u = *num_unique;
  h[threadIdx.x] = 0;
  __syncthreads();
  for (int k = 0; k < kRadixItems; ++k) {
    const int64_t j = tile * kRadixTile + k * kRadixThreads + threadIdx.x;
    if (j < u) atomicAdd(&h[(keys[j] >> shift) & 255u], 1u);
  }
  __syncthreads();
  ghist[threadIdx.x * ntiles + tile] = h[threadIdx.x];
}

// exclusive scan of one digit's tile counts (block d), and the digit's total
__global__ void __launch_bounds__(kRadixThreads) radix_scan_kernel(uint32_t* ghist, int64_t ntiles,
                                                                   const int64_t* __restrict__ num_unique,
                                                                   uint32_t* dtotal) {
  __shared__ uint32_t s[kRadixThreads];
  const int d = blockIdx.x;
  const int64_t nt = used_tiles(num_unique);
  uint32_t carry = 0;
  for (int64_t base = 0; base < nt; base += kRadixThreads) {
    const int64_t t = base + threadIdx.x;
    const uint32_t v = t < nt ? ghist[d * ntiles + t] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < kRadixThreads; off <<= 1) {  // inclusive Hillis-Steele scan
      const uint32_t x = threadIdx.x >= off ? s[threadIdx.x - off] : 0u;
      __syncthreads();
      s[threadIdx.x] += x;
      __syncthreads();
    }
    if (t < nt) ghist[d * ntiles + t] = carry + s[threadIdx.x] - v;
    carry += s[kRadixThreads - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) dtotal[d] = carry;
}

// stable scatter of one tile: destination = digit base + this tile's offset
// within the digit + rank among the tile's elements of that digit (in order)
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const uint64_t* __restrict__ kin, const int64_t* __restrict__ pin, uint64_t* __restrict__ kout,
    int64_t* __restrict__ pout, const int64_t* __restrict__ num_unique, int shift, const uint32_t* __restrict__ ghist,
    int64_t ntiles, const uint32_t* __restrict__ dtotal) {
  __shared__ uint32_t s_base[256], s_run[256], s_scan[256];
  __shared__ uint32_t s_w[kRadixThreads / 32][256];
  const int64_t tile = blockIdx.x;
  if (tile >= used_tiles(num_unique)) return;
  const int64_t u = *num_unique;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // digit bases: exclusive scan of the digit totals
  const uint32_t tot = dtotal[tid];
  s_scan[tid] = tot;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const uint32_t x = tid >= off ? s_scan[tid - off] : 0u;
    __syncthreads();
    s_scan[tid] += x;
    __syncthreads();
  }
  s_base[tid] = s_scan[tid] - tot + ghist[tid * ntiles + tile];
  s_run[tid] = 0;
  for (int k = 0; k < kRadixItems; ++k) {
    const int64_t j = tile * kRadixTile + k * kRadixThreads + tid;
    const bool valid = j < u;
    const uint64_t key = valid ? kin[j] : 0ull;
    const uint32_t d = valid ? static_cast<uint32_t>((key >> shift) & 255u) : 256u + lane;
#pragma unroll
    for (int w = 0; w < kRadixThreads / 32; ++w) s_w[w][tid] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(kFull, d);
    const int lrank = __popc(peers & ((1u << lane) - 1u));
    if (valid && lrank == 0) s_w[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t prefix = 0;
      for (int w = 0; w < warp; ++w) prefix += s_w[w][d];
      const uint32_t pos = s_base[d] + s_run[d] + prefix + static_cast<uint32_t>(lrank);
      kout[pos] = key;
      pout[pos] = pin[j];
    }
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < kRadixThreads / 32; ++w) add += s_w[w][tid];
    s_run[tid] += add;
    __syncthreads();
  }
}

// rank[perm[k]] = k; unique rows in sorted order
__global__ void lex_gather_kernel(const int64_t* __restrict__ uniq_fo, int n, const int64_t* __restrict__ perm,
                                  int64_t* __restrict__ rank, int64_t* __restrict__ unique_out,
                                  const int64_t* __restrict__ num_unique) {
  const int64_t u = *num_unique;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < u;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t src = perm[k];
    rank[src] = k;
    for (int c = 0; c < n; ++c) unique_out[k * n + c] = uniq_fo[src * n + c];
  }
}

__global__ void lex_inverse_kernel(int64_t* inverse, int64_t t, const int64_t* __restrict__ rank) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < t;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    inverse[i] = rank[inverse[i]];
}

// --------------------------------------------------------------------------
// Segment counting.
// --------------------------------------------------------------------------
// Shared-memory histogram of one segment; warp-aggregated for hot IDs.
template <bool kClip>
__global__ void __launch_bounds__(256)
    segment_smem_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ seg_len,
                        const int64_t* __restrict__ seg_off, int64_t b, int64_t u,
                        int32_t* __restrict__ counts_out, const int32_t* __restrict__ ref_max,
                        int64_t* __restrict__ num_out, int32_t* err) {
  extern __shared__ int s_cnt[];
  __shared__ unsigned long long s_hits;
  const int lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x; i < b; i += gridDim.x) {
    for (int64_t c = threadIdx.x; c < u; c += blockDim.x) s_cnt[c] = 0;
    if (threadIdx.x == 0) s_hits = 0;
    __syncthreads();
    const int64_t off = seg_off[i], len = seg_len[i];
    unsigned long long hits = 0;
    for (int64_t base = 0; base < len; base += blockDim.x) {
      const int64_t j = base + threadIdx.x;
      long long id = -1;
      if (j < len) {
        id = ids[off + j];
        if (id < 0 || id >= u) {
          atomicOr(err, TB_FLAG_ID_RANGE);
          id = -1;
        }
      }
      const unsigned act = __ballot_sync(kFull, id >= 0);
      if (id >= 0) {
        const unsigned peers = __match_any_sync(act, id);
        if (lane == __ffs(peers) - 1) {
          const int k = __popc(peers);
          const int old = atomicAdd(&s_cnt[id], k);
          if (kClip) {
            const int m = ref_max[i * u + id];
            const int avail = m > old ? m - old : 0;
            hits += avail < k ? avail : k;
          }
        }
      }
    }
    if (kClip) {
      for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(kFull, hits, o);
      if (lane == 0 && hits) atomicAdd(&s_hits, hits);
    }
    __syncthreads();
    if (kClip) {
      if (threadIdx.x == 0) num_out[i] = static_cast<int64_t>(s_hits);
    } else {
      int32_t* row = counts_out + i * u;
      for (int64_t c = threadIdx.x; c < u; c += blockDim.x) row[c] = s_cnt[c];
    }
    __syncthreads();
  }
}

// U too large for shared memory: the same algorithm on a global row.
template <bool kClip>
__global__ void __launch_bounds__(256)
    segment_global_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ seg_len,
                          const int64_t* __restrict__ seg_off, int64_t b, int64_t u,
                          int32_t* __restrict__ counts_out, const int32_t* __restrict__ ref_max,
                          int64_t* __restrict__ num_out, int32_t* scratch, int32_t* err) {
  __shared__ unsigned long long s_hits;
  const int lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x; i < b; i += gridDim.x) {
    int* cnt = kClip ? scratch + static_cast<int64_t>(blockIdx.x) * u : counts_out + i * u;
    for (int64_t c = threadIdx.x; c < u; c += blockDim.x) cnt[c] = 0;
    if (threadIdx.x == 0) s_hits = 0;
    __syncthreads();
    const int64_t off = seg_off[i], len = seg_len[i];
    unsigned long long hits = 0;
    for (int64_t base = 0; base < len; base += blockDim.x) {
      const int64_t j = base + threadIdx.x;
      long long id = -1;
      if (j < len) {
        id = ids[off + j];
        if (id < 0 || id >= u) {
          atomicOr(err, TB_FLAG_ID_RANGE);
          id = -1;
        }
      }
      const unsigned act = __ballot_sync(kFull, id >= 0);
      if (id >= 0) {
        const unsigned peers = __match_any_sync(act, id);
        if (lane == __ffs(peers) - 1) {
          const int k = __popc(peers);
          const int old = atomicAdd(&cnt[id], k);
          if (kClip) {
            const int m = ref_max[i * u + id];
            const int avail = m > old ? m - old : 0;
            hits += avail < k ? avail : k;
          }
        }
      }
    }
    if (kClip) {
      for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(kFull, hits, o);
      if (lane == 0 && hits) atomicAdd(&s_hits, hits);
    }
    __syncthreads();
    if (kClip && threadIdx.x == 0) num_out[i] = static_cast<int64_t>(s_hits);
    __syncthreads();
  }
}

__global__ void check_total_kernel(const int64_t* total, int64_t expect, int32_t* err) {
  if (threadIdx.x == 0 && *total != expect) atomicOr(err, TB_FLAG_SEGMENTS);
}

__global__ void count_binary_kernel(const int32_t* a, const int32_t* b, int32_t* out, int64_t count,
                                    int op) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t x = a[i], y = b[i];
    out[i] = op == 0 ? (x > y ? x : y) : (x < y ? x : y);
  }
}

unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

// exclusive scan of seg_lengths into `off` (b+...), with total check
int scan_segments(const int64_t* seg_lengths, int64_t b, int64_t num_ids, int64_t* off,
                  int64_t* bsum, int64_t* total, int32_t* err, cudaStream_t stream) {
  const int64_t nb = (b + kTile - 1) / kTile;
  SegLenValue f{seg_lengths};
  tile_sum_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(f, b, bsum);
  scan_bsums_kernel<<<1, kScanThreads, 0, stream>>>(bsum, nb, total);
  tile_scan_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(f, b, bsum, OffsetSink{off});
  check_total_kernel<<<1, 32, 0, stream>>>(total, num_ids, err);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

size_t segment_ws(int64_t b) {
  const int64_t nb = (b + kTile - 1) / kTile;
  return static_cast<size_t>(round_up(b * 8, 256) + round_up((nb + 1) * 8, 256) + 256);
}

}  // namespace

extern "C" {

size_t tb_windows_workspace_bytes(int64_t batch) {
  const int64_t nb = (batch + kTile - 1) / kTile;
  return static_cast<size_t>(round_up((batch + 1) * 8, 256) + round_up((nb + 1) * 8, 256) + 256);
}

int tb_flatten_windows(int32_t token_bytes, const void* ids, int64_t ld, int64_t width, const int64_t* lengths,
                       int64_t batch, int32_t n, int64_t* out, int64_t* total_out, void* workspace,
                       size_t workspace_bytes, void* stream_) {
  StreamDeviceGuard device_guard(stream_);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if ((token_bytes != 4 && token_bytes != 8) || batch < 0 || width < 0 || ld < width || n < 1 || !total_out)
    return TB_ERR_INVALID_ARG;
  if (batch == 0) {
    TB_CUDA(cudaMemsetAsync(total_out, 0, sizeof(int64_t), stream));
    return TB_OK;
  }
  if (!lengths || (!ids && width > 0) || !out) return TB_ERR_INVALID_ARG;
  if (workspace_bytes < tb_windows_workspace_bytes(batch) || !workspace) return TB_ERR_WORKSPACE;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  auto* off = reinterpret_cast<int64_t*>(ws);
  auto* bsum = reinterpret_cast<int64_t*>(ws + round_up((batch + 1) * 8, 256));
  const int64_t nb = (batch + kTile - 1) / kTile;
  WindowCount cnt{lengths, width, n};
  tile_sum_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(cnt, batch, bsum);
  scan_bsums_kernel<<<1, kScanThreads, 0, stream>>>(bsum, nb, total_out);
  tile_scan_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(cnt, batch, bsum, OffsetSink{off});
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((batch + 7) / 8, 4 * num_sms() * 8));
  if (token_bytes == 4)
    windows_fill_kernel<int32_t><<<grid, 256, 0, stream>>>(static_cast<const int32_t*>(ids), ld, batch, n, cnt,
                                                            off, out);
  else
    windows_fill_kernel<int64_t><<<grid, 256, 0, stream>>>(static_cast<const int64_t*>(ids), ld, batch, n, cnt,
                                                            off, out);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

size_t tb_unique_rows_workspace_bytes(int64_t t, int32_t n) {
  int64_t cap = 32;
  while (cap < 2 * t) cap <<= 1;
  const int64_t nb = (t + kTile - 1) / kTile;
  const int64_t nt = (t + kRadixTile - 1) / kRadixTile;
  // hash table (keys, representatives, ids) + tile sums, then the sort:
  // first-occurrence unique rows, keys x2, permutation x2, ranks, histograms
  return static_cast<size_t>(3 * round_up(cap * 8, 256) + round_up((nb + 1) * 8, 256) + 256 +
                             round_up(t * (n > 0 ? n : 1) * 8, 256) + 5 * round_up(t * 8, 256) +
                             round_up(256 * nt * 4, 256) + 256 * 4 + 256);
}

int tb_unique_rows(const int64_t* rows, int64_t t, int32_t n, int64_t* unique_out, int64_t* inverse_out,
                   int64_t* num_unique, void* workspace, size_t workspace_bytes, void* stream_) {
  StreamDeviceGuard device_guard(stream_);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (t < 0 || n < 0 || !num_unique) return TB_ERR_INVALID_ARG;
  if (t == 0) {
    TB_CUDA(cudaMemsetAsync(num_unique, 0, sizeof(int64_t), stream));
    return TB_OK;
  }
  if (!rows || !unique_out || !inverse_out) return TB_ERR_INVALID_ARG;
  if (workspace_bytes < tb_unique_rows_workspace_bytes(t, n) || !workspace) return TB_ERR_WORKSPACE;
  int64_t cap = 32;
  while (cap < 2 * t) cap <<= 1;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  auto* keys = reinterpret_cast<unsigned long long*>(ws);
  auto* rep = reinterpret_cast<long long*>(ws + round_up(cap * 8, 256));
  auto* id_of_slot = reinterpret_cast<int64_t*>(ws + 2 * round_up(cap * 8, 256));
  auto* bsum = reinterpret_cast<int64_t*>(ws + 3 * round_up(cap * 8, 256));
  const int64_t nb = (t + kTile - 1) / kTile;

  // the sort's buffers after the hash table
  unsigned char* q = ws + 3 * round_up(cap * 8, 256) + round_up((nb + 1) * 8, 256) + 256;
  auto take = [&](int64_t bytes) {
    unsigned char* r = q;
    q += round_up(bytes, 256);
    return r;
  };
  auto* uniq_fo = reinterpret_cast<int64_t*>(take(t * (n > 0 ? n : 1) * 8));
  auto* keys_a = reinterpret_cast<uint64_t*>(take(t * 8));
  auto* keys_b = reinterpret_cast<uint64_t*>(take(t * 8));
  auto* perm_a = reinterpret_cast<int64_t*>(take(t * 8));
  auto* perm_b = reinterpret_cast<int64_t*>(take(t * 8));
  auto* rank = reinterpret_cast<int64_t*>(take(t * 8));
  const int64_t ntiles = (t + kRadixTile - 1) / kRadixTile;
  auto* ghist = reinterpret_cast<uint32_t*>(take(256 * ntiles * 4));
  auto* dtotal = reinterpret_cast<uint32_t*>(take(256 * 4));

  // 1. hash dictionary: unique rows in first-occurrence order, inverse ids
  dict_init_kernel<<<grid_for(cap, 256), 256, 0, stream>>>(keys, rep, cap);
  dict_insert_kernel<<<grid_for(t, 256), 256, 0, stream>>>(rows, t, n, keys, rep,
                                                            static_cast<uint64_t>(cap - 1), inverse_out);
  FirstOccValue f{inverse_out, reinterpret_cast<const int64_t*>(rep)};
  tile_sum_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(f, t, bsum);
  scan_bsums_kernel<<<1, kScanThreads, 0, stream>>>(bsum, nb, num_unique);
  tile_scan_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(
      f, t, bsum, DictSink{rows, n, inverse_out, id_of_slot, uniq_fo});
  dict_finalize_kernel<<<grid_for(t, 256), 256, 0, stream>>>(inverse_out, t, id_of_slot);
  // 2. lexicographic order of the unique rows (stable LSD radix sort)
  for (int col = n - 1; col >= 0; --col) {
    lex_keys_kernel<<<grid_for(t, 256), 256, 0, stream>>>(uniq_fo, n, col, perm_a, col == n - 1, keys_a,
                                                          num_unique);
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 8 * pass;
      uint64_t* kin = (pass & 1) ? keys_b : keys_a;
      uint64_t* kout = (pass & 1) ? keys_a : keys_b;
      int64_t* pin = (pass & 1) ? perm_b : perm_a;
      int64_t* pout = (pass & 1) ? perm_a : perm_b;
      radix_hist_kernel<<<static_cast<unsigned>(ntiles), kRadixThreads, 0, stream>>>(kin, num_unique, shift, ghist,
                                                                                      ntiles);
      radix_scan_kernel<<<256, kRadixThreads, 0, stream>>>(ghist, ntiles, num_unique, dtotal);
      radix_scatter_kernel<<<static_cast<unsigned>(ntiles), kRadixThreads, 0, stream>>>(
          kin, pin, kout, pout, num_unique, shift, ghist, ntiles, dtotal);
    }
  }
  if (n == 0) lex_keys_kernel<<<grid_for(t, 256), 256, 0, stream>>>(uniq_fo, 1, 0, perm_a, true, keys_a, num_unique);
  // 3. rows in sorted order, inverse renumbered
  lex_gather_kernel<<<grid_for(t, 256), 256, 0, stream>>>(uniq_fo, n, perm_a, rank, unique_out, num_unique);
  lex_inverse_kernel<<<grid_for(t, 256), 256, 0, stream>>>(inverse_out, t, rank);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

size_t tb_segment_workspace_bytes(int64_t b, int64_t num_unique) {
  if (b < 0 || num_unique < 0) return 0;
  size_t ws = segment_ws(b);
  // clipped_numerators with U beyond shared memory: per-CTA count rows
  if (num_unique * 4 + 4096 > smem_optin()) {
    int64_t grid = b < 2 * num_sms() ? b : 2 * num_sms();
    ws += static_cast<size_t>(round_up(grid * num_unique * 4, 256));
  }
  return ws;
}

static int segment_common(bool clip, const int64_t* ids, int64_t num_ids, const int64_t* seg_lengths,
                          int64_t b, int64_t u, int32_t* counts_out, const int32_t* ref_max,
                          int64_t* num_out, int32_t* err, void* workspace, size_t workspace_bytes,
                          cudaStream_t stream) {
  if (b < 0 || u < 0 || num_ids < 0 || !err) return TB_ERR_INVALID_ARG;
  if (u > 0 && b > LLONG_MAX / u) return TB_ERR_CAPACITY;  // ngrams.py:109-113
  if (b == 0) return TB_OK;
  if (!seg_lengths || (num_ids > 0 && !ids)) return TB_ERR_INVALID_ARG;
  if (clip ? (!num_out || (u > 0 && !ref_max)) : (u > 0 && !counts_out)) return TB_ERR_INVALID_ARG;
  if (workspace_bytes < tb_segment_workspace_bytes(b, u) || !workspace) return TB_ERR_WORKSPACE;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  const int64_t nb = (b + kTile - 1) / kTile;
  int64_t* off = reinterpret_cast<int64_t*>(ws);
  int64_t* bsum = reinterpret_cast<int64_t*>(ws + round_up(b * 8, 256));
  int64_t* total = reinterpret_cast<int64_t*>(ws + round_up(b * 8, 256) + round_up((nb + 1) * 8, 256));
  int rc = scan_segments(seg_lengths, b, num_ids, off, bsum, total, err, stream);
  if (rc != TB_OK) return rc;
  const size_t smem = static_cast<size_t>(u) * 4;
  const int limit = smem_optin() - 4096;
  const int sms = num_sms();
  if (static_cast<int64_t>(smem) <= limit) {
    auto kern = clip ? segment_smem_kernel<true> : segment_smem_kernel<false>;
    if (smem > 48 * 1024)
      TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 1;
    TB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
    if (occ < 1) occ = 1;
    int64_t grid = static_cast<int64_t>(occ) * sms;
    if (grid > b) grid = b;
    kern<<<static_cast<unsigned>(grid), 256, smem, stream>>>(ids, seg_lengths, off, b, u, counts_out, ref_max,
                                                             num_out, err);
  } else {
    int64_t grid = b < 2 * sms ? b : 2 * sms;
    int32_t* scratch = reinterpret_cast<int32_t*>(ws + segment_ws(b));
    auto kern = clip ? segment_global_kernel<true> : segment_global_kernel<false>;
    kern<<<static_cast<unsigned>(grid), 256, 0, stream>>>(ids, seg_lengths, off, b, u, counts_out, ref_max,
                                                          num_out, scratch, err);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_segment_bincount(const int64_t* ids, int64_t num_ids, const int64_t* seg_lengths, int64_t b,
                        int64_t num_unique, int32_t* counts_out, int32_t* err_flag, void* workspace,
                        size_t workspace_bytes, void* stream) {
  StreamDeviceGuard device_guard(stream);
  return segment_common(false, ids, num_ids, seg_lengths, b, num_unique, counts_out, nullptr, nullptr,
                        err_flag, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int tb_clipped_numerators(const int64_t* ids, int64_t num_ids, const int64_t* seg_lengths, int64_t b,
                          const int32_t* ref_max, int64_t num_unique, int64_t* num_out, int32_t* err_flag,
                          void* workspace, size_t workspace_bytes, void* stream) {
  StreamDeviceGuard device_guard(stream);
  return segment_common(true, ids, num_ids, seg_lengths, b, num_unique, nullptr, ref_max, num_out, err_flag,
                        workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int tb_count_binary(const int32_t* a, const int32_t* b, int32_t* out, int64_t count, int32_t op, void* stream) {
  StreamDeviceGuard device_guard(stream);
  if (count < 0 || (op != 0 && op != 1)) return TB_ERR_INVALID_ARG;
  if (count == 0) return TB_OK;
  if (!a || !b || !out) return TB_ERR_INVALID_ARG;
  count_binary_kernel<<<grid_for(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, out, count, op);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

}  // extern "C"
