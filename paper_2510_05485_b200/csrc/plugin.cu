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

size_t tb_unique_rows_workspace_bytes(int64_t t, int32_t n) {
  (void)n;
  int64_t cap = 32;
  while (cap < 2 * t) cap <<= 1;
  const int64_t nb = (t + kTile - 1) / kTile;
  return static_cast<size_t>(3 * round_up(cap * 8, 256) + round_up((nb + 1) * 8, 256) + 256);
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

  dict_init_kernel<<<grid_for(cap, 256), 256, 0, stream>>>(keys, rep, cap);
  dict_insert_kernel<<<grid_for(t, 256), 256, 0, stream>>>(rows, t, n, keys, rep,
                                                            static_cast<uint64_t>(cap - 1), inverse_out);
  FirstOccValue f{inverse_out, reinterpret_cast<const int64_t*>(rep)};
  tile_sum_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(f, t, bsum);
  scan_bsums_kernel<<<1, kScanThreads, 0, stream>>>(bsum, nb, num_unique);
  tile_scan_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, stream>>>(
      f, t, bsum, DictSink{rows, n, inverse_out, id_of_slot, unique_out});
  dict_finalize_kernel<<<grid_for(t, 256), 256, 0, stream>>>(inverse_out, t, id_of_slot);
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
