// tb_launch.cuh — shape plan + launch helper shared by the kernel translation
// units and the runtime (tb_runtime.cu).
#pragma once

#include "tb_common.cuh"

namespace tbk {

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
  // warp-per-group kernel first (R <= kSparseMaxRefs); the pair / multi kernel
  // then scores the groups it lists, at workspace offset list_off
  bool sparse = false;
  size_t list_off = 0;
  size_t smem_bytes = 0;   // dynamic smem (smem mode)
  size_t gtab_stride = 0;  // per-CTA table bytes (global mode)
  int64_t grid = 0;
  size_t acc_bytes = 0;
  size_t ws_bytes = 0;
};

constexpr size_t kStaticSmemReserve = 2048;  // static __shared__ of the stats kernels (upper bound)
constexpr size_t kMultiStaticReserve = 3072;  // the multi-reference kernel's (its filter lists)
constexpr int64_t kGlobalGridCap = 2 * 148;
// fixed-size completion region at the start of the workspace, independent of N
constexpr size_t kAccBytes = ((kAccCopies * (2 * TB_MAX_ORDER + 2) * 8 + 256) + 255) / 256 * 256;

template <typename K>
int launch_kernel(K kern, const StatsParams& prm, const Plan& pl, int sms, bool persistent_fill,
                  size_t* attr_set, cudaStream_t stream, int threads = kThreads) {
  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  if (attr_set[dev & 63] < pl.smem_bytes + 1) {
    // (always: static + dynamic shared memory above 48 KiB needs the opt-in even
    // when the dynamic part alone is below it)
    TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(pl.smem_bytes)));
    // one shared-memory carveout for every stats kernel (no reconfiguration
    // between back-to-back launches of different kernels)
    if (!getenv("TB_DEBUG_NO_CARVEOUT"))
      TB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
    attr_set[dev & 63] = pl.smem_bytes + 1;
  }
  int64_t grid = pl.grid;
  if (persistent_fill) {
    // occupancy per (device, dynamic smem) of this kernel instantiation, cached:
    // the query costs microseconds on every launch otherwise
    // (keyed by the kernel too: every stats kernel has the same C++ type)
    static thread_local struct { const void* kern; int dev; size_t smem; int threads; int occ; } cache[16] = {};
    static thread_local int next = 0;
    int occ = 0;
    const void* kp = reinterpret_cast<const void*>(kern);
    for (auto& e : cache)
      if (e.occ > 0 && e.kern == kp && e.dev == dev && e.smem == pl.smem_bytes && e.threads == threads) occ = e.occ;
    if (occ == 0) {
      TB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, pl.smem_bytes));
      if (occ < 1) occ = 1;
      cache[next] = {kp, dev, pl.smem_bytes, threads, occ};
      next = (next + 1) & 15;
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
  // list mode (after the filter kernel): plain stream order — measured: with
  // programmatic serialization the hash-table kernel ran 1.6x slower behind it
  cfg.numAttrs = (no_pdl() || (prm.glist && pdl_mode() != 1)) ? 0 : 1;
  TB_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

// per-kernel launchers (one translation unit each); token_bytes 4 or 8
int launch_sparse(const StatsParams& prm, int sms, cudaStream_t stream, int token_bytes);
int launch_pair(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes);
int launch_multi(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes);
int launch_group(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes);
int launch_global(const StatsParams& prm, const Plan& pl, int sms, cudaStream_t stream, int token_bytes);
#ifdef TB_PHASES
int set_phases_pair(void* buf);
int set_phases_multi(void* buf);
int set_phases_group(void* buf);
#endif

}  // namespace tbk
