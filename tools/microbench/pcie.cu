// PCIe host->device microbenchmark for the e2e path design:
// copy-engine H2D vs. kernel zero-copy reads of pinned (mapped) host memory,
// with LDG.128 and with cp.async.bulk (TMA engine) into shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie pcie.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

// each CTA reads `row_bytes[b]` bytes of row b (row stride `ld`)
__global__ void zc_ldg(const int4* __restrict__ src, int64_t ld16, const int* __restrict__ row16, int rows,
                       unsigned long long* out) {
  unsigned long long acc = 0;
  for (int b = blockIdx.x; b < rows; b += gridDim.x) {
    const int4* r = src + b * ld16;
    const int n = row16[b];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int4 v = r[i];
      acc += (unsigned)(v.x ^ v.y ^ v.z ^ v.w);
    }
  }
  if (acc == 0x1234567) atomicAdd(out, acc);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void zc_bulk(const char* __restrict__ src, int64_t ld, const int* __restrict__ row16, int rows,
                        unsigned long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 16;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  unsigned long long acc = 0;
  for (int b = blockIdx.x; b < rows; b += gridDim.x) {
    const uint32_t bytes = row16[b] * 16;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf)), "l"(src + b * ld), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
    }
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(mbar)), "r"(phase));
    }
    phase ^= 1;
    for (int i = threadIdx.x; i < (int)(bytes / 4); i += blockDim.x) acc += reinterpret_cast<unsigned*>(buf)[i];
    __syncthreads();
  }
  if (acc == 0x1234567) atomicAdd(out, acc);
}

int main() {
  const int rows = 1024;          // 512 cand + 512 ref rows
  const int64_t L = 1024;         // int64 tokens
  const int64_t ld = L * 8;       // bytes
  const size_t total = rows * ld; // 8 MiB
  char* h;
  CK(cudaHostAlloc(&h, total, cudaHostAllocDefault));
  for (size_t i = 0; i < total; ++i) h[i] = (char)(i * 7);
  void* pageable = malloc(total);
  char* d;
  CK(cudaMalloc(&d, total));
  std::vector<int> full(rows), pref(rows);
  srand(1);
  int64_t pref_bytes = 0;
  for (int b = 0; b < rows; ++b) {
    full[b] = (int)(ld / 16);
    const int len = 512 + rand() % 513;
    pref[b] = (len * 8 + 15) / 16;
    pref_bytes += pref[b] * 16;
  }
  int *dfull, *dpref;
  CK(cudaMalloc(&dfull, rows * 4));
  CK(cudaMalloc(&dpref, rows * 4));
  CK(cudaMemcpy(dfull, full.data(), rows * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpref, pref.data(), rows * 4, cudaMemcpyHostToDevice));
  unsigned long long* dout;
  CK(cudaMalloc(&dout, 8));
  char* hd = nullptr;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  printf("host %p device-view %p (same=%d)\n", (void*)h, (void*)hd, hd == h);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, double bytes, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1000 / reps;
    printf("%-40s %8.1f us  %7.1f GB/s  (%.2f MB)\n", name, us, bytes / us / 1e3, bytes / 1e6);
  };
  timeit("memcpy H2D pinned (full)", total, [&] { CK(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice)); });
  timeit("memcpy H2D pageable (full)", total, [&] { CK(cudaMemcpyAsync(d, pageable, total, cudaMemcpyHostToDevice)); });
  timeit("memcpy D2D (full)", total, [&] { CK(cudaMemcpyAsync(d, d + total / 2, total / 2, cudaMemcpyDeviceToDevice)); });
  for (int grid : {148, 296, 592, 1024}) {
    for (int thr : {128, 256, 512}) {
      char name[64];
      snprintf(name, sizeof name, "zc LDG128 full g=%d t=%d", grid, thr);
      timeit(name, total, [&] { zc_ldg<<<grid, thr>>>((const int4*)hd, ld / 16, dfull, rows, dout); });
      snprintf(name, sizeof name, "zc LDG128 prefix g=%d t=%d", grid, thr);
      timeit(name, pref_bytes, [&] { zc_ldg<<<grid, thr>>>((const int4*)hd, ld / 16, dpref, rows, dout); });
    }
  }
  CK(cudaFuncSetAttribute(zc_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 + ld));
  for (int grid : {296, 592, 1024}) {
    char name[64];
    snprintf(name, sizeof name, "zc bulk(TMA) prefix g=%d", grid);
    timeit(name, pref_bytes, [&] { zc_bulk<<<grid, 256, 16 + ld>>>(hd, ld, dpref, rows, dout); });
    CK(cudaGetLastError());
  }
  timeit("device LDG128 prefix g=1024 t=256", pref_bytes, [&] { zc_ldg<<<1024, 256>>>((const int4*)d, ld / 16, dpref, rows, dout); });
  CK(cudaDeviceSynchronize());
  printf("ok\n");
  return 0;
}
