// PCIe read bandwidth from pinned host memory on one B200: copy engine vs
// kernel loads (16-byte vector loads, grid-stride) vs TMA bulk copies
// (cp.async.bulk global->shared from host-mapped memory), 3-8 MB like the
// host-buffer path.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pcie_read.cu -o pcie_read
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void load_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + i);
}

__global__ void load_kernel_unroll(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = __ldg(src + i);
}

__global__ void bulk_kernel(const char* src, size_t bytes, uint32_t chunk, unsigned long long* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t bar;
  const size_t nchunks = (bytes + chunk - 1) / chunk;
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t nb = (uint32_t)((c + 1) * chunk <= bytes ? chunk : bytes - c * chunk);
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(nb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(sm)),
                   "l"(src + c * chunk), "r"(nb), "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(phase) : "memory");
    phase ^= 1;
    acc += sm[threadIdx.x % nb];
    __syncthreads();
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const size_t sizes[] = {3u << 20, 8u << 20};
  for (size_t bytes : sizes) {
    char* h; void* d; void* hd; unsigned long long* sink;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    for (size_t i = 0; i < bytes; ++i) h[i] = (char)i;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    auto timeit = [&](const char* name, auto fn) {
      for (int i = 0; i < 3; ++i) fn();
      cudaEventRecord(e0);
      const int reps = 20;
      for (int i = 0; i < reps; ++i) fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1000.0 * ms / reps;
      printf("%5.1f MB  %-34s %8.1f us  %6.1f GB/s\n", bytes / 1048576.0, name, us, bytes / us / 1e3);
    };
    timeit("cudaMemcpyAsync H2D", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); });
    const size_t n = bytes / 16;
    for (int blocks : {148, 296, 592, 1184}) {
      char nm[64];
      snprintf(nm, sizeof nm, "ld.16B grid %d x 256", blocks);
      timeit(nm, [&] { load_kernel<<<blocks, 256>>>((const int4*)hd, (int4*)d, n); });
      snprintf(nm, sizeof nm, "ld.16B x4 unrolled grid %d x 256", blocks);
      timeit(nm, [&] { load_kernel_unroll<<<blocks, 256>>>((const int4*)hd, (int4*)d, n); });
    }
    for (uint32_t chunk : {4096u, 16384u, 65536u}) {
      cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      for (int blocks : {296, 592, 1184}) {
        char nm[64];
        snprintf(nm, sizeof nm, "bulk %u B chunks grid %d", chunk, blocks);
        timeit(nm, [&] { bulk_kernel<<<blocks, 128, chunk>>>((const char*)hd, bytes, chunk, sink); });
      }
    }
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    cudaFreeHost(h); cudaFree(d); cudaFree(sink);
  }
  return 0;
}
