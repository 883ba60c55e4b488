// Dependent-chain latency of shared-memory ops on the B200 (one warp, one CTA per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_latency smem_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void lat(unsigned long long* out, int iters) {
  __shared__ uint32_t tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = (i * 7 + 13) & 4095;
  __syncthreads();
  uint32_t idx = (threadIdx.x * 97) & 4095;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v;
    if (MODE == 0) {
      v = tab[idx];
    } else if (MODE == 1) {  // CAS that fails (value != compare): returns current
      asm volatile("atom.shared::cta.cas.b32 %0, [%1], %2, %3;" : "=r"(v) : "r"(base + 4 * idx), "r"(0xdeadbeefu), "r"(0u) : "memory");
    } else if (MODE == 2) {  // atomic add returning old
      asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(v) : "r"(base + 4 * idx), "r"(0u) : "memory");
    } else {  // volatile load
      asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4 * idx));
    }
    idx = (v + i) & 4095;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (idx == 0xffffffff) out[0] = 0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * sizeof(unsigned long long));
  unsigned long long h[1024];
  const char* names[] = {"lds", "atom cas (fail)", "atom add ret", "ld.volatile"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int threads : {1, 32}) {
      for (int it = 0; it < 2; ++it) {
        switch (mode) {
          case 0: lat<0><<<148, threads>>>(d, 1000); break;
          case 1: lat<1><<<148, threads>>>(d, 1000); break;
          case 2: lat<2><<<148, threads>>>(d, 1000); break;
          case 3: lat<3><<<148, threads>>>(d, 1000); break;
        }
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      printf("%-16s threads %2d: %llu cycles per dependent op\n", names[mode], threads, h[0]);
    }
  }
  return 0;
}
