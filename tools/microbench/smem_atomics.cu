// Microbenchmark: latency of shared-memory loads / atomics on the B200, as seen
// by one warp per phase with 4 CTAs per SM (the fused kernel's regime).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_atomics smem_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) bench(unsigned long long* out, int active_threads) {
  __shared__ uint32_t tab[8192];
  for (int i = threadIdx.x; i < 8192; i += 256) tab[i] = 0xffffffffu;
  __syncthreads();
  const uint32_t slot = (threadIdx.x * 2654435761u + blockIdx.x * 97u) & 8191u;
  unsigned long long t0 = clock64();
  if (threadIdx.x < active_threads) {
    for (int rep = 0; rep < 8; ++rep) {
      const uint32_t s = (slot + rep * 611u) & 8191u;
      if (MODE == 0) {  // load + store
        uint32_t v = *reinterpret_cast<volatile uint32_t*>(&tab[s]);
        tab[s] = v + threadIdx.x;
      } else if (MODE == 1) {  // CAS on an empty slot
        atomicCAS(&tab[s], 0xffffffffu, threadIdx.x);
      } else if (MODE == 2) {  // atomic add
        atomicAdd(&tab[s], 1u);
      } else if (MODE == 3) {  // CAS via explicit PTX shared
        uint32_t old;
        asm volatile("atom.shared::cta.cas.b32 %0, [%1], %2, %3;" : "=r"(old)
                     : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&tab[s]))), "r"(0xffffffffu), "r"(threadIdx.x) : "memory");
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * sizeof(unsigned long long));
  unsigned long long h[4096];
  const char* names[] = {"ld+st", "atomicCAS", "atomicAdd", "ptx cas"};
  for (int active : {32, 128, 256}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int it = 0; it < 3; ++it) {
        switch (mode) {
          case 0: bench<0><<<592, 256>>>(d, active); break;
          case 1: bench<1><<<592, 256>>>(d, active); break;
          case 2: bench<2><<<592, 256>>>(d, active); break;
          case 3: bench<3><<<592, 256>>>(d, active); break;
        }
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 592 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long s = 0, mx = 0;
      for (int i = 0; i < 592; ++i) { s += h[i]; if (h[i] > mx) mx = h[i]; }
      printf("active %3d  %-10s: mean %6.0f cycles (8 ops/thread), max %llu\n", active, names[mode], double(s) / 592, mx);
    }
  }
  return 0;
}
