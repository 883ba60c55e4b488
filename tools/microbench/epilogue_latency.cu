// Latency (SM cycles, one warp alone) of the per-group fp64 epilogue pieces of
// tensorbleu.cu: fp64 division, brevity penalty, the whole warp_epilogue.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o epilogue_latency epilogue_latency.cu
#include "../../paper_2510_05485_b200/csrc/tensorbleu.cu"

__global__ void probe(const int64_t* in, double* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const int64_t num = in[lane], den = in[32 + lane], c = in[64], r = in[65];
  double acc = 0;
  __syncwarp();
  long long t0 = clock64();
  double q = __ddiv_rn(static_cast<double>(num), static_cast<double>(den));
  acc += q;
  __syncwarp();
  long long t1 = clock64();
  double bp = brevity_penalty_fp64(c, r);
  acc += bp;
  __syncwarp();
  long long t2 = clock64();
  warp_epilogue(num, den, c, r, 4, TB_SMOOTH_NONE, 0.1, 1.0, lane < 4 ? 0.25 : 0.0, out + 8, out + 1, out + 2);
  __syncwarp();
  long long t3 = clock64();
  warp_epilogue(num, den, c, r, 4, TB_SMOOTH_EXP, 0.1, 1.0, lane < 4 ? 0.25 : 0.0, out + 8, out + 1, out + 2);
  __syncwarp();
  long long t4 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    out[0] = acc;
  }
}

int main() {
  int64_t h[66];
  for (int i = 0; i < 32; ++i) {
    h[i] = i < 4 ? 10 + i : 0;
    h[32 + i] = i < 4 ? 700 - i : 0;
  }
  h[64] = 700;
  h[65] = 720;
  int64_t* d;
  double* o;
  long long* cy;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 64 * 8);
  cudaMalloc(&cy, 4 * 8);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) {
    probe<<<1, 32>>>(d, o, cy);
    long long c[4];
    cudaMemcpy(c, cy, sizeof c, cudaMemcpyDeviceToHost);
    printf("ddiv %lld  bp %lld  warp_epilogue(none, all p>0) %lld  (exp) %lld cycles\n", c[0], c[1], c[2], c[3]);
  }
  h[1] = 0;  // p_2 = 0 -> score 0 path
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  probe<<<1, 32>>>(d, o, cy);
  long long c[4];
  cudaMemcpy(c, cy, sizeof c, cudaMemcpyDeviceToHost);
  printf("with a zero precision: warp_epilogue(none) %lld  (exp) %lld cycles\n", c[2], c[3]);
  return 0;
}
