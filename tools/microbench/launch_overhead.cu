// Host-side cost of the C ABI calls, without Python: tb_bleu_stats (launch
// only, and launch + sync) and tb_bleu_host on a tiny batch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_overhead launch_overhead.cu \
//        -I../../include -L../../paper_2510_05485_b200 -ltensorbleu_b200 -Xlinker -rpath=$PWD/../../paper_2510_05485_b200
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "tensorbleu.h"

__global__ void empty_kernel() {}
// completion by a flag in mapped pinned memory (host spins instead of syncing)
__global__ void flag_kernel(volatile unsigned* flag, unsigned seq) {
  __threadfence_system();
  *flag = seq;
}

template <typename F>
double time_us(F f, int reps = 2000) {
  for (int i = 0; i < 50; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  const int B = 1, L = 8, N = 4;
  int64_t *d_ids, *d_len, *d_num;
  double* d_sc;
  int32_t* d_err;
  void* ws;
  cudaMalloc(&d_ids, B * L * 8);
  cudaMalloc(&d_len, B * 8);
  cudaMalloc(&d_num, B * N * 8);
  cudaMalloc(&d_sc, B * 8);
  cudaMalloc(&d_err, 4);
  cudaMemset(d_ids, 0, B * L * 8);
  int64_t len = L;
  cudaMemcpy(d_len, &len, 8, cudaMemcpyHostToDevice);
  int64_t w = L;
  size_t wsb = tb_bleu_workspace_bytes(B, 1, L, &w, 8, N);
  cudaMalloc(&ws, wsb);
  cudaMemset(ws, 0, wsb);
  double wts[4] = {0.25, 0.25, 0.25, 0.25};
  const void* rids[1] = {d_ids};
  int64_t rld[1] = {L}, rw[1] = {L};
  const int64_t* rlen[1] = {d_len};
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto launch = [&] {
    tb_bleu_stats(8, d_ids, L, L, d_len, 1, rids, rld, rw, rlen, B, N, 0, 0.1, 1.0, wts, nullptr, nullptr,
                  nullptr, nullptr, d_sc, nullptr, nullptr, nullptr, nullptr, d_err, ws, wsb, st);
  };
  printf("tb_bleu_stats launch only      %7.2f us\n", time_us(launch));
  cudaStreamSynchronize(st);
  printf("tb_bleu_stats launch + sync    %7.2f us\n", time_us([&] { launch(); cudaStreamSynchronize(st); }));
  printf("empty kernel + sync            %7.2f us\n", time_us([&] { empty_kernel<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st); }));
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float tot = 0;
    for (int i = 0; i < 200; ++i) {
      cudaEventRecord(e0, st);
      launch();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("tb_bleu_stats event-timed      %7.2f us\n", tot * 1000 / 200);
    tot = 0;
    for (int i = 0; i < 200; ++i) {
      cudaEventRecord(e0, st);
      empty_kernel<<<1, 32, 0, st>>>();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("empty kernel event-timed       %7.2f us\n", tot * 1000 / 200);
  }
  printf("empty stream sync              %7.2f us\n", time_us([&] { cudaStreamSynchronize(st); }));
  {
    unsigned* hflag;
    cudaHostAlloc(&hflag, 64, cudaHostAllocMapped);
    unsigned* dflag;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), hflag, 0);
    unsigned seq = 0;
    *hflag = 0;
    printf("flag kernel + host spin        %7.2f us\n", time_us([&] {
      ++seq;
      flag_kernel<<<1, 32, 0, st>>>(dflag, seq);
      while (*reinterpret_cast<volatile unsigned*>(hflag) != seq) {
      }
    }));
    cudaStreamSynchronize(st);
    printf("flag kernel + sync             %7.2f us\n", time_us([&] {
      ++seq;
      flag_kernel<<<1, 32, 0, st>>>(dflag, seq);
      cudaStreamSynchronize(st);
    }));
    unsigned* hflag2;
    cudaHostAlloc(&hflag2, 64, cudaHostAllocMapped);
    printf("host->pinned write + read      %7.2f us\n", time_us([&] { *reinterpret_cast<volatile unsigned*>(hflag2) = seq; }));
  }
  int64_t *h_ids, *h_len;
  cudaHostAlloc(&h_ids, B * L * 8, 0);
  cudaHostAlloc(&h_len, B * 8, 0);
  memset(h_ids, 0, B * L * 8);
  *h_len = L;
  const void* hr[1] = {h_ids};
  const int64_t* hl[1] = {h_len};
  double sc;
  int32_t flags;
  auto host = [&] {
    tb_bleu_host(8, h_ids, L, L, h_len, 1, hr, rld, rw, hl, B, N, 0, 0.1, 1.0, wts, nullptr, nullptr, nullptr,
                 nullptr, &sc, nullptr, nullptr, nullptr, nullptr, &flags, st);
  };
  printf("tb_bleu_host (pinned) blocking %7.2f us\n", time_us(host));
  std::vector<int64_t> pg_ids(B * L, 0), pg_len(B, L);
  const void* pr[1] = {pg_ids.data()};
  const int64_t* pl[1] = {pg_len.data()};
  auto pageable = [&] {
    tb_bleu_host(8, pg_ids.data(), L, L, pg_len.data(), 1, pr, rld, rw, pl, B, N, 0, 0.1, 1.0, wts, nullptr,
                 nullptr, nullptr, nullptr, &sc, nullptr, nullptr, nullptr, nullptr, &flags, st);
  };
  printf("tb_bleu_host (pageable)        %7.2f us\n", time_us(pageable));
  cudaPointerAttributes a;
  printf("cudaPointerGetAttributes       %7.2f us\n", time_us([&] { cudaPointerGetAttributes(&a, h_ids); }));
  printf("sc=%f flags=%d\n", sc, flags);
  {  // c2-shaped host call: 512 x 1024 int32 pinned rows, lengths U[512, 1024]
    const int B2 = 512, L2 = 1024;
    int32_t *hc, *hr;
    int64_t *lc, *lr;
    cudaHostAlloc(&hc, B2 * L2 * 4, 0);
    cudaHostAlloc(&hr, B2 * L2 * 4, 0);
    cudaHostAlloc(&lc, B2 * 8, 0);
    cudaHostAlloc(&lr, B2 * 8, 0);
    srand(3);
    for (int i = 0; i < B2 * L2; ++i) {
      hc[i] = rand() % 128000;
      hr[i] = rand() % 128000;
    }
    for (int i = 0; i < B2; ++i) {
      lc[i] = 512 + rand() % 513;
      lr[i] = 512 + rand() % 513;
    }
    std::vector<double> scores(B2);
    const void* r2[1] = {hr};
    const int64_t* l2[1] = {lr};
    int64_t ld2[1] = {L2}, w2[1] = {L2};
    auto call = [&] {
      tb_bleu_host(4, hc, L2, L2, lc, 1, r2, ld2, w2, l2, B2, N, 0, 0.1, 1.0, wts, nullptr, nullptr, nullptr,
                   nullptr, scores.data(), nullptr, nullptr, nullptr, nullptr, &flags, st);
    };
    printf("tb_bleu_host c2 int32 pinned   %7.2f us\n", time_us(call, 200));
    cudaEvent_t a, b2;
    cudaEventCreate(&a);
    cudaEventCreate(&b2);
    float tot = 0;
    for (int i = 0; i < 50; ++i) {
      cudaEventRecord(a, st);
      call();
      cudaEventRecord(b2, st);
      cudaEventSynchronize(b2);
      float ms;
      cudaEventElapsedTime(&ms, a, b2);
      tot += ms;
    }
    printf("  (events around it: %7.2f us)\n", tot * 1000 / 50);
  }
  return 0;
}
