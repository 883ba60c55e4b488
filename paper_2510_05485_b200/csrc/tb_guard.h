// tb_guard.h — host-side helper shared by the C-ABI entry points.
#pragma once

#include <cuda_runtime.h>

// Makes the stream's device current for the duration of a C-ABI call (and
// restores the caller's): launches on a stream of another device than the
// current one would otherwise be refused.
struct StreamDeviceGuard {
  int prev = -1;
  explicit StreamDeviceGuard(const void* stream) {
    int d = 0, cur = 0;
    cudaStream_t st = static_cast<cudaStream_t>(const_cast<void*>(stream));
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    // (a stream being captured into a graph is left alone: queries on it would
    // invalidate the capture, and the capturing caller has its device current)
    if (stream && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone &&
        cudaStreamGetDevice(st, &d) == cudaSuccess &&
        cudaGetDevice(&cur) == cudaSuccess && cur != d && cudaSetDevice(d) == cudaSuccess)
      prev = cur;
    cudaGetLastError();
  }
  ~StreamDeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

