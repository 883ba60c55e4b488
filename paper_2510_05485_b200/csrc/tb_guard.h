// tb_guard.h — host-side helper shared by the C-ABI entry points.
#pragma once

#include <cuda_runtime.h>

// Makes the stream's device current for the duration of a C-ABI call (and
// restores the caller's): launches on a stream of another device than the
// current one would otherwise be refused.
struct StreamDeviceGuard {
  int prev = -1;
  explicit StreamDeviceGuard(const void* stream) {
    // the stream -> device map of the last stream seen on this thread is
    // cached: the queries cost more than the launch on the hot path
    static thread_local const void* last_stream = nullptr;
    static thread_local int last_dev = -1;
    if (!stream) return;
    int d = last_dev;
    if (stream != last_stream) {
      cudaStream_t st = static_cast<cudaStream_t>(const_cast<void*>(stream));
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      // (a stream being captured into a graph is left alone: queries on it
      // would invalidate the capture, and the capturing caller has its device current)
      if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone ||
          cudaStreamGetDevice(st, &d) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      last_stream = stream;
      last_dev = d;
    }
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != d && cudaSetDevice(d) == cudaSuccess) prev = cur;
  }
  ~StreamDeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
