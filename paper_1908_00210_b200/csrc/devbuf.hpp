// RAII device allocation shared by the host-side parts of libgdi.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace gdi {

// Device buffers come from the device's stream-ordered memory pool
// (cudaMallocAsync/cudaFreeAsync on the legacy stream, pool kept warm by a
// release threshold set in use_device): one-shot batches create and destroy
// a session per call, and plain cudaMalloc/cudaFree (which synchronises the
// device) cost ~10-20 ms per call for the trace buffers. Owners synchronise
// their own streams before releasing (sessions, partitions and graphs are
// destroyed only after their work is done).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool plain = false;  // cudaMalloc'd (exportable through CUDA IPC; pool memory is not)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      if (plain)
        cudaFree(p);
      else
        cudaFreeAsync(p, 0);
    }
    p = nullptr;
    bytes = 0;
    plain = false;
  }
  cudaError_t alloc_plain(size_t b) {
    reset();
    bytes = b;
    plain = true;
    return b ? cudaMalloc(&p, b) : cudaSuccess;
  }
  cudaError_t alloc(size_t b) {
    reset();
    bytes = b;
    if (!b) return cudaSuccess;
    cudaError_t e = cudaMallocAsync(&p, b, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);  // usable from any stream from here on
    return e;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Page-locked host staging buffer (device -> host copies at DMA speed), also
// mapped into the device address space (kernels may write it directly).
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaHostAlloc(&p, b, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace gdi
