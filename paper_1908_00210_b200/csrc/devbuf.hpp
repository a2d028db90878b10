// RAII device allocation shared by the host-side parts of libgdi.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace gdi {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t alloc(size_t b) {
    reset();
    bytes = b;
    return b ? cudaMalloc(&p, b) : cudaSuccess;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace gdi
