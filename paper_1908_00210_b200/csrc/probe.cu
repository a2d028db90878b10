// Measurement utility: sustained read bandwidth of an L2-resident buffer.
// The GDI sweep kernels work on graphs whose CSR and spins fit in L2 / shared
// memory, so their roofline denominator is the L2 read rate, which
// MEASURED_PEAKS.json does not record (it has the HBM copy rate). Vectorised
// 16-byte loads, grid = 4 CTAs per SM, buffer re-read `iters` times.
#include <cuda_runtime.h>

#include <cstdint>

namespace gdi {

namespace {

__global__ void __launch_bounds__(512) l2_read(const int4* __restrict__ buf, size_t n16, int iters, int* sink) {
  int acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int it = 0; it < iters; it++)
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride) {
      const int4 v = __ldcg(buf + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x7f7f7f7f) sink[0] = acc;
}

}  // namespace

cudaError_t probe_l2_read(size_t bytes, int iters, double* gbs) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int4* buf = nullptr;
  int* sink = nullptr;
  cudaError_t e = cudaMalloc(&buf, bytes);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&sink, sizeof(int));
  if (e != cudaSuccess) {
    cudaFree(buf);
    return e;
  }
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t n16 = bytes / 16;
  l2_read<<<4 * sms, 512>>>(buf, n16, 2, sink);  // warm: bring the buffer into L2
  cudaEventRecord(a);
  l2_read<<<4 * sms, 512>>>(buf, n16, iters, sink);
  cudaEventRecord(b);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *gbs = static_cast<double>(bytes) * iters / (ms * 1e-3) / 1e9;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace gdi
