// Host-side row-parallel loop for the per-call conversions around the device
// path (input validation, trace/record conversion into caller buffers): the
// one-shot batch API converts ~1M trace records per call, which single-threaded
// costs more than the PCIe copy that brought them over.
#pragma once

#include <cstddef>
#include <thread>
#include <vector>

namespace gdi {

// f(lo, hi) over [0, count) split into contiguous blocks; runs inline when
// count < min_rows (thread start-up would dominate). Returns the thread count.
template <typename F>
unsigned parallel_rows(std::size_t count, std::size_t min_rows, F&& f) {
  unsigned threads = std::thread::hardware_concurrency();
  threads = threads < 1 ? 1 : threads > 16 ? 16 : threads;
  if (count < min_rows || threads == 1) {
    f(std::size_t{0}, count);
    return 1;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  for (unsigned t = 1; t < threads; t++)
    pool.emplace_back([&f, count, threads, t]() { f(count * t / threads, count * (t + 1) / threads); });
  f(std::size_t{0}, count / threads);
  for (auto& th : pool) th.join();
  return threads;
}

}  // namespace gdi
