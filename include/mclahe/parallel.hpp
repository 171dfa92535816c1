// mclahe/parallel.hpp -- the reference's host worker helpers
// (/root/reference/proj/core/include/mclahe/parallel.hpp:12-61), kept so
// callers that use them compile.  The GPU path does not: a CUDA grid replaces
// parallel_for inside mclahe::mclahe.
//
// Contract (as the reference's): threads == 0 means every hardware thread;
// chunk bounds are a function of (count, workers) only, so per-index
// computations reproduce bit for bit for any worker count; the first
// exception thrown by a worker is rethrown on the caller's thread.
#pragma once

#include <algorithm>
#include <cstddef>
#include <exception>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

namespace mclahe {

inline unsigned resolve_threads(unsigned requested) {
  if (requested) return requested;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? hw : 1u;
}

template <typename Fn>
void parallel_for(std::size_t count, unsigned threads, Fn&& fn) {
  if (count == 0) return;
  const std::size_t workers = std::min<std::size_t>(resolve_threads(threads), count);
  if (workers <= 1) {
    fn(std::size_t{0}, count);
    return;
  }
  // worker w gets [w * count / workers, (w + 1) * count / workers)
  auto bound = [&](std::size_t w) { return w * (count / workers) + std::min(w, count % workers); };
  std::exception_ptr first_error;
  std::mutex guard;
  auto body = [&](std::size_t w) {
    try {
      fn(bound(w), bound(w + 1));
    } catch (...) {
      std::lock_guard<std::mutex> lock(guard);
      if (!first_error) first_error = std::current_exception();
    }
  };
  std::vector<std::thread> helpers;
  helpers.reserve(workers - 1);
  for (std::size_t w = 1; w < workers; ++w) helpers.emplace_back(body, w);
  body(0);
  for (auto& t : helpers) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

}  // namespace mclahe
