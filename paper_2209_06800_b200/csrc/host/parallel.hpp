// Minimal fork-join helper for the host builders. std::thread rather than
// OpenMP so the library never drags a second OpenMP runtime into a process
// that already has PyTorch's.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <thread>
#include <vector>

namespace mgg::detail {

inline unsigned host_threads() {
  static const unsigned n = [] {
    unsigned h = std::thread::hardware_concurrency();
    return std::clamp(h, 1u, 64u);
  }();
  return n;
}

/// Runs fn(t, begin, end) over `chunks` contiguous slices of [0, n) on up to
/// host_threads() threads; slice t is always [n*t/chunks, n*(t+1)/chunks).
/// Exceptions from any slice are rethrown (first one wins).
template <class Fn>
void parallel_slices(std::uint64_t n, unsigned chunks, Fn&& fn) {
  if (chunks <= 1 || n < 2) {
    fn(0u, std::uint64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(chunks);
  const unsigned workers = std::min(chunks, host_threads());
  for (unsigned w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (unsigned t = w; t < chunks; t += workers) {
        try {
          fn(t, n * t / chunks, n * (t + 1) / chunks);
        } catch (...) {
          errs[t] = std::current_exception();
        }
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

/// Same, sized for n items with at least `grain` items per slice.
template <class Fn>
void parallel_for(std::uint64_t n, std::uint64_t grain, Fn&& fn) {
  const std::uint64_t want = grain ? n / grain : n;
  const unsigned chunks =
      static_cast<unsigned>(std::clamp<std::uint64_t>(want, 1, host_threads() * 4ull));
  parallel_slices(n, chunks, [&](unsigned, std::uint64_t b, std::uint64_t e) {
    fn(b, e);
  });
}

}  // namespace mgg::detail
