// Host-side parallel loop for the setup code (the reference's parallel_for,
// proj/src/core.cpp:67-85, plays the same role). Every index writes its own
// output slots, so results do not depend on the thread count.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace tgb {

inline int host_threads() {
  if (const char* s = std::getenv("TG_HOST_THREADS")) {
    const int v = std::atoi(s);
    if (v > 0) return v;
  }
  return std::max(1u, std::thread::hardware_concurrency());
}

// fn(i) for i in [0, n), dynamic chunks of `grain`; the first exception thrown
// by any index is rethrown on the calling thread after all workers stop.
template <class F>
void parallel_for(long n, F&& fn, long grain = 64) {
  const long chunks = (n + grain - 1) / grain;
  const int nt = static_cast<int>(std::min<long>(host_threads(), chunks));
  if (nt <= 1) {
    for (long i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<long> next{0};
  std::exception_ptr err;
  std::mutex mu;
  auto work = [&] {
    try {
      for (;;) {
        const long b = next.fetch_add(grain);
        if (b >= n) break;
        const long e = std::min(n, b + grain);
        for (long i = b; i < e; ++i) fn(i);
      }
    } catch (...) {
      std::lock_guard<std::mutex> lock(mu);
      if (!err) err = std::current_exception();
      next = n;
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace tgb
