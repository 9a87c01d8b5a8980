// host_par.h -- host-side parallel loop for setup / upload work (planners, copies): the full-size
// levels are O(nnz) = 10^8-10^9 host operations.
#pragma once
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

namespace igb {

// f(lo, hi) over contiguous chunks of [0, n) on up to 32 threads (serial below `grain` per thread).
template <class F>
void parallel_for(long long n, F&& f, long long grain = 1 << 16) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::max(1LL, std::min<long long>(std::min(hw, 32), n / grain));
  if (T <= 1) {
    f(0LL, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  f(0LL, n / T);
  for (auto& th : pool) th.join();
}

inline void par_memcpy(void* dst, const void* src, size_t bytes) {
  parallel_for((long long)bytes, [&](long long lo, long long hi) {
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, (size_t)(hi - lo));
  }, 1 << 24);
}

}  // namespace igb
