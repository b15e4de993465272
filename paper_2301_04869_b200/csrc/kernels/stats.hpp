// Process-wide counters for the bench contract: kernels launched by this
// library and bytes moved across PCIe by it.
#pragma once

#include <atomic>

namespace bipm {

struct Stats {
  std::atomic<long long> launches{0};
  std::atomic<long long> h2d_bytes{0};
  std::atomic<long long> d2h_bytes{0};
};

inline Stats& stats() {
  static Stats s;
  return s;
}

inline void note_launch(int n = 1) { stats().launches += n; }

}  // namespace bipm
