// Host <-> device scalar traffic of the interior-point control flow.
//
// The host only ever reads the few scalars that steer control flow (norms,
// step sizes, merit values, factorisation status).  HostLink reads them
// through one pinned staging buffer on the engine stream and, when the engine
// is one rank of a sharded solve, all-reduces them across ranks first
// (all_reduce_sum, executor.cpp:39-61).
#pragma once

#include <algorithm>
#include <array>

#include "engine.hpp"

namespace bipm {

class HostLink {
 public:
  explicit HostLink(Engine& eng) : e(eng) {
    cuda_check(cudaMallocHost(&pinned_, kSlots * sizeof(double)), "cudaMallocHost");
    slot_.resize(2);
  }
  ~HostLink() {
    if (pinned_) cudaFreeHost(pinned_);
  }
  HostLink(const HostLink&) = delete;
  HostLink& operator=(const HostLink&) = delete;

  // K doubles of device memory, stream-ordered after everything queued on e.st
  template <int K>
  std::array<double, K> fetch(const double* d) {
    static_assert(K <= kSlots, "HostLink: fetch too wide");
    cuda_check(cudaMemcpyAsync(pinned_, d, K * sizeof(double), cudaMemcpyDeviceToHost, e.st),
               "fetch");
    stats().d2h_bytes += K * (long long)sizeof(double);
    e.sync();
    std::array<double, K> r;
    std::copy(pinned_, pinned_ + K, r.begin());
    return r;
  }
  double fetch1(const double* d) { return fetch<1>(d)[0]; }
  // queue a one-double read into pinned slot k (read it after the next sync)
  void fetch_async(const double* d, int k) {
    cuda_check(cudaMemcpyAsync(pinned_ + k, d, sizeof(double), cudaMemcpyDeviceToHost, e.st),
               "fetch");
    stats().d2h_bytes += (long long)sizeof(double);
  }
  double pinned(int k) const { return pinned_[k]; }

  // cross-rank exchange; no-ops on a single GPU
  void allred(double* d, size_t n, RedOpKind op) {
    if (e.multi()) e.comm->allreduce(d, n, op, e.st);
  }
  double host_all(double v, RedOpKind op) {
    if (!e.multi()) return v;
    cuda_check(cudaMemcpyAsync(slot_.get(), &v, sizeof(double), cudaMemcpyHostToDevice, e.st),
               "h2d");
    e.comm->allreduce(slot_.get(), 1, op, e.st);
    return fetch1(slot_.get());
  }
  // lowest global scenario index over the ranks (-1: none)
  idx global_first_bad(idx local_bad) {
    if (!e.multi()) return local_bad;
    const double v = host_all(local_bad >= 0 ? double(local_bad) : 1e300, RedOpKind::kMin);
    return v < 1e299 ? idx(v) : -1;
  }

  static constexpr int kSlots = 64;

 private:
  Engine& e;
  double* pinned_ = nullptr;
  DArr<double> slot_;
};

}  // namespace bipm
