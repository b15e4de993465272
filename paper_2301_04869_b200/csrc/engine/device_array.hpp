// Minimal owning device array, move-only, on a process-wide caching
// allocator: released blocks are kept (by rounded size) and handed to the next
// array of that size, so a new context / solver of a size seen before costs no
// cudaMalloc / cudaFree (cudaFree synchronises the device and, measured on
// the bench box, a fresh 1354/256 context's allocations took 0.03-0.7 s).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../kernels/stats.hpp"

namespace bipm {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Blocks freed by an owner may still be read by kernels in flight (owners
// do not know their streams): they wait in `pending` until the next
// allocation, which first synchronises their device once (allocations happen
// at setup) and only then recycles them.  Blocks are keyed by (rounded size,
// device).  Cached bytes are capped; beyond the cap blocks go back to the
// driver.
class DeviceCache {
 public:
  static DeviceCache& get() {
    static DeviceCache* c = new DeviceCache();  // never destroyed: no teardown-order issues
    return *c;
  }
  void* alloc(size_t bytes) {
    const size_t b = round(bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(m_);
    if (!pending_.empty()) {
      // synchronise every device the pending blocks live on, once
      std::vector<int> devs;
      for (const auto& pb : pending_)
        if (std::find(devs.begin(), devs.end(), pb.first.second) == devs.end())
          devs.push_back(pb.first.second);
      for (int d : devs) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
      }
      cudaSetDevice(dev);
      for (const auto& pb : pending_) free_.emplace(pb.first, pb.second);
      pending_.clear();
    }
    auto it = free_.find(Key{b, dev});
    if (it != free_.end()) {
      void* p = it->second;
      cached_ -= b;
      free_.erase(it);
      return p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {  // out of memory: give the cache back and retry once
      cudaGetLastError();
      trim_locked();
      cuda_check(cudaMalloc(&p, b), "cudaMalloc");
    }
    return p;
  }
  void release(void* p, size_t bytes) {
    if (!p) return;
    const size_t b = round(bytes);
    cudaPointerAttributes at{};
    int dev = 0;
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess) dev = at.device;
    cudaGetLastError();
    std::lock_guard<std::mutex> g(m_);
    if (cached_ + b > kCap) {
      cudaFree(p);  // synchronising, like the plain allocator
      return;
    }
    cached_ += b;
    pending_.emplace_back(Key{b, dev}, p);
  }

 private:
  static constexpr size_t kCap = size_t(24) << 30;
  static size_t round(size_t n) {
    const size_t q = n > (size_t(1) << 20) ? (size_t(2) << 20) : 512;
    return (n + q - 1) / q * q;
  }
  void trim_locked() {
    int dev = 0;
    cudaGetDevice(&dev);
    for (auto& pb : pending_) {
      cudaSetDevice(pb.first.second);
      cudaFree(pb.second);  // cudaFree synchronises its device
    }
    for (auto& kv : free_) {
      cudaSetDevice(kv.first.second);
      cudaFree(kv.second);
    }
    cudaSetDevice(dev);
    pending_.clear();
    free_.clear();
    cached_ = 0;
  }
  using Key = std::pair<size_t, int>;  // (rounded bytes, device)
  std::mutex m_;
  std::multimap<Key, void*> free_;
  std::vector<std::pair<Key, void*>> pending_;
  size_t cached_ = 0;
};

template <typename T>
class DArr {
 public:
  DArr() = default;
  explicit DArr(size_t n) { resize(n); }
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DArr& operator=(DArr&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DArr() { release(); }

  void resize(size_t n) {
    if (n == n_) return;
    release();
    if (n) p_ = static_cast<T*>(DeviceCache::get().alloc(n * sizeof(T)));
    n_ = n;
  }
  void upload(const std::vector<T>& v) {
    resize(v.size());
    if (n_) cuda_check(cudaMemcpy(p_, v.data(), n_ * sizeof(T), cudaMemcpyHostToDevice), "upload");
    stats().h2d_bytes += (long long)(n_ * sizeof(T));
  }
  void upload(const T* src, size_t n, cudaStream_t st) {
    resize(n);
    if (n_) cuda_check(cudaMemcpyAsync(p_, src, n_ * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
    stats().h2d_bytes += (long long)(n_ * sizeof(T));
  }
  // copy n <= size() elements into the front of the array (keeps its size:
  // some arrays carry alignment padding past their logical length)
  void copy_from(const T* src, size_t n, cudaStream_t st) {
    if (n > n_) throw std::runtime_error("copy_from: source longer than the array");
    if (n) cuda_check(cudaMemcpyAsync(p_, src, n * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
    stats().h2d_bytes += (long long)(n * sizeof(T));
  }
  void download(T* dst, size_t n, cudaStream_t st) const {
    if (n) cuda_check(cudaMemcpyAsync(dst, p_, n * sizeof(T), cudaMemcpyDeviceToHost, st), "download");
    stats().d2h_bytes += (long long)(n * sizeof(T));
  }
  std::vector<T> to_host() const {
    std::vector<T> v(n_);
    if (n_) cuda_check(cudaMemcpy(v.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "to_host");
    stats().d2h_bytes += (long long)(n_ * sizeof(T));
    return v;
  }
  void zero(cudaStream_t st) {
    if (n_) cuda_check(cudaMemsetAsync(p_, 0, n_ * sizeof(T), st), "memset");
  }
  T* get() { return p_; }
  const T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  void release() {
    if (p_) DeviceCache::get().release(p_, n_ * sizeof(T));
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace bipm
