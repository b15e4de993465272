// Minimal owning device array (cudaMalloc / cudaFree), move-only.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels/stats.hpp"

namespace bipm {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

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
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
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
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace bipm
