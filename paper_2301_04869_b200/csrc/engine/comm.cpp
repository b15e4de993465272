#include "comm.hpp"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/common.hpp"

namespace bipm {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- NCCL through dlopen (ABI of nccl.h 2.x; only the calls used here)
using ncclComm_t = void*;
struct NcclId {
  char internal[128];
};
enum { kNcclDouble = 8, kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclId, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*CommCount)(const ncclComm_t, int*) = nullptr;
  int (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    if (!api.h) {
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
      }
      if (!api.h) throw Error(kUnsupported, "NCCL not found (libnccl.so.2)");
      auto sym = [&](const char* s) {
        void* p = dlsym(api.h, s);
        if (!p) throw Error(kUnsupported, std::string("NCCL symbol missing: ") + s);
        return p;
      };
      api.GetUniqueId = reinterpret_cast<int (*)(NcclId*)>(sym("ncclGetUniqueId"));
      api.CommInitRank =
          reinterpret_cast<int (*)(ncclComm_t*, int, NcclId, int)>(sym("ncclCommInitRank"));
      api.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, ncclComm_t,
                                               cudaStream_t)>(sym("ncclAllReduce"));
      api.CommDestroy = reinterpret_cast<int (*)(ncclComm_t)>(sym("ncclCommDestroy"));
      api.CommCount = reinterpret_cast<int (*)(const ncclComm_t, int*)>(sym("ncclCommCount"));
      api.CommUserRank =
          reinterpret_cast<int (*)(const ncclComm_t, int*)>(sym("ncclCommUserRank"));
      api.GetErrorString = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
    }
    return api;
  }
  void check(int r, const char* what) {
    if (r != 0) throw std::runtime_error(std::string(what) + ": " + GetErrorString(r));
  }
};

class NcclCommImpl final : public Comm {
 public:
  NcclCommImpl(const uint8_t id[128], int nranks, int rank, int device) : n_(nranks), r_(rank) {
    NcclApi& api = NcclApi::get();
    NcclId nid;
    std::memcpy(nid.internal, id, 128);
    ck(cudaSetDevice(device), "cudaSetDevice");
    api.check(api.CommInitRank(&comm_, nranks, nid, rank), "ncclCommInitRank");
    // what the communicator itself reports (evidence the ranks joined)
    api.check(api.CommCount(comm_, &n_), "ncclCommCount");
    api.check(api.CommUserRank(comm_, &r_), "ncclCommUserRank");
    if (n_ != nranks || r_ != rank)
      throw std::runtime_error("ncclCommInitRank: communicator reports a different rank layout");
  }
  ~NcclCommImpl() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
  }
  int rank() const override { return r_; }
  int size() const override { return n_; }
  int kind() const override { return 1; }
  void allreduce(double* d, size_t n, RedOpKind op, cudaStream_t st) override {
    if (!n) return;
    const int o = op == RedOpKind::kSum ? kNcclSum : (op == RedOpKind::kMax ? kNcclMax : kNcclMin);
    NcclApi& api = NcclApi::get();
    api.check(api.AllReduce(d, d, n, kNcclDouble, o, comm_, st), "ncclAllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
  int n_, r_;
};

class HostCommImpl final : public Comm {
 public:
  HostCommImpl(HostAllreduceFn fn, void* user, int nranks, int rank)
      : fn_(fn), user_(user), n_(nranks), r_(rank) {}
  ~HostCommImpl() override {
    if (buf_) cudaFreeHost(buf_);
  }
  int rank() const override { return r_; }
  int size() const override { return n_; }
  int kind() const override { return 2; }
  void allreduce(double* d, size_t n, RedOpKind op, cudaStream_t st) override {
    if (!n) return;
    if (n > cap_) {
      if (buf_) cudaFreeHost(buf_);
      ck(cudaMallocHost(&buf_, n * sizeof(double)), "cudaMallocHost");
      cap_ = n;
    }
    ck(cudaMemcpyAsync(buf_, d, n * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
    fn_(user_, buf_, int64_t(n), int32_t(op));
    ck(cudaMemcpyAsync(d, buf_, n * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    ck(cudaStreamSynchronize(st), "sync");
  }

 private:
  HostAllreduceFn fn_;
  void* user_;
  int n_, r_;
  double* buf_ = nullptr;
  size_t cap_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const uint8_t id[128], int nranks, int rank, int device) {
  return std::make_unique<NcclCommImpl>(id, nranks, rank, device);
}

std::unique_ptr<Comm> make_host_comm(HostAllreduceFn fn, void* user, int nranks, int rank) {
  return std::make_unique<HostCommImpl>(fn, user, nranks, rank);
}

void nccl_unique_id(uint8_t out[128]) {
  NcclApi& api = NcclApi::get();
  NcclId id;
  api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

}  // namespace bipm
