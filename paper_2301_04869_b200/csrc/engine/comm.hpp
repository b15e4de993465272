// Cross-GPU exchange for the scenario-sharded solve.
//
// Each rank owns a contiguous scenario group (partition, executor.cpp:7-19)
// and keeps its bundle, factors and panels resident.  The only exchanges are
// all-reduces of device buffers: the reduced matrix and rhs partial sums
// (finish_reduce -> all_reduce_sum, kkt.cpp:468-488, executor.cpp:39-61), the
// u-row sums, and the scalar norms / merit terms of the globalisation.
//
//   NcclComm  - ncclAllReduce on the engine stream (NVLink / NVSwitch); NCCL
//               is loaded with dlopen so single-GPU use needs no NCCL.
//   HostComm  - stages through pinned host memory and calls a user callback
//               (tests run two ranks on one GPU with a gloo all-reduce).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

namespace bipm {

enum class RedOpKind : int { kSum = 0, kMax = 1, kMin = 2 };

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual int kind() const = 0;  // 1 NCCL, 2 host callback
  // in-place all-reduce of n doubles of device memory, ordered on stream st
  virtual void allreduce(double* d, size_t n, RedOpKind op, cudaStream_t st) = 0;
};

using HostAllreduceFn = void (*)(void* user, double* buf, int64_t n, int32_t op);

std::unique_ptr<Comm> make_nccl_comm(const uint8_t id[128], int nranks, int rank, int device);
std::unique_ptr<Comm> make_host_comm(HostAllreduceFn fn, void* user, int nranks, int rank);
void nccl_unique_id(uint8_t out[128]);

}  // namespace bipm
