// Streamed Schur reduction (reduce_stream.cu): the multi-RHS tile loop of
// reduce_group (kkt.cpp:371-466) as a warp-specialised kernel.  One producer
// warp stages every step's data (host/stream_plan.hpp) into a shared-memory
// ring with bulk async copies (TMA, mbarrier complete_tx); 16 consumer warps
// run the steps on an n_x x K panel resident in shared memory.
#pragma once

#include <cuda_runtime.h>

#include "device_plan.cuh"

namespace bipm {

constexpr int kStreamArrays = 7;

struct StreamLaunch {
  int n_x, n_u, M, K, nq, steps, ring_bytes, t0, tl;
  int chunk, nchunks;
  int consumers;        // consumer threads per CTA (128, 256 or 512; + one producer warp)
  int ctas_per_sm;      // co-resident CTAs the shared memory plan allows
  int list_cap;         // tile list entries (G_u + K_xu columns, each rounded to even)
  const int* pat;       // pattern blocks
  const int* issue;     // StepIssue records (12 ints each)
  const int* ring_off;  // per step: ring word (reduce_stream.cu kRw*: offset, skip control)
  const double* arr[kStreamArrays];
  long long stride[kStreamArrays];
  DevCsr gu, kxu, kuu;  // transposed views give a tile's columns
  const int* iperm;
  const double *gu_v, *kxu_v, *kuu_v;
  double dw;
  // presolved forward half (ReachPlan, reach_gemm.cu): the tile starts from
  // y_N (reach rows, [M][nnz_yn], column-major by control) and X_T
  // ([M][n_u][ldy]) instead of G_u
  int presolved, ldy, nnz_yn;
  const int *yn_ptr, *yn_row;
  const double *yn_v, *xt;
  double* zt;  // [M][n_u][ldy]: Z_T of every column (kStoreTail)
  double* partial;   // [nchunks][n_u * n_u] column-major
  double* scratch;   // per CTA: n_x * K (S = K~_xx T + K_xu V staging)
  long long* phase;  // optional: clock64 per step of CTA 0's first scenario
  int debug;         // timing experiments only (BIPM_STREAM_DEBUG): 1 skip sweeps, 2 no team barriers, 4 no K~_xx product stores
};

// largest consumer count per CTA (one producer warp is added)
constexpr int kStreamConsumers = 512;
// producer lookahead cap in steps (< the kernel's 32 mbarrier slots)
constexpr int kStreamLookahead = 24;
// accumulator registers per consumer: n_u * K <= 512 * kStreamMaxQ
constexpr int kStreamMaxQ = 10;

size_t stream_smem_bytes(int n_x, int K, int tl, int steps, int list_cap, int ring_bytes);
// largest ring that fits next to the panel (0 when the panel does not fit)
int stream_ring_capacity(int n_x, int K, int tl, int steps, int list_cap, int ctas_per_sm);
void plan_stream_chunks(StreamLaunch& a, int sm_count);
void launch_reduce_stream(const StreamLaunch& a, cudaStream_t st);
// out[col q][row q] = sum_s kuu[s][q] (the K_uu V terms of K_hat)
void launch_kuu_sum(const double* kuu, long long stride, const int* row, const int* col, int nnz,
                    int M, int n_u, double* out, cudaStream_t st);
// out[s][q] = in[s][slot[q]]  (column-order copies of K_xu and G_u values)
void launch_gather_values(const double* in, long long in_stride, const int* slot, int n,
                          double* out, long long out_stride, int M, cudaStream_t st);

}  // namespace bipm
