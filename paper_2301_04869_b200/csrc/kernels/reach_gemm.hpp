// Forward half of the Schur reduction solved once per scenario for all
// control columns (host/stream_plan.hpp ReachPlan), and the batched FP64
// tensor-core GEMM that applies the dense tail inverse to it.
#pragma once

#include <cuda_runtime.h>

namespace bipm {

struct ReachDev {
  int n_u, tl, ldy, nnz_yn;
  int ymax;           // largest column reach (y_N entries of one column)
  int group;          // lanes per column (4, 8, 16 or 32: ~ entries per op)
  const int* op_ptr;  // [n_u + 1]
  const int4* ops;    // {dest, G_u slot or -1, entry begin, entry end}
  const int2* ent;    // {source y_N entry (column-local), L factor slot}
  const int* yn_ptr;  // [n_u + 1]
  // packed: y_T holds only y_T's pattern (yt_ptr / yt_row order), [M][nnz_yt]
  int packed, nnz_yt;
  const int* yt_ptr;  // [n_u + 1]
};

// y_N [M][nnz_yn] and y_T -- [M][n_u][ldy] (rows >= tl zero), or packed
// [M][nnz_yt] -- from the factors
// F [M][nnz_f] and the G_u values [M][gu_nnz]
void launch_reach_solve(const ReachDev& p, int M, const double* F, long long nnz_f,
                        const double* gu, long long gu_nnz, double* yn, double* yt,
                        cudaStream_t st);

// X_T = W y_T for every scenario with y_T's column pattern (yt_ptr, yt_row,
// tail-local rows) and packed values ytc [M][nnz_yt]: WT = W' = W transposed,
// rows of ldw doubles, scenario stride sw; xt [M][n_u][ldy]
void launch_xt_sparse(const double* WT, int ldw, long long sw, const double* ytc, int nnz_yt,
                      const int* yt_ptr, const int* yt_row, int n_u, int tl, int M, double* xt,
                      int ldy, cudaStream_t st);

// C[b](i, j) = alpha sum_k A[b][i lda + k] B[b][j ldb + k]  (both operands
// k-contiguous, C column-major: C[b][j ldc + i]), i < m, j < n, k < kd;
// FP64 on the tensor pipe (DMMA m8n8k4).  lda, ldb even; A, B 16-byte aligned.
// splits > 0: batch sum instead -- C[z] = alpha sum over the z-th of `splits`
// contiguous batch ranges of A[b]' B[b] (C[z] at C + z sc; fixed order).
// lower: C tiles entirely above the diagonal (all i < j) are skipped (m == n)
struct GemmTN {
  int m, n, kd, batch, splits;
  double alpha;
  int lower;
  const double* A;
  long long lda, sa;
  const double* B;
  long long ldb, sb;
  double* C;
  long long ldc, sc;
};
void launch_gemm_tn(const GemmTN& g, cudaStream_t st);

// row-major batched C[b] = alpha A[b] B[b] + beta C[b]: A m x kd (lda), B kd x n
// (ldb), C m x n (ldc), batch strides sa, sb, sc; any alignment (FP64 DMMA)
struct GemmNN {
  int m, n, kd, batch;
  double alpha, beta;
  const double* A;
  long long lda, sa;
  const double* B;
  long long ldb, sb;
  double* C;
  long long ldc, sc;
};
void launch_gemm_nn(const GemmNN& g, cudaStream_t st);

}  // namespace bipm
