// CTA-wide sparse triangular sweeps over a panel of k right-hand sides
// (row-major X[row * ldx + c], rows in the permuted order).
//
// Level-scheduled part: each level's (row, column) items are independent.
// A level with few items gets g > 1 lanes per item (power of two, inside one
// warp) that split the row's dot product and combine it with xor shuffles.
// Item metadata is one packed int4 (row, begin, end) and values are read
// directly at the entry position (F for L/U, the transposed copy FT for
// U'/L'), so a level costs one metadata load plus the entry stream.
//
// Dense tail: the trailing separator block [t0, n) of the elimination order is
// a long chain of one-row levels; it is solved as a dense triangle with the
// panel column held in registers of one warp (row i on lane i % 32, register
// i / 32) and the pivot value broadcast by shuffle, one step per row.
#pragma once

#include "device_plan.cuh"

namespace bipm {

// Per-scenario factor arrays: F = [L rows | U rows], FT = [U' rows | L' rows],
// D = four column-major tl x tl dense tail blocks (L_TT, L_TT', U_TT, U_TT').
struct FactorView {
  const double* F;
  const double* FT;
  const double* D;
};

template <int BLOCK, typename Range, typename Term, typename Finish>
__device__ __forceinline__ void group_dot(int items, Range range, Term term, Finish finish) {
  constexpr int kWarps = BLOCK / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int g = 1;
  while (g < 32 && items * (g * 2) <= BLOCK) g *= 2;
  const int per_warp = 32 / g;
  const int sub = lane & (g - 1);
  const int gid = lane / g;
  for (int base = warp * per_warp; base < items; base += kWarps * per_warp) {
    const int item = base + gid;
    double a0 = 0.0, a1 = 0.0;
    if (item < items) {
      int b, e;
      range(item, b, e);
      int t = b + sub;
      for (; t + g < e; t += 2 * g) {
        a0 += term(item, t);
        a1 += term(item, t + g);
      }
      if (t < e) a0 += term(item, t);
    }
    double acc = a0 + a1;
    for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (item < items && sub == 0) finish(item, acc);
  }
}

// One level-scheduled sweep.  kDiag: the first entry of each row is the
// diagonal (divide by it); the remaining entries are the off-diagonals.
template <int BLOCK, bool kDiag>
__device__ void level_sweep(const DevSweep& S, const double* __restrict__ V, double* X, int k,
                            int ldx) {
  const int4* items = reinterpret_cast<const int4*>(S.items);
  for (int lv = 0; lv < S.n_lvl; ++lv) {
    const int i0 = S.lvl_ptr[lv];
    const int n = (S.lvl_ptr[lv + 1] - i0) * k;
    group_dot<BLOCK>(
        n,
        [&](int it, int& b, int& e) {
          const int4 m = items[i0 + it / k];
          b = m.y + (kDiag ? 1 : 0);
          e = m.z;
        },
        [&](int it, int t) { return V[t] * X[S.col[t] * ldx + it % k]; },
        [&](int it, double acc) {
          const int4 m = items[i0 + it / k];
          double* x = X + m.x * ldx + it % k;
          if (kDiag)
            *x = (*x - acc) / V[m.y];
          else
            *x -= acc;
        });
    __syncthreads();
  }
}

// Forward sweeps: subtract the non-tail part of every tail row (one level).
template <int BLOCK, bool kDiag>
__device__ void tail_gather(const DevSweep& S, const double* __restrict__ V, double* X, int k,
                            int ldx) {
  if (S.n_tail == 0) return;
  const int4* items = reinterpret_cast<const int4*>(S.tail_items);
  group_dot<BLOCK>(
      S.n_tail * k,
      [&](int it, int& b, int& e) {
        const int4 m = items[it / k];
        b = m.y + (kDiag ? 1 : 0);
        e = m.z;
      },
      [&](int it, int t) { return V[t] * X[S.col[t] * ldx + it % k]; },
      [&](int it, double acc) { X[items[it / k].x * ldx + it % k] -= acc; });
  __syncthreads();
}

// Dense triangular solve of the tail block for every panel column: one warp
// per column, the column in registers.  D is the column-major tl x tl matrix
// of the triangle being solved (lower when kForward, upper otherwise).
template <int NQ, bool kUnit, bool kForward>
__device__ void dense_tail_nq(const double* __restrict__ D, double* X, int t0, int tl, int k,
                              int ldx, int nwarps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < k; c += nwarps) {
    double xr[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = q * 32 + lane;
      xr[q] = i < tl ? X[(t0 + i) * ldx + c] : 0.0;
    }
    if (kForward) {
#pragma unroll
      for (int qj = 0; qj < NQ; ++qj) {
        if (qj * 32 >= tl) break;
#pragma unroll 4
        for (int jj = 0; jj < 32; ++jj) {
          const int j = qj * 32 + jj;
          if (j >= tl) break;
          const double* col = D + size_t(j) * tl;
          double cv[NQ];
#pragma unroll
          for (int q = qj; q < NQ; ++q) {
            const int i = q * 32 + lane;
            cv[q] = (i > j && i < tl) ? col[i] : 0.0;
          }
          if (!kUnit && lane == jj) xr[qj] /= col[j];
          const double xj = __shfl_sync(0xffffffffu, xr[qj], jj);
#pragma unroll
          for (int q = qj; q < NQ; ++q) xr[q] -= cv[q] * xj;
        }
      }
    } else {
#pragma unroll
      for (int qj = NQ - 1; qj >= 0; --qj) {
        if (qj * 32 >= tl) continue;
#pragma unroll 4
        for (int jj = 31; jj >= 0; --jj) {
          const int j = qj * 32 + jj;
          if (j >= tl) continue;
          const double* col = D + size_t(j) * tl;
          double cv[NQ];
#pragma unroll
          for (int q = 0; q <= qj; ++q) {
            const int i = q * 32 + lane;
            cv[q] = i < j ? col[i] : 0.0;
          }
          if (!kUnit && lane == jj) xr[qj] /= col[j];
          const double xj = __shfl_sync(0xffffffffu, xr[qj], jj);
#pragma unroll
          for (int q = 0; q <= qj; ++q) xr[q] -= cv[q] * xj;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = q * 32 + lane;
      if (i < tl) X[(t0 + i) * ldx + c] = xr[q];
    }
  }
}

template <int BLOCK, bool kUnit, bool kForward>
__device__ void dense_tail(const DevLu& P, const double* D, double* X, int k, int ldx) {
  if (P.tl == 0) return;
  constexpr int kWarps = BLOCK / 32;
  if (P.tl <= 64)
    dense_tail_nq<2, kUnit, kForward>(D, X, P.t0, P.tl, k, ldx, kWarps);
  else if (P.tl <= 128)
    dense_tail_nq<4, kUnit, kForward>(D, X, P.t0, P.tl, k, ldx, kWarps);
  else
    dense_tail_nq<8, kUnit, kForward>(D, X, P.t0, P.tl, k, ldx, kWarps);
  __syncthreads();
}

__device__ __forceinline__ const double* dense_block(const DevLu& P, const FactorView& f, int b) {
  return f.D + size_t(b) * P.tl * P.tl;
}

// X <- L^{-1} X
template <int BLOCK>
__device__ void sweep_L(const DevLu& P, const FactorView& f, double* X, int k, int ldx) {
  level_sweep<BLOCK, false>(P.sL, f.F, X, k, ldx);
  tail_gather<BLOCK, false>(P.sL, f.F, X, k, ldx);
  dense_tail<BLOCK, true, true>(P, dense_block(P, f, 0), X, k, ldx);
}

// X <- U^{-1} X
template <int BLOCK>
__device__ void sweep_U(const DevLu& P, const FactorView& f, double* X, int k, int ldx) {
  dense_tail<BLOCK, false, false>(P, dense_block(P, f, 2), X, k, ldx);
  level_sweep<BLOCK, true>(P.sU, f.F + P.nnz_l, X, k, ldx);
}

// X <- U^{-T} X
template <int BLOCK>
__device__ void sweep_Ut(const DevLu& P, const FactorView& f, double* X, int k, int ldx) {
  level_sweep<BLOCK, true>(P.sUt, f.FT, X, k, ldx);
  tail_gather<BLOCK, true>(P.sUt, f.FT, X, k, ldx);
  dense_tail<BLOCK, false, true>(P, dense_block(P, f, 3), X, k, ldx);
}

// X <- L^{-T} X
template <int BLOCK>
__device__ void sweep_Lt(const DevLu& P, const FactorView& f, double* X, int k, int ldx) {
  dense_tail<BLOCK, true, false>(P, dense_block(P, f, 1), X, k, ldx);
  level_sweep<BLOCK, false>(P.sLt, f.FT + (P.nnz_f - P.nnz_l), X, k, ldx);
}

}  // namespace bipm
