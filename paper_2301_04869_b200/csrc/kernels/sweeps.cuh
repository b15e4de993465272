// CTA-wide sparse triangular sweeps over a panel of K right-hand sides
// (row-major X[row * K + c], rows in the permuted order, K compile-time).
//
// Level-scheduled part: each level's (row, column) items are independent.
// A level with few items gets g > 1 lanes per item (power of two, inside one
// warp) that split the row's dot product and combine it with xor shuffles.
// Item metadata is one packed int4 (row, begin, end) and values are read
// directly at the entry position (F for L/U, the transposed copy FT for
// U'/L'), so a level costs one metadata load plus the entry stream; the
// per-item index arithmetic is hoisted out of the entry loop.
//
// Dense tail: the trailing separator block [t0, n) of the elimination order is
// a long chain of one-row levels; it is solved as a dense triangle with the
// panel column held in registers of one warp (row i on lane i % 32, register
// i / 32), the pivot value broadcast by shuffle and the next column of the
// dense block prefetched one step ahead.  The L and U tails (and the U' and
// L' tails) are adjacent in the solve order and run back to back without
// leaving registers.
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

// Generic level step: for every item, acc = sum of term(item, t) over the
// item's entry range, g lanes per item; finish(item, acc) on the group lead.
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
    double acc = 0.0;
    if (item < items) {
      int b, e;
      range(item, b, e);
      for (int t = b + sub; t < e; t += g) acc += term(item, t);
    }
    for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (item < items && sub == 0) finish(item, acc);
  }
}

// One level-scheduled sweep.  kDiag: the first entry of each row is its
// diagonal (divide by it); the remaining entries are the off-diagonals.
// kTail: process the forward sweep's tail gather (entries with col < t0 of
// every tail row) as one extra level.
template <int BLOCK, int K, bool kDiag>
__device__ __forceinline__ void level_items(const int4* __restrict__ items, int nrows,
                                            const int* __restrict__ col,
                                            const double* __restrict__ V, double* X,
                                            bool subtract_only) {
  constexpr int kWarps = BLOCK / 32;
  const int n = nrows * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int g = 1;
  while (g < 32 && n * (g * 2) <= BLOCK) g *= 2;
  const int per_warp = 32 / g;
  const int sub = lane & (g - 1);
  const int gid = lane / g;
  for (int base = warp * per_warp; base < n; base += kWarps * per_warp) {
    const int item = base + gid;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int4 m = make_int4(0, 0, 0, 0);
    const int c = item % K;
    if (item < n) {
      m = items[item / K];
      const double* __restrict__ xc = X + c;
      const int b = m.y + (kDiag ? 1 : 0);
      int t = b + sub;
      for (; t + 3 * g < m.z; t += 4 * g) {  // four independent entries in flight
        const int c0 = col[t], c1 = col[t + g], c2 = col[t + 2 * g], c3 = col[t + 3 * g];
        const double v0 = V[t], v1 = V[t + g], v2 = V[t + 2 * g], v3 = V[t + 3 * g];
        a0 += v0 * xc[c0 * K];
        a1 += v1 * xc[c1 * K];
        a2 += v2 * xc[c2 * K];
        a3 += v3 * xc[c3 * K];
      }
      for (; t < m.z; t += g) a0 += V[t] * xc[col[t] * K];
    }
    double acc = (a0 + a1) + (a2 + a3);
    for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (item < n && sub == 0) {
      double* x = X + m.x * K + c;
      if (kDiag && !subtract_only)
        *x = (*x - acc) / V[m.y];
      else
        *x -= acc;
    }
  }
}

template <int BLOCK, int K, bool kDiag>
__device__ void level_sweep(const DevSweep& S, const double* __restrict__ V, double* X) {
  const int4* items = reinterpret_cast<const int4*>(S.items);
  for (int lv = 0; lv < S.n_lvl; ++lv) {
    const int i0 = S.lvl_ptr[lv];
    level_items<BLOCK, K, kDiag>(items + i0, S.lvl_ptr[lv + 1] - i0, S.col, V, X, false);
    __syncthreads();
  }
}

// Forward sweeps: subtract the non-tail part of every tail row (one level).
template <int BLOCK, int K, bool kDiag>
__device__ void tail_gather(const DevSweep& S, const double* __restrict__ V, double* X) {
  if (S.n_tail == 0) return;
  level_items<BLOCK, K, kDiag>(reinterpret_cast<const int4*>(S.tail_items), S.n_tail, S.col, V,
                               X, true);
  __syncthreads();
}

// Dense triangular solves of the tail block in registers of one warp.
// D is the column-major tl x tl matrix; lower/forward or upper/backward.
// Columns stream through a 4-deep register ring (prefetch distance 4).
template <int NQ>
__device__ __forceinline__ void load_col(const double* __restrict__ D, int tl, int j,
                                         double (&v)[NQ]) {
  const int lane = threadIdx.x & 31;
  const bool ok = j >= 0 && j < tl;
  const double* __restrict__ col = D + size_t(ok ? j : 0) * tl;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = q * 32 + lane;
    v[q] = (ok && i < tl) ? col[i] : 0.0;
  }
}

template <int NQ, bool kUnit>
__device__ __forceinline__ void dense_forward(const double* __restrict__ D, int tl, double (&xr)[NQ]) {
  constexpr int R = NQ <= 4 ? 4 : 2;  // ring depth (register budget)
  const int lane = threadIdx.x & 31;
  double ring[R][NQ];
#pragma unroll
  for (int u = 0; u < R; ++u) load_col<NQ>(D, tl, u, ring[u]);
#pragma unroll
  for (int qj = 0; qj < NQ; ++qj) {
    if (qj * 32 >= tl) break;
    // not unrolled: the ring is loop-carried, so each column load is issued
    // R steps before its use instead of being sunk next to it
#pragma unroll 1
    for (int jb = 0; jb < 32; jb += R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int jj = jb + u, j = qj * 32 + jj;
        if (j < tl) {
          if (!kUnit && lane == jj) xr[qj] /= ring[u][qj];
          const double xj = __shfl_sync(0xffffffffu, xr[qj], jj);
#pragma unroll
          for (int q = qj; q < NQ; ++q)
            if (q * 32 + lane > j) xr[q] -= ring[u][q] * xj;
        }
        load_col<NQ>(D, tl, j + R, ring[u]);
      }
    }
  }
}

template <int NQ, bool kUnit>
__device__ __forceinline__ void dense_backward(const double* __restrict__ D, int tl, double (&xr)[NQ]) {
  constexpr int R = NQ <= 4 ? 4 : 2;
  const int lane = threadIdx.x & 31;
  // walk j = NQ*32-1 down to 0; columns >= tl are skipped
  double ring[R][NQ];
  const int top = NQ * 32 - 1;
#pragma unroll
  for (int u = 0; u < R; ++u) load_col<NQ>(D, tl, top - u, ring[u]);
#pragma unroll
  for (int qj = NQ - 1; qj >= 0; --qj) {
#pragma unroll 1
    for (int jb = 31; jb >= 0; jb -= R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int jj = jb - u, j = qj * 32 + jj;
        if (j < tl) {
          if (!kUnit && lane == jj) xr[qj] /= ring[u][qj];
          const double xj = __shfl_sync(0xffffffffu, xr[qj], jj);
#pragma unroll
          for (int q = 0; q <= qj; ++q)
            if (q * 32 + lane < j) xr[q] -= ring[u][q] * xj;
        }
        load_col<NQ>(D, tl, j - R, ring[u]);
      }
    }
  }
}

// Tail pair on every panel column: forward triangle D1 (unit when kUnit1),
// then backward triangle D2 (unit when kUnit2).  D1 or D2 may be null.
template <int NQ, bool kUnit1, bool kUnit2>
__device__ void dense_tail_pair_nq(const double* D1, const double* D2, double* X, int t0, int tl,
                                   int K, int nwarps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < K; c += nwarps) {
    double xr[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = q * 32 + lane;
      xr[q] = i < tl ? X[(t0 + i) * K + c] : 0.0;
    }
    if (D1) dense_forward<NQ, kUnit1>(D1, tl, xr);
    if (D2) dense_backward<NQ, kUnit2>(D2, tl, xr);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = q * 32 + lane;
      if (i < tl) X[(t0 + i) * K + c] = xr[q];
    }
  }
}

template <int BLOCK, int K, bool kUnit1, bool kUnit2>
__device__ void dense_tail_pair(const DevLu& P, const double* D1, const double* D2, double* X) {
  if (P.tl == 0) return;
  constexpr int kWarps = BLOCK / 32;
  if (P.tl <= 64)
    dense_tail_pair_nq<2, kUnit1, kUnit2>(D1, D2, X, P.t0, P.tl, K, kWarps);
  else if (P.tl <= 128)
    dense_tail_pair_nq<4, kUnit1, kUnit2>(D1, D2, X, P.t0, P.tl, K, kWarps);
  else
    dense_tail_pair_nq<8, kUnit1, kUnit2>(D1, D2, X, P.t0, P.tl, K, kWarps);
  __syncthreads();
}

__device__ __forceinline__ const double* dense_block(const DevLu& P, const FactorView& f, int b) {
  return f.D + size_t(b) * P.tl * P.tl;
}

// X <- U^{-1} L^{-1} X  (G_x solve in the permuted basis)
template <int BLOCK, int K>
__device__ void solve_LU(const DevLu& P, const FactorView& f, double* X) {
  level_sweep<BLOCK, K, false>(P.sL, f.F, X);
  tail_gather<BLOCK, K, false>(P.sL, f.F, X);
  dense_tail_pair<BLOCK, K, true, false>(P, dense_block(P, f, 0), dense_block(P, f, 2), X);
  level_sweep<BLOCK, K, true>(P.sU, f.F + P.nnz_l, X);
}

// X <- L^{-T} U^{-T} X  (G_x' solve in the permuted basis)
template <int BLOCK, int K>
__device__ void solve_LUt(const DevLu& P, const FactorView& f, double* X) {
  level_sweep<BLOCK, K, true>(P.sUt, f.FT, X);
  tail_gather<BLOCK, K, true>(P.sUt, f.FT, X);
  dense_tail_pair<BLOCK, K, false, true>(P, dense_block(P, f, 3), dense_block(P, f, 1), X);
  level_sweep<BLOCK, K, false>(P.sLt, f.FT + (P.nnz_f - P.nnz_l), X);
}

}  // namespace bipm
