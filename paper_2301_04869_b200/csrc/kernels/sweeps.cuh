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
// a long chain of one-row levels.  Its L and U triangles (and the U', L'
// ones) are adjacent in the solve order, so the pair is one multiplication by
// W = (L_TT U_TT)^{-1} (W' for the transposed solve), formed once per
// refactor: 2 tl dependent steps become one parallel tl x tl x K product.
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
  int lg = 0;  // g = 2^lg lanes per item (shifts: g is not a compile-time constant)
  while (lg < 5 && items * (2 << lg) <= BLOCK) ++lg;
  const int g = 1 << lg;
  const int per_warp = 32 >> lg;
  const int sub = lane & (g - 1);
  const int gid = lane >> lg;
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
  int lg = 0;
  while (lg < 5 && n * (2 << lg) <= BLOCK) ++lg;
  const int g = 1 << lg;
  const int per_warp = 32 >> lg;
  const int sub = lane & (g - 1);
  const int gid = lane >> lg;
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

// Single right-hand side (one CTA per scenario: no other CTA hides the
// per-level memory round trips, items -> col / V -> X).  Everything but the
// X gathers is independent of the previous levels, so it is software
// pipelined: the item records of level l + 2 and the first two entries
// (columns, values, diagonal) of level l + 1 are loaded while level l runs.
// Same summation order as level_items (bitwise identical results).
#ifndef BIPM_SWEEP1_PF
#define BIPM_SWEEP1_PF 2  // prefetched entries per item (0: plain level_items sweeps)
#endif
template <int BLOCK, bool kDiag>
__device__ void level_sweep1(const DevSweep& S, const double* __restrict__ V, double* X) {
  constexpr int kWarps = BLOCK / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4* __restrict__ items = reinterpret_cast<const int4*>(S.items);
  const int* __restrict__ col = S.col;
  const int nl = S.n_lvl;
  struct Geo {
    int i0, n, lg;  // g = 2^lg lanes per item
  };
  // the level pointers in shared memory: the item records two levels ahead
  // are then one memory round trip away, not two
  constexpr int kLvlCap = 1024;
  __shared__ int s_lvl[kLvlCap + 1];
  const bool lvl_smem = nl <= kLvlCap;
  if (lvl_smem) {
    for (int i = threadIdx.x; i <= nl; i += BLOCK) s_lvl[i] = S.lvl_ptr[i];
    __syncthreads();
  }
  auto geo = [&](int lv) {
    Geo q{0, 0, 0};
    if (lv < nl) {
      q.i0 = lvl_smem ? s_lvl[lv] : __ldg(S.lvl_ptr + lv);
      q.n = (lvl_smem ? s_lvl[lv + 1] : __ldg(S.lvl_ptr + lv + 1)) - q.i0;
      while (q.lg < 5 && q.n * (2 << q.lg) <= BLOCK) ++q.lg;
    }
    return q;
  };
  // this thread's first item of a level (the first pass over its items)
  auto first_item = [&](const Geo& q) { return ((warp << 5) + lane) >> q.lg; };
  auto load_meta = [&](const Geo& q) {
    const int item = first_item(q);
    return item < q.n ? items[q.i0 + item] : make_int4(0, 0, 0, 0);
  };
  constexpr int kPf = BIPM_SWEEP1_PF > 0 ? BIPM_SWEEP1_PF : 1;
  struct Ent {
    int c[kPf];
    double v[kPf], d;
  };
  auto load_ent = [&](const Geo& q, const int4& m) {
    Ent e;
    const int g = 1 << q.lg;
    const int t = m.y + (kDiag ? 1 : 0) + (lane & (g - 1));
#pragma unroll
    for (int k = 0; k < kPf; ++k) {
      const bool ok = t + k * g < m.z;
      e.c[k] = ok ? col[t + k * g] : 0;
      e.v[k] = ok ? V[t + k * g] : 0.0;
    }
    e.d = kDiag && m.z > m.y ? V[m.y] : 1.0;
    return e;
  };
  Geo g_cur = geo(0), g_nxt = geo(1);
  int4 m_cur = load_meta(g_cur), m_nxt = load_meta(g_nxt);
  Ent e_cur = load_ent(g_cur, m_cur);
  for (int lv = 0; lv < nl; ++lv) {
    const Geo g_nn = geo(lv + 2);
    const int4 m_nn = load_meta(g_nn);    // two levels ahead
    const Ent e_nxt = load_ent(g_nxt, m_nxt);  // one level ahead
    {
      const Geo& q = g_cur;
      const int g = 1 << q.lg, per_warp = 32 >> q.lg, sub = lane & (g - 1);
      // first pass: the prefetched item
      {
        const int item = first_item(q);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (item < q.n) {
          const int4 m = m_cur;
          int t = m.y + (kDiag ? 1 : 0) + sub;
          auto ev = [&](int k) { return k < kPf ? e_cur.v[k] : V[t + k * g]; };
          auto ec = [&](int k) { return k < kPf ? e_cur.c[k] : col[t + k * g]; };
          if (t + 3 * g < m.z) {
            a0 += ev(0) * X[ec(0)];
            a1 += ev(1) * X[ec(1)];
            a2 += ev(2) * X[ec(2)];
            a3 += ev(3) * X[ec(3)];
            t += 4 * g;
            for (; t + 3 * g < m.z; t += 4 * g) {
              const int c0 = col[t], c1 = col[t + g], c2 = col[t + 2 * g], c3 = col[t + 3 * g];
              const double v0 = V[t], v1 = V[t + g], v2 = V[t + 2 * g], v3 = V[t + 3 * g];
              a0 += v0 * X[c0];
              a1 += v1 * X[c1];
              a2 += v2 * X[c2];
              a3 += v3 * X[c3];
            }
            for (; t < m.z; t += g) a0 += V[t] * X[col[t]];
          } else {
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (t + k * g < m.z) a0 += ev(k) * X[ec(k)];
          }
        }
        double acc = (a0 + a1) + (a2 + a3);
        for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (item < q.n && sub == 0) {
          double* x = X + m_cur.x;
          if (kDiag)
            *x = (*x - acc) / e_cur.d;
          else
            *x -= acc;
        }
      }
      // further passes (levels with more items than threads): as level_items
      if (q.n > kWarps * per_warp) {
        const int4* it = items + q.i0;
        const int gid = lane >> q.lg;
        for (int base = (warp + kWarps) * per_warp; base < q.n; base += kWarps * per_warp) {
          const int item = base + gid;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int4 m = make_int4(0, 0, 0, 0);
          if (item < q.n) {
            m = it[item];
            int t = m.y + (kDiag ? 1 : 0) + sub;
            for (; t + 3 * g < m.z; t += 4 * g) {
              const int c0 = col[t], c1 = col[t + g], c2 = col[t + 2 * g], c3 = col[t + 3 * g];
              const double v0 = V[t], v1 = V[t + g], v2 = V[t + 2 * g], v3 = V[t + 3 * g];
              a0 += v0 * X[c0];
              a1 += v1 * X[c1];
              a2 += v2 * X[c2];
              a3 += v3 * X[c3];
            }
            for (; t < m.z; t += g) a0 += V[t] * X[col[t]];
          }
          double acc = (a0 + a1) + (a2 + a3);
          for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          if (item < q.n && sub == 0) {
            double* x = X + m.x;
            if (kDiag)
              *x = (*x - acc) / V[m.y];
            else
              *x -= acc;
          }
        }
      }
    }
    __syncthreads();
    g_cur = g_nxt;
    m_cur = m_nxt;
    e_cur = e_nxt;
    g_nxt = g_nn;
    m_nxt = m_nn;
  }
}

template <int BLOCK, int K, bool kDiag>
__device__ void level_sweep(const DevSweep& S, const double* __restrict__ V, double* X) {
  if constexpr (K == 1 && BIPM_SWEEP1_PF > 0) {
    level_sweep1<BLOCK, kDiag>(S, V, X);
    return;
  }
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

// Dense tail: X_T <- W X_T for every panel column, W = (L_TT U_TT)^{-1} (or
// its transpose) precomputed by the refactor, row-major tl x tl.  Up to 8
// outputs per thread are formed in registers before any is written back.
template <int BLOCK, int K>
__device__ void dense_tail_gemm(const DevLu& P, const double* __restrict__ W, double* X) {
  const int tl = P.tl, t0 = P.t0;
  if (tl == 0) return;
  if constexpr (K == 1) {
    // single right-hand side: a warp per output row, lanes split the row of W
    // (coalesced), four rows' loads in flight per warp, shuffle reduction;
    // result j of a warp (row warp*4 + (j/4)*stride + j%4) is kept by lane j%32
    constexpr int kWarps = BLOCK / 32, kRows = 4, kStride = kWarps * kRows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double res0 = 0.0, res1 = 0.0;
    int j = 0;
    for (int i0 = warp * kRows; i0 < tl; i0 += kStride) {
      double acc[kRows];
#pragma unroll
      for (int q = 0; q < kRows; ++q) acc[q] = 0.0;
      for (int k = lane; k < tl; k += 32) {
        const double xk = X[t0 + k];
#pragma unroll
        for (int q = 0; q < kRows; ++q)
          if (i0 + q < tl) acc[q] += __ldg(W + size_t(i0 + q) * tl + k) * xk;
      }
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
        if (lane == ((j + q) & 31)) {
          if ((j + q) >> 5)
            res1 = acc[q];
          else
            res0 = acc[q];
        }
      }
      j += kRows;
    }
    __syncthreads();
    for (int slot = 0; slot < 2; ++slot) {
      const int jj = slot * 32 + lane;
      const int row = warp * kRows + (jj / kRows) * kStride + (jj % kRows);
      if (jj < j && row < tl) X[t0 + row] = slot ? res1 : res0;
    }
    __syncthreads();
    return;
  }
  constexpr int kMaxOut = 8;
  const int n = tl * K;
  double r[kMaxOut];
#pragma unroll
  for (int q = 0; q < kMaxOut; ++q) {
    const int o = threadIdx.x + q * BLOCK;
    r[q] = 0.0;
    if (o < n) {
      const int i = o / K, c = o % K;
      const double* __restrict__ w = W + size_t(i) * tl;
      const double* __restrict__ xc = X + t0 * K + c;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int k = 0;
      for (; k + 3 < tl; k += 4) {
        a0 += w[k] * xc[k * K];
        a1 += w[k + 1] * xc[(k + 1) * K];
        a2 += w[k + 2] * xc[(k + 2) * K];
        a3 += w[k + 3] * xc[(k + 3) * K];
      }
      for (; k < tl; ++k) a0 += w[k] * xc[k * K];
      r[q] = (a0 + a1) + (a2 + a3);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kMaxOut; ++q) {
    const int o = threadIdx.x + q * BLOCK;
    if (o < n) X[(t0 + o / K) * K + o % K] = r[q];
  }
  __syncthreads();
}

// D = [W row-major | W' row-major], W = (L_TT U_TT)^{-1}
__device__ __forceinline__ const double* dense_block(const DevLu& P, const FactorView& f, int b) {
  return f.D + size_t(b) * P.tl * P.tl;
}

// X <- U^{-1} L^{-1} X  (G_x solve in the permuted basis)
template <int BLOCK, int K>
__device__ void solve_LU(const DevLu& P, const FactorView& f, double* X) {
  level_sweep<BLOCK, K, false>(P.sL, f.F, X);
  tail_gather<BLOCK, K, false>(P.sL, f.F, X);
  dense_tail_gemm<BLOCK, K>(P, dense_block(P, f, 0), X);
  level_sweep<BLOCK, K, true>(P.sU, f.F + P.nnz_l, X);
}

// X <- L^{-T} U^{-T} X  (G_x' solve in the permuted basis)
template <int BLOCK, int K>
__device__ void solve_LUt(const DevLu& P, const FactorView& f, double* X) {
  level_sweep<BLOCK, K, true>(P.sUt, f.FT, X);
  tail_gather<BLOCK, K, true>(P.sUt, f.FT, X);
  dense_tail_gemm<BLOCK, K>(P, dense_block(P, f, 1), X);
  level_sweep<BLOCK, K, false>(P.sLt, f.FT + (P.nnz_f - P.nnz_l), X);
}

}  // namespace bipm
