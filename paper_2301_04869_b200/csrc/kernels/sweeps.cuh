// CTA-wide level-scheduled sparse triangular sweeps over a panel of k
// right-hand sides (row-major X[row * ldx + c], rows in the permuted order).
//
// Every level's (row, column) items are independent.  A level with few items
// gets g > 1 lanes per item (power of two, inside one warp); the lanes split
// the row's dot product and combine it with xor shuffles, so narrow levels at
// the top of the elimination tree do not serialise on one thread.
#pragma once

#include "device_plan.cuh"

namespace bipm {

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

// X <- L^{-1} X  (unit lower, forward levels)
template <int BLOCK>
__device__ void sweep_L(const DevLu& P, const double* __restrict__ F, double* X, int k, int ldx) {
  for (int lv = 0; lv < P.n_fwd; ++lv) {
    const int r0 = P.fwd_ptr[lv];
    const int items = (P.fwd_ptr[lv + 1] - r0) * k;
    group_dot<BLOCK>(
        items,
        [&](int it, int& b, int& e) {
          const int row = P.fwd_rows[r0 + it / k];
          b = P.l_ptr[row];
          e = P.l_ptr[row + 1];
        },
        [&](int it, int t) { return F[t] * X[P.l_col[t] * ldx + it % k]; },
        [&](int it, double acc) {
          const int row = P.fwd_rows[r0 + it / k];
          X[row * ldx + it % k] -= acc;
        });
    __syncthreads();
  }
}

// X <- U^{-1} X  (upper with diagonal, backward levels)
template <int BLOCK>
__device__ void sweep_U(const DevLu& P, const double* __restrict__ F, double* X, int k, int ldx) {
  for (int lv = 0; lv < P.n_bwd; ++lv) {
    const int r0 = P.bwd_ptr[lv];
    const int items = (P.bwd_ptr[lv + 1] - r0) * k;
    group_dot<BLOCK>(
        items,
        [&](int it, int& b, int& e) {
          const int row = P.bwd_rows[r0 + it / k];
          b = P.u_ptr[row];
          e = P.u_ptr[row + 1];
        },
        [&](int it, int t) { return F[P.u_slot[t]] * X[P.u_col[t] * ldx + it % k]; },
        [&](int it, double acc) {
          const int row = P.bwd_rows[r0 + it / k];
          double* x = X + row * ldx + it % k;
          *x = (*x - acc) / F[P.diag[row]];
        });
    __syncthreads();
  }
}

// X <- U^{-T} X  (lower sweep over the columns of U, forward levels)
template <int BLOCK>
__device__ void sweep_Ut(const DevLu& P, const double* __restrict__ F, double* X, int k, int ldx) {
  for (int lv = 0; lv < P.n_fwd; ++lv) {
    const int r0 = P.fwd_ptr[lv];
    const int items = (P.fwd_ptr[lv + 1] - r0) * k;
    group_dot<BLOCK>(
        items,
        [&](int it, int& b, int& e) {
          const int row = P.fwd_rows[r0 + it / k];
          b = P.ut_ptr[row];
          e = P.ut_ptr[row + 1];
        },
        [&](int it, int t) { return F[P.ut_slot[t]] * X[P.ut_row[t] * ldx + it % k]; },
        [&](int it, double acc) {
          const int row = P.fwd_rows[r0 + it / k];
          double* x = X + row * ldx + it % k;
          *x = (*x - acc) / F[P.diag[row]];
        });
    __syncthreads();
  }
}

// X <- L^{-T} X  (unit upper sweep over the columns of L, backward levels)
template <int BLOCK>
__device__ void sweep_Lt(const DevLu& P, const double* __restrict__ F, double* X, int k, int ldx) {
  for (int lv = 0; lv < P.n_bwd; ++lv) {
    const int r0 = P.bwd_ptr[lv];
    const int items = (P.bwd_ptr[lv + 1] - r0) * k;
    group_dot<BLOCK>(
        items,
        [&](int it, int& b, int& e) {
          const int row = P.bwd_rows[r0 + it / k];
          b = P.lt_ptr[row];
          e = P.lt_ptr[row + 1];
        },
        [&](int it, int t) { return F[P.lt_slot[t]] * X[P.lt_row[t] * ldx + it % k]; },
        [&](int it, double acc) {
          const int row = P.bwd_rows[r0 + it / k];
          X[row * ldx + it % k] -= acc;
        });
    __syncthreads();
  }
}

}  // namespace bipm
