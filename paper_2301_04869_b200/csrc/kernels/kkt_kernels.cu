// Reduced-space KKT kernels for sm_100a: batched static-pivot LU refactor of
// G_x, the multi-RHS Schur reduction K_hat = sum_i Z_i' K_i Z_i, the reduced
// right-hand side, state/adjoint and slack/dual recovery, condensation and the
// dense Cholesky of K_hat.
//
// Reference operators replaced (proj/core/src):
//   launch_lu_refactor     BlockDiagFactor::factor     linalg.cpp:51-89
//   launch_reduce_tiles    reduce_group (tile loop)    kkt.cpp:371-466
//   launch_sum_parts       finish_reduce/all_reduce    kkt.cpp:468-488, executor.cpp:39-61
//   launch_reduce_rhs      reduce_rhs_group            kkt.cpp:209-239
//   launch_recover_state   recover_state_adjoint       kkt.cpp:507-532
//   launch_recover_slack   recover_slack_dual          kkt.cpp:172-188
//   launch_condense        condense / run_condense     kkt.cpp:123-170, sparse.cpp:208-214
//   launch_shift_cholesky  solve_reduced shift+factor  kkt.cpp:965-971, linalg.cpp:129-145
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <stdexcept>

#include "kkt_kernels.hpp"
#include "reach_gemm.hpp"
#include "sweeps.cuh"

#include "stats.hpp"

namespace cg = cooperative_groups;

namespace bipm {

namespace {

constexpr int kSolveBlock = 512;   // single right-hand side kernels (1024 when few scenarios)
constexpr int kReduceBlock = 512;  // multi-RHS reduction: one CTA per SM, 128-register budget
constexpr int kLuBlock = 256;
constexpr int kDenseBlock = 1024;

template <int BLOCK>
__device__ double block_reduce(double v, bool is_max) {
  __shared__ double red[BLOCK / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, off);
    v = is_max ? fmax(v, o) : v + o;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < BLOCK / 32 ? red[lane] : (is_max ? 0.0 : 0.0);
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v, off);
      v = is_max ? fmax(v, o) : v + o;
    }
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// slot of column c in CSR row `row`, or -1
__device__ __forceinline__ int find_in_row(const int* ptr, const int* ind, int row, int c) {
  int lo = ptr[row], hi = ptr[row + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int v = ind[mid];
    if (v == c) return mid;
    if (v < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  return -1;
}

// ---------------------------------------------------------------- LU refactor
// Two kernels (BlockDiagFactor::factor, linalg.cpp:51-89, with one static
// symbolic pattern):
//  refactor_levels_kernel  the level-scheduled Crout program of the pivots
//    j < t0 (no shared memory, so several scenarios share an SM and hide each
//    other's memory latency), then for every factor slot of the dense tail
//    block its partial sum A - sum_{k < t0} L(i,k) U(k,j);
//  refactor_tail_kernel    right-looking dense LU of that tail block in shared
//    memory (static pivots), W = (L_TT U_TT)^{-1}, the pivot guard and the
//    sweep layouts (FT, VS) of the solve kernels.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) refactor_levels_kernel(DevLu P,
                                                                const double* __restrict__ gx,
                                                                int nnz_gx, double* F,
                                                                double* scale_out) {
  const int s = blockIdx.x;
  const double* __restrict__ A = gx + size_t(s) * nnz_gx;
  double* Fs = F + size_t(s) * P.nnz_f;
  double mx = 0.0;
  for (int i = threadIdx.x; i < nnz_gx; i += BLOCK) mx = fmax(mx, fabs(A[i]));
  const double scale = block_reduce<BLOCK>(mx, true);
  if (threadIdx.x == 0) scale_out[s] = scale;
  constexpr int kWarps = BLOCK / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ph = 0; ph < P.rf_nphase; ++ph) {
    const int b0 = P.rf_phase_ptr[ph], items = P.rf_phase_ptr[ph + 1] - b0;
    int g = 1;
    while (g < 32 && items * (g * 2) <= BLOCK) g *= 2;
    const int per_warp = 32 / g, sub = lane & (g - 1), gid = lane / g;
    for (int base = warp * per_warp; base < items; base += kWarps * per_warp) {
      const int item = base + gid;
      double acc = 0.0;
      int4 r = make_int4(0, 0, 0, -1);
      if (item < items) {
        r = P.rf_rec[b0 + item];
        // four multiply pairs (and their eight factor values) in flight
        int t = r.y + sub;
        for (; t + 3 * g < r.z; t += 4 * g) {
          int2 pr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) pr[u] = P.rf_pair[t + u * g];
          double l[4], uu[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            l[u] = Fs[pr[u].x];
            uu[u] = Fs[pr[u].y];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) acc += l[u] * uu[u];
        }
        for (; t < r.z; t += g) {
          const int2 pr = P.rf_pair[t];
          acc += Fs[pr.x] * Fs[pr.y];
        }
      }
      for (int off = g >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (item < items && sub == 0) {
        double v = (r.w >= 0 ? A[r.w] : 0.0) - acc;
        const int piv = P.rf_piv[b0 + item];
        if (piv >= 0) v /= Fs[piv];
        Fs[r.x] = v;
      }
    }
    __syncthreads();
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) refactor_tail_kernel(DevLu P, double* F, double* FT,
                                                              double* D,
                                                              const double* __restrict__ scale_in,
                                                              int* status, double piv_tol,
                                                              const int* vs_src, int nnz_vs,
                                                              double* VS) {
  const int s = blockIdx.x;
  double* Fs = F + size_t(s) * P.nnz_f;
  const int tl = P.tl, tt = tl * tl;
  extern __shared__ double sm[];
  double* T = sm;       // tail block, column-major; L strict lower + U upper after the LU
  double* Wm = sm + tt;  // W column j solved by thread j
  if (tl > 0) {
    for (int q = threadIdx.x; q < tt; q += BLOCK) {
      const int a = q % tl, b = q / tl;
      const int src = a > b ? P.dense_src[q] : P.dense_src[tt + q];
      T[q] = src >= 0 ? Fs[src] : 0.0;
    }
    __syncthreads();
    // right-looking LU without pivoting (the static pivot order)
    for (int k = 0; k < tl - 1; ++k) {
      const double piv = T[k * tl + k];
      for (int i = k + 1 + threadIdx.x; i < tl; i += BLOCK) T[k * tl + i] /= piv;
      __syncthreads();
      const int m = tl - 1 - k;
      for (int q = threadIdx.x; q < m * m; q += BLOCK) {
        const int i = k + 1 + q % m, j = k + 1 + q / m;
        T[j * tl + i] -= T[k * tl + i] * T[j * tl + k];
      }
      __syncthreads();
    }
    // back into the factor (structural slots only)
    for (int q = threadIdx.x; q < tt; q += BLOCK) {
      const int a = q % tl, b = q / tl;
      const int src = a > b ? P.dense_src[q] : P.dense_src[tt + q];
      if (src >= 0) Fs[src] = T[q];
    }
  }
  __syncthreads();
  // pivot guard (linalg.cpp:69-73): every diagonal of U against max |G_x|;
  // growth guard: every factor entry against growth * max |G_x|
  double bad = 0.0, big = 0.0;
  const double floor_ = piv_tol * fmax(scale_in[s], 1e-300);
  for (int j = threadIdx.x; j < P.n; j += BLOCK) {
    const double d = Fs[P.diag[j]];
    if (!(fabs(d) >= floor_) || !isfinite(d)) bad = 1.0;
  }
  for (int q = threadIdx.x; q < P.nnz_f; q += BLOCK) big = fmax(big, fabs(Fs[q]));
  bad = block_reduce<BLOCK>(bad, true);
  big = block_reduce<BLOCK>(big, true);
  if (threadIdx.x == 0)
    status[s] = bad > 0.0 ? 1 : (big > P.growth * fmax(scale_in[s], 1e-300) ? 2 : 0);
  // solve layouts: transposed copy and the sweep-ordered copy
  double* FTs = FT + size_t(s) * P.nnz_f;
  for (int q = threadIdx.x; q < P.nnz_f; q += BLOCK) FTs[q] = Fs[P.ft_src[q]];
  if (VS) {
    double* VSs = VS + size_t(s) * nnz_vs;
    for (int q = threadIdx.x; q < nnz_vs; q += BLOCK) {
      const int src = vs_src[q];
      VSs[q] = src >= 0 ? Fs[src] : 0.0;
    }
  }
  if (tl == 0) return;
  // W = (L_TT U_TT)^{-1}: thread j solves L U w = e_j for column j
  for (int j = threadIdx.x; j < tl; j += BLOCK) {
    for (int i = 0; i < j; ++i) Wm[i * tl + j] = 0.0;
    Wm[j * tl + j] = 1.0;
    for (int i = j + 1; i < tl; ++i) {  // y = L^{-1} e_j
      double acc = 0.0;
      for (int k = j; k < i; ++k) acc += T[k * tl + i] * Wm[k * tl + j];
      Wm[i * tl + j] = -acc;
    }
    for (int i = tl - 1; i >= 0; --i) {  // w = U^{-1} y
      double acc = Wm[i * tl + j];
      for (int k = i + 1; k < tl; ++k) acc -= T[k * tl + i] * Wm[k * tl + j];
      Wm[i * tl + j] = acc / T[i * tl + i];
    }
  }
  __syncthreads();
  // D = [W row-major | W' row-major]
  double* W = D + size_t(s) * 2 * tt;
  for (int q = threadIdx.x; q < tt; q += BLOCK) {
    W[q] = Wm[q];
    W[tt + q] = Wm[(q % tl) * tl + q / tl];
  }
}

// Large tails (2 tl^2 doubles beyond shared memory): blocked Gauss-Jordan
__device__ __forceinline__ void gj_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// shared-memory strides of the Gauss-Jordan tail kernel (doubles): 16-wide
// blocks padded to 20 and tl-wide rows to 16k + 4 so the m8n8k4 fragment
// loads (8 rows x 4 columns / 4 rows x 8 columns) hit distinct banks
constexpr int kGjB = 16, kGjLdb = 20;
constexpr int kGjMaxTail = 512;  // host/plan.hpp kMaxTail must not exceed it
inline __host__ __device__ int gj_tp(int tl) { return (tl + 7) & ~7; }
inline __host__ __device__ int gj_ldr(int tl) { return ((gj_tp(tl) + 15) & ~15) + 4; }
inline size_t gj_smem_bytes(int tl) {
  return (size_t(gj_tp(tl)) * kGjLdb + size_t(2) * kGjB * gj_ldr(tl) + kGjB * kGjLdb) *
         sizeof(double);
}

// inversion of the tail block S = L_TT U_TT into D's W slot (row-major,
// global memory, L2-resident), static pivots, 16 pivots per pass so the block
// is streamed tl/16 times instead of tl times; W = S^{-1}.  A pass is one
// rank-16 update W <- W' - C' R2 on the FP64 tensor pipe (m8n8k4 DMMA) with
// the Gauss-Jordan bookkeeping folded into the operands: C' = W[:, P] with
// the pivot rows replaced by -e_p, R2 = A11^{-1} W[P, :] with the pivot
// columns replaced by A11^{-1}, and W' = W with the pivot rows and columns
// zeroed.  Passes ping-pong between D's two tt slots (the W' slot is scratch
// until the layouts kernel) and end in the W slot.  A thread-block cluster of
// CL CTAs may share one scenario (small M: the GPU would otherwise idle):
// every CTA forms the 16x16 pivot inverse redundantly and updates its share
// of the 8 x 64 output strips, one cluster barrier per pass.  The pivots of
// the elimination are U_TT's diagonal: they go to the factor's diagonal slots
// for the guard.  The tail block's L/U values are never read by the sweeps
// (the tail is applied through W), so F keeps S there.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) refactor_tail_gj_kernel(DevLu P, double* F, double* FT,
                                                                 double* D,
                                                                 const double* __restrict__ scale_in,
                                                                 int* status, double piv_tol,
                                                                 const int* vs_src, int nnz_vs,
                                                                 double* VS, int blk0, int blkn,
                                                                 int gather, int guard) {
  constexpr int kB = kGjB, kLb = kGjLdb;
  extern __shared__ double gj[];
  cg::cluster_group cluster = cg::this_cluster();
  const int ncl = int(cluster.num_blocks()), crank = int(cluster.block_rank());
  // a lone CTA needs no cluster barrier (and its fence)
  auto sync_all = [&] {
    if (ncl > 1)
      cluster.sync();
    else
      __syncthreads();
  };
  const int s = blockIdx.x / ncl;
  double* Fs = F + size_t(s) * P.nnz_f;
  // the diagonal block [blk0, blk0 + blkn) of the tail is inverted in place
  // (the whole tail: blk0 = 0, blkn = tl); rows keep the tail's stride tl
  const int tl = P.tl, tt = tl * tl, t0 = P.t0, n = blkn;
  const int tp = gj_tp(n), ldr = gj_ldr(n), ntp = tp / 8;
  double* Cb = gj;                          // [tp][kLb]  C' = W[:, P], pivot rows -e_p
  double* Rb = Cb + size_t(tp) * kLb;       // [kB][ldr]  W[P, :]
  double* R2 = Rb + size_t(kB) * ldr;       // [kB][ldr]  A11^{-1} W[P, :], pivot cols A11^{-1}
  double* Ai = R2 + size_t(kB) * ldr;       // [kB][kLb]  A11^{-1}
  double* const Wbase = D + size_t(s) * 2 * tt;  // slot b at Wbase + b tt
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gm = lane >> 2, gk = lane & 3;
  constexpr int kWarps = BLOCK / 32;
  constexpr int kJ = kGjMaxTail / 32;  // a row's columns over the lanes
  if (gather) {
    // S from the factor: every load of a row in flight at once
    double* W = Wbase;
    for (int i = crank * kWarps + warp; i < tl; i += kWarps * ncl) {
      int src[kJ];
#pragma unroll
      for (int q = 0; q < kJ; ++q) {
        const int j = lane + 32 * q;
        src[q] = j >= tl ? -1 : i > j ? P.dense_src[j * tl + i] : P.dense_src[tt + j * tl + i];
      }
      double v[kJ];
#pragma unroll
      for (int q = 0; q < kJ; ++q) v[q] = src[q] >= 0 ? Fs[src[q]] : 0.0;
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (lane + 32 * q < tl) W[i * tl + lane + 32 * q] = v[q];
    }
  }
  sync_all();
  double* const Wblk = Wbase + size_t(blk0) * tl + blk0;
  for (int k0 = 0, pass = 0; k0 < n; k0 += kB, ++pass) {
    // in place: every element's update reads only itself and the staged
    // C' / R2, so slot 0 serves every pass (the working set of the CTAs in
    // flight, 148 x tl^2 doubles, then stays in L2 instead of ping-ponging
    // two slots through HBM)
    const int bb = min(kB, n - k0);
    const double* W = Wblk;
    double* Wn = Wblk;
    {
      // C' and W[P, :]: all of a thread's loads in flight, then the stores
      constexpr int kQ = (kGjMaxTail * kB + BLOCK - 1) / BLOCK;
      double v[kQ];
#pragma unroll
      for (int u = 0; u < kQ; ++u) {
        const int q = threadIdx.x + u * BLOCK;
        const int i = q / kB, p = q % kB;
        v[u] = 0.0;
        if (i >= k0 && i < k0 + bb)
          v[u] = p == i - k0 ? -1.0 : 0.0;
        else if (i < n && p < bb)
          v[u] = W[size_t(i) * tl + k0 + p];
      }
#pragma unroll
      for (int u = 0; u < kQ; ++u) {
        const int q = threadIdx.x + u * BLOCK;
        if (q < tp * kB) Cb[(q / kB) * kLb + q % kB] = v[u];
      }
#pragma unroll
      for (int u = 0; u < kQ; ++u) {
        const int q = threadIdx.x + u * BLOCK;
        const int pr = q / tp, j = q % tp;
        v[u] = (pr < bb && j < n) ? W[size_t(k0 + pr) * tl + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kQ; ++u) {
        const int q = threadIdx.x + u * BLOCK;
        if (q < tp * kB) Rb[(q / tp) * ldr + q % tp] = v[u];
      }
    }
    __syncthreads();
    if (ncl > 1) cluster.sync();  // no CTA overwrites W before every CTA staged C', W[P, :]
    // A11^{-1} by Gauss-Jordan in one warp (lane = column), pivots to the factor
    if (warp == 0) {
      // padded with the identity beyond bb: a branch-free loop keeps the
      // shuffles warp-converged
      double col[kB];  // lane's column of the working matrix
#pragma unroll
      for (int r = 0; r < kB; ++r)
        col[r] = (lane < bb && r < bb) ? Rb[r * ldr + k0 + lane] : (r == lane ? 1.0 : 0.0);
      double inv[kB];  // lane's column of the identity being transformed
#pragma unroll
      for (int r = 0; r < kB; ++r) inv[r] = (r == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const double piv = __shfl_sync(0xffffffffu, col[k], k);
        if (crank == 0 && lane == 0 && k < bb) Fs[P.diag[t0 + blk0 + k0 + k]] = piv;
        const double rp = 1.0 / piv;
        col[k] *= rp;
        inv[k] *= rp;
#pragma unroll
        for (int r = 0; r < kB; ++r) {
          const double f = __shfl_sync(0xffffffffu, col[r], k);  // A(r, k)
          if (r != k) {
            col[r] -= f * col[k];
            inv[r] -= f * inv[k];
          }
        }
      }
      if (lane < kB)
#pragma unroll
        for (int r = 0; r < kB; ++r) Ai[r * kLb + lane] = inv[r];
    }
    __syncthreads();
    // R2 = A11^{-1} W[P, :] (2 x ntp fragments), pivot columns A11^{-1}
    for (int t = warp; t < 2 * ntp; t += kWarps) {
      const int I = t & 1, J = t >> 1;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < kB; kk += 4)
        gj_dmma(d0, d1, Ai[(I * 8 + gm) * kLb + kk + gk], Rb[(kk + gk) * ldr + J * 8 + gm]);
      const int r = I * 8 + gm, c = J * 8 + 2 * gk;
      R2[r * ldr + c] = (c >= k0 && c < k0 + bb) ? Ai[r * kLb + c - k0] : d0;
      R2[r * ldr + c + 1] = (c + 1 >= k0 && c + 1 < k0 + bb) ? Ai[r * kLb + c + 1 - k0] : d1;
    }
    __syncthreads();
    // W_next = W' - C' R2 over this CTA's 8 x 32 strips; the next strip's
    // loads are issued before this strip's DMMAs.  Strips clear of the pivot
    // rows / columns and of the ragged edge (most of them) take a path
    // without per-element predicates.
    constexpr int kSJ = 4;  // 8-column tiles per strip
    const int nch = (ntp + kSJ - 1) / kSJ, nit = ntp * nch;
    auto clean = [&](int it) {
      const int r0 = (it / nch) * 8, c0s = (it % nch) * 8 * kSJ;
      return it < nit && r0 + 8 <= n && c0s + 8 * kSJ <= n &&
             (r0 + 8 <= k0 || r0 >= k0 + bb) && (c0s + 8 * kSJ <= k0 || c0s >= k0 + bb);
    };
    auto load_strip = [&](int it, double (&o)[kSJ][2]) {
      const int I = it / nch, ch = it % nch;
      const int r = I * 8 + gm;
      if (clean(it)) {
        const double* wr = W + size_t(r) * tl + ch * 8 * kSJ + 2 * gk;
#pragma unroll
        for (int jj = 0; jj < kSJ; ++jj) {
          o[jj][0] = wr[8 * jj];
          o[jj][1] = wr[8 * jj + 1];
        }
        return;
      }
      const bool rp = r >= k0 && r < k0 + bb;
#pragma unroll
      for (int jj = 0; jj < kSJ; ++jj)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int c = (ch * kSJ + jj) * 8 + 2 * gk + v;
          const bool cp = c >= k0 && c < k0 + bb;
          o[jj][v] = (it < nit && r < n && c < n && !rp && !cp) ? W[size_t(r) * tl + c] : 0.0;
        }
    };
    const int it0 = crank * kWarps + warp, its = kWarps * ncl;
    // two strips' loads in flight ahead of the current one
    double old[kSJ][2], nx1[kSJ][2];
    load_strip(it0, old);
    load_strip(it0 + its, nx1);
    for (int it = it0; it < nit; it += its) {
      double nxt[kSJ][2];
      load_strip(it + 2 * its, nxt);
      const int I = it / nch, ch = it % nch;
      const int r = I * 8 + gm;
      double af[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) af[kk] = Cb[r * kLb + 4 * kk + gk];
      const double* r2 = R2 + gk * ldr + ch * 8 * kSJ + gm;
      double d[kSJ][2];
#pragma unroll
      for (int jj = 0; jj < kSJ; ++jj) {
        d[jj][0] = d[jj][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) gj_dmma(d[jj][0], d[jj][1], af[kk], r2[4 * kk * ldr + 8 * jj]);
      }
      if (clean(it)) {
        double* wn = Wn + size_t(r) * tl + ch * 8 * kSJ + 2 * gk;
#pragma unroll
        for (int jj = 0; jj < kSJ; ++jj) {
          wn[8 * jj] = old[jj][0] - d[jj][0];
          wn[8 * jj + 1] = old[jj][1] - d[jj][1];
        }
      } else if (r < n) {
#pragma unroll
        for (int jj = 0; jj < kSJ; ++jj) {
          const int c = (ch * kSJ + jj) * 8 + 2 * gk;
          if (c < n) Wn[size_t(r) * tl + c] = old[jj][0] - d[jj][0];
          if (c + 1 < n) Wn[size_t(r) * tl + c + 1] = old[jj][1] - d[jj][1];
        }
      }
#pragma unroll
      for (int jj = 0; jj < kSJ; ++jj) {
        old[jj][0] = nx1[jj][0];
        old[jj][1] = nx1[jj][1];
        nx1[jj][0] = nxt[jj][0];
        nx1[jj][1] = nxt[jj][1];
      }
    }
    sync_all();  // every CTA's strips of Wn written before the next pass reads them
  }
  if (crank != 0 || !guard) return;
  // pivot guard (linalg.cpp:69-73): every diagonal of U against max |G_x|;
  // growth guard: every factor entry against growth * max |G_x|
  double bad = 0.0, big = 0.0;
  const double floor_ = piv_tol * fmax(scale_in[s], 1e-300);
  for (int j = threadIdx.x; j < P.n; j += BLOCK) {
    const double d = Fs[P.diag[j]];
    if (!(fabs(d) >= floor_) || !isfinite(d)) bad = 1.0;
  }
  for (int q = threadIdx.x; q < P.nnz_f; q += BLOCK) big = fmax(big, fabs(Fs[q]));
  bad = block_reduce<BLOCK>(bad, true);
  big = block_reduce<BLOCK>(big, true);
  if (threadIdx.x == 0)
    status[s] = bad > 0.0 ? 1 : (big > P.growth * fmax(scale_in[s], 1e-300) ? 2 : 0);
}

// Cluster-resident Gauss-Jordan (opt-in, BIPM_GJ_CLUSTER_RESIDENT=1): a cluster
// of R CTAs holds W of one scenario in distributed shared memory, CTA r
// owning rows [r rb, r rb + rb) (rb a multiple of the 16-pivot block), so no
// pass touches global memory (the global-memory kernel above streams the
// whole tl x tl block through L2/HBM twice per pass: 4.9 GB per refactor at
// 1354/256).  Pass p, pivots P = [16 p, 16 p + 16) owned by CTA o:
//   o:   A11^{-1} (one warp; its pivots are U_TT's diagonal, written to the
//        factor for the guard), R2 = A11^{-1} W[P, :] with the pivot columns
//        replaced by A11^{-1}, into R2 slot p & 1;      cluster barrier
//   all: copy o's R2 slot over DSMEM, stage C' = own rows' pivot columns
//        (pivot rows -e_p), own rows <- W' - C' R2 on DMMA (8 x 32 strips),
//        W' = W with the pivot rows and columns zeroed
// Two R2 slots: one cluster barrier per pass (pass p + 2 reuses slot p & 1
// only after every CTA crossed pass p + 1's barrier, i.e. finished copying).
// Measured slower than the global-memory kernel (1354/256: 5.9 against 3.0 ms
// per refactor; pushing R2 with DSMEM stores instead of pulling it: 7.2 ms):
// the per-pass chain (one warp's A11 inverse, R2, the DSMEM transfer, the
// cluster barrier) is serial while 6 of 7 CTAs wait, and only 2 clusters of
// 7-8 one-CTA-per-SM members fit a GPC.  Kept for the record, not the default.
constexpr int kCgjLdb = 20;
inline __host__ __device__ int cgj_ldr(int tl) { return ((tl + 15) & ~15) + 4; }
inline size_t cgj_smem_bytes(int tl, int rb) {
  return (size_t(rb) * cgj_ldr(tl) + size_t(2) * kGjB * cgj_ldr(tl) + size_t(rb) * kCgjLdb +
          size_t(kGjB) * kCgjLdb) *
         sizeof(double);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    refactor_tail_cgj_kernel(DevLu P, double* F, double* D, const double* __restrict__ scale_in,
                             int* status, double piv_tol, int rb) {
  constexpr int kB = kGjB, kLb = kCgjLdb, kWarps = BLOCK / 32;
  extern __shared__ double cgj[];
  cg::cluster_group cluster = cg::this_cluster();
  const int R = int(cluster.num_blocks()), cr = int(cluster.block_rank());
  const int s = blockIdx.x / R;
  double* Fs = F + size_t(s) * P.nnz_f;
  const int tl = P.tl, tt = tl * tl, t0 = P.t0;
  const int ldr = cgj_ldr(tl);
  double* Wl = cgj;                        // [rb][ldr] own rows of W
  double* R2s = Wl + size_t(rb) * ldr;     // [2][kB][ldr]
  double* Cp = R2s + size_t(2) * kB * ldr;  // [rb][kLb] C'
  double* Ai = Cp + size_t(rb) * kLb;      // [kB][kLb] A11^{-1}
  const int r0 = cr * rb, nr = max(0, min(rb, tl - r0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gm = lane >> 2, gk = lane & 3;
  // own rows of S from the factor (zero beyond tl: padding columns stay 0)
  for (int i = warp; i < rb; i += kWarps) {
    const int gi = r0 + i;
    for (int j = lane; j < ldr; j += 32) {
      double v = 0.0;
      if (i < nr && j < tl) {
        const int src = gi > j ? P.dense_src[j * tl + gi] : P.dense_src[tt + j * tl + gi];
        v = src >= 0 ? Fs[src] : 0.0;
      }
      Wl[i * ldr + j] = v;
    }
  }
  cluster.sync();
  const int npass = (tl + kB - 1) / kB, ntp = (tl + 7) / 8, nch = (tl + 31) / 32;
  for (int p = 0; p < npass; ++p) {
    const int k0 = p * kB, bb = min(kB, tl - k0), o = k0 / rb;
    double* R2 = R2s + size_t(p & 1) * kB * ldr;
    if (cr == o) {
      const int lr0 = k0 - r0;
      if (warp == 0) {  // A11^{-1} by Gauss-Jordan, lane = column (identity-padded)
        double col[kB], inv[kB];
#pragma unroll
        for (int r = 0; r < kB; ++r) {
          col[r] = (lane < bb && r < bb) ? Wl[(lr0 + r) * ldr + k0 + lane] : (r == lane ? 1.0 : 0.0);
          inv[r] = (r == lane) ? 1.0 : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
          const double piv = __shfl_sync(0xffffffffu, col[k], k);
          if (lane == 0 && k < bb) Fs[P.diag[t0 + k0 + k]] = piv;
          const double rp = 1.0 / piv;
          col[k] *= rp;
          inv[k] *= rp;
#pragma unroll
          for (int r = 0; r < kB; ++r) {
            const double f = __shfl_sync(0xffffffffu, col[r], k);
            if (r != k) {
              col[r] -= f * col[k];
              inv[r] -= f * inv[k];
            }
          }
        }
        if (lane < kB)
#pragma unroll
          for (int r = 0; r < kB; ++r) Ai[r * kLb + lane] = inv[r];
      }
      __syncthreads();
      // R2 = A11^{-1} W[P, :] (2 x ntp fragments), pivot columns A11^{-1}
      for (int t = warp; t < 2 * ntp; t += kWarps) {
        const int I = t & 1, J = t >> 1;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < kB; kk += 4)
          gj_dmma(d0, d1, Ai[(I * 8 + gm) * kLb + kk + gk], Wl[(lr0 + kk + gk) * ldr + J * 8 + gm]);
        const int r = I * 8 + gm, c = J * 8 + 2 * gk;
        R2[r * ldr + c] = (c >= k0 && c < k0 + bb) ? Ai[r * kLb + c - k0] : d0;
        R2[r * ldr + c + 1] = (c + 1 >= k0 && c + 1 < k0 + bb) ? Ai[r * kLb + c + 1 - k0] : d1;
      }
    }
    cluster.sync();  // R2 of pass p complete in o's slot
    if (cr != o) {
      const double2* src = reinterpret_cast<const double2*>(cluster.map_shared_rank(R2, o));
      double2* dst = reinterpret_cast<double2*>(R2);
      for (int q = tid; q < kB * ldr / 2; q += BLOCK) dst[q] = src[q];
    }
    for (int q = tid; q < rb * kB; q += BLOCK) {
      const int i = q / kB, pp = q % kB, gi = r0 + i;
      double v = 0.0;
      if (pp < bb && i < nr)
        v = (gi >= k0 && gi < k0 + bb) ? (gi - k0 == pp ? -1.0 : 0.0) : Wl[i * ldr + k0 + pp];
      Cp[i * kLb + pp] = v;
    }
    __syncthreads();
    // own rows <- W' - C' R2 (in place: an element's update reads itself and
    // the staged operands only)
    for (int it = warp; it < (nr + 7) / 8 * nch; it += kWarps) {
      const int I = it / nch, ch = it % nch;
      const int r = I * 8 + gm, gi = r0 + r;
      double af[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) af[kk] = Cp[r * kLb + 4 * kk + gk];
      const double* r2 = R2 + gk * ldr + ch * 32 + gm;
      double d[4][2];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        d[jj][0] = d[jj][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          gj_dmma(d[jj][0], d[jj][1], af[kk], r2[4 * kk * ldr + 8 * jj]);
      }
      const bool prow = gi >= k0 && gi < k0 + bb;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int c = ch * 32 + 8 * jj + 2 * gk + v;
          if (r < nr && c < ldr) {
            const bool z = prow || (c >= k0 && c < k0 + bb);
            Wl[r * ldr + c] = (z ? 0.0 : Wl[r * ldr + c]) - d[jj][v];
          }
        }
    }
    __syncthreads();  // the next pass's pivot rows are final before o reads them
  }
  // W (row-major) to D's W slot
  double* W = D + size_t(s) * 2 * tt;
  for (int i = warp; i < nr; i += kWarps)
    for (int j = lane; j < tl; j += 32) W[size_t(r0 + i) * tl + j] = Wl[i * ldr + j];
  cluster.sync();  // every owner's pivots are in the factor before the guard
  if (cr != 0) return;
  double bad = 0.0, big = 0.0;
  const double floor_ = piv_tol * fmax(scale_in[s], 1e-300);
  for (int j = tid; j < P.n; j += BLOCK) {
    const double dd = Fs[P.diag[j]];
    if (!(fabs(dd) >= floor_) || !isfinite(dd)) bad = 1.0;
  }
  for (int q = tid; q < P.nnz_f; q += BLOCK) big = fmax(big, fabs(Fs[q]));
  bad = block_reduce<BLOCK>(bad, true);
  big = block_reduce<BLOCK>(big, true);
  if (tid == 0) status[s] = bad > 0.0 ? 1 : (big > P.growth * fmax(scale_in[s], 1e-300) ? 2 : 0);
}

// the solve layouts after the Gauss-Jordan tail, spread over the whole GPU:
// FT and VS gathers from F, W' = transpose(W)
__global__ void refactor_layouts_kernel(DevLu P, const double* __restrict__ F, double* FT,
                                        double* D, const int* __restrict__ vs_src, int nnz_vs,
                                        double* VS, int M) {
  const long long n1 = (long long)M * P.nnz_f, n2 = (long long)M * nnz_vs;
  const int tl = P.tl, tt = tl * tl;
  const long long n3 = 0;  // W' by transpose_w_kernel
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n1 + n2 + n3;
       q += stride) {
    if (q < n1) {
      const int s = int(q / P.nnz_f), e = int(q % P.nnz_f);
      FT[q] = F[size_t(s) * P.nnz_f + P.ft_src[e]];
    } else if (q < n1 + n2) {
      const long long r = q - n1;
      const int s = int(r / nnz_vs), e = int(r % nnz_vs);
      const int src = vs_src[e];
      VS[r] = src >= 0 ? F[size_t(s) * P.nnz_f + src] : 0.0;
    } else {
      const long long r = q - n1 - n2;
      const int s = int(r / tt), e = int(r % tt);
      const int i = e / tl, j = e % tl;  // W'(i, j) = W(j, i)
      double* W = D + size_t(s) * 2 * tt;
      W[tt + e] = W[j * tl + i];
    }
  }
}

// W' = transpose(W) per scenario through 32 x 32 shared-memory tiles (both
// sides coalesced; the element-wise form in refactor_layouts_kernel read W
// with a stride of tl doubles), and the reduction's row-padded copy (Dp, rows
// of ldw doubles, zero beyond tl) of W, W' or both (slot 0, 1, -1) from the
// same tiles, which replaces pad_dense_kernel's second pass over D
__global__ void transpose_w_kernel(double* D, int tl, double* Dp, int ldw, int slot) {
  __shared__ double t[32][33];
  const int tt = tl * tl, s = blockIdx.z;
  double* W = D + size_t(s) * 2 * tt;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;  // W rows i0.., columns j0..
  const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
  // padded row r of slot k of this scenario (Dp keeps the [M][2][tl][ldw]
  // layout when only one slot is written, as pad_dense_kernel does)
  auto prow = [&](int k, int r) -> double* {
    return Dp + ((size_t(s) * 2 + k) * tl + r) * ldw;
  };
  for (int r = y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + x;
    const double v = i < tl && j < tl ? W[size_t(i) * tl + j] : 0.0;
    t[r][x] = v;
    if (Dp && slot != 1 && i < tl && j < ldw) prow(0, i)[j] = v;
  }
  __syncthreads();
  for (int r = y; r < 32; r += 8) {  // W'(j0 + r, i0 + x) = W(i0 + x, j0 + r)
    const int i = j0 + r, j = i0 + x;
    if (i >= tl) continue;
    if (j < tl) W[tt + size_t(i) * tl + j] = t[x][r];
    if (Dp && slot != 0 && j < ldw) prow(1, i)[j] = j < tl ? t[x][r] : 0.0;
  }
}

// W, W' (row-major tl x tl, two per scenario) -> rows padded to ldw doubles
// (slot >= 0: that slot only, n then counts [M][tl][ldw])
__global__ void pad_dense_kernel(const double* __restrict__ D, double* __restrict__ Dp, int tl,
                                 int ldw, long long n, int slot) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    long long row = q / ldw;  // over [M][2][tl] (or [M][tl] for one slot)
    const int j = int(q % ldw);
    long long o = q;
    if (slot >= 0) {
      row = (row / tl) * 2 * tl + slot * tl + row % tl;
      o = row * ldw + j;
    }
    Dp[o] = j < tl ? D[row * tl + j] : 0.0;
  }
}

// ----------------------------------------------------------- Schur reduction
__device__ __forceinline__ FactorView factor_of(const DevLu& P, const double* F, const double* FT,
                                                const double* D, int s) {
  return FactorView{F + size_t(s) * P.nnz_f, FT + size_t(s) * P.nnz_f,
                    D + size_t(s) * 2 * P.tl * P.tl};
}

template <int BLOCK, int K>
__global__ void __launch_bounds__(BLOCK, 1) reduce_tiles_kernel(ReduceLaunch a) {
  extern __shared__ double sm[];
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int cta = chunk * gridDim.x + tile;
  const int j0 = tile * K;
  const int k = min(K, a.n_u - j0);
  const int n_x = a.n_x, n_u = a.n_u;
  const size_t per_cta = size_t(n_x) * K * (a.panel_in_smem ? 1 : 2);
  double* acc = sm;
  double* S = a.scratch + size_t(cta) * per_cta;
  double* X = a.panel_in_smem ? sm + size_t(n_u) * K : S + size_t(n_x) * K;
  const DevLu& P = a.lu;

  for (int i = threadIdx.x; i < n_u * K; i += BLOCK) acc[i] = 0.0;
  const int s_lo = chunk * a.chunk, s_hi = min(a.M, s_lo + a.chunk);
  const bool stamp = a.phase && cta == 0 && threadIdx.x == 0;
  int np = 0;
  auto mark = [&](int s) {
    if (stamp && s == s_lo) a.phase[np++] = clock64();
  };
  for (int s = s_lo; s < s_hi; ++s) {
    const FactorView F = factor_of(P, a.F, a.FT, a.D, s);
    mark(s);
    const double* __restrict__ gu = a.gu_v + size_t(s) * a.gu.nnz;
    const double* __restrict__ kxx = a.kxx_v + size_t(s) * a.kxx.nnz;
    const double* __restrict__ kxu = a.kxu_v + size_t(s) * a.kxu.nnz;
    const double* __restrict__ kuu = a.kuu_v + size_t(s) * a.kuu.nnz;
    const double* __restrict__ sig = a.sigma_x + size_t(s) * n_x;

    // V = Cartesian columns [j0, j0+k): X = P G_u V (columns >= k stay zero)
    for (int i = threadIdx.x; i < n_x * K; i += BLOCK) X[i] = 0.0;
    __syncthreads();
    {
      const int q0 = a.gu.t_ptr[j0], q1 = a.gu.t_ptr[j0 + k];
      for (int q = q0 + threadIdx.x; q < q1; q += BLOCK) {
        int c = 0;
        while (a.gu.t_ptr[j0 + c + 1] <= q) ++c;
        X[P.iperm[a.gu.t_row[q]] * K + c] = gu[a.gu.t_slot[q]];
      }
    }
    __syncthreads();
    mark(s);
    // X = G_x^{-1} G_u V, T = -X
    level_sweep<BLOCK, K, false>(P.sL, F.F, X);
    mark(s);
    tail_gather<BLOCK, K, false>(P.sL, F.F, X);
    mark(s);
    dense_tail_gemm<BLOCK, K>(P, dense_block(P, F, 0), X);
    mark(s);
    level_sweep<BLOCK, K, true>(P.sU, F.F + P.nnz_l, X);
    mark(s);

    // acc += K_xu' T + K_uu V;  S = P (K~_xx T + K_xu V)
    for (int it = threadIdx.x; it < n_u * K; it += BLOCK) {
      const int u = it / K, c = it % K;
      double v = 0.0;
      for (int q = a.kxu.t_ptr[u]; q < a.kxu.t_ptr[u + 1]; ++q)
        v -= kxu[a.kxu.t_slot[q]] * X[P.iperm[a.kxu.t_row[q]] * K + c];
      if (c < k) {
        const int ku = find_in_row(a.kuu.ptr, a.kuu.ind, u, j0 + c);
        if (ku >= 0) v += kuu[ku];
      }
      acc[it] += v;
    }
    for (int it = threadIdx.x; it < n_x * K; it += BLOCK) {
      const int p = it / K, c = it % K;
      const int i = P.perm[p];
      double v = 0.0;
      for (int t = a.kxx.ptr[i]; t < a.kxx.ptr[i + 1]; ++t)
        v -= kxx[t] * X[P.iperm[a.kxx.ind[t]] * K + c];
      v -= (sig[i] + a.dw) * X[p * K + c];
      if (c < k) {
        const int ks = find_in_row(a.kxu.ptr, a.kxu.ind, i, j0 + c);
        if (ks >= 0) v += kxu[ks];
      }
      S[p * K + c] = v;
    }
    __syncthreads();
    mark(s);
    for (int i = threadIdx.x; i < n_x * K; i += BLOCK) X[i] = S[i];
    __syncthreads();
    // X = P G_x^{-T} L_x  (Y[perm[p]] = X[p])
    level_sweep<BLOCK, K, true>(P.sUt, F.FT, X);
    mark(s);
    tail_gather<BLOCK, K, true>(P.sUt, F.FT, X);
    mark(s);
    dense_tail_gemm<BLOCK, K>(P, dense_block(P, F, 1), X);
    mark(s);
    level_sweep<BLOCK, K, false>(P.sLt, F.FT + (P.nnz_f - P.nnz_l), X);
    mark(s);
    // acc -= G_u' Y
    for (int it = threadIdx.x; it < n_u * K; it += BLOCK) {
      const int u = it / K, c = it % K;
      double v = 0.0;
      for (int q = a.gu.t_ptr[u]; q < a.gu.t_ptr[u + 1]; ++q)
        v += gu[a.gu.t_slot[q]] * X[P.iperm[a.gu.t_row[q]] * K + c];
      acc[it] -= v;
    }
    __syncthreads();
    mark(s);
  }
  double* out = a.partial + size_t(chunk) * n_u * n_u;
  for (int it = threadIdx.x; it < n_u * K; it += BLOCK) {
    const int u = it / K, c = it % K;
    if (c < k) out[size_t(j0 + c) * n_u + u] = acc[it];
  }
}

// sym_n > 0: the parts are n x n column-major and only their lower triangles
// are read (the reduction's tail GEMM writes no upper tiles); the result is
// mirrored, so K_hat is exactly symmetric
__global__ void sum_parts_kernel(const double* parts, int nparts, long long len,
                                 double* out, const double* diag_add, double dw, int n_mat,
                                 const double* sub_vec, int sym_n) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= len) return;
  const long long col = sym_n > 0 ? j / sym_n : 0, row = sym_n > 0 ? j % sym_n : 0;
  if (sym_n > 0 && row < col) return;
  // fixed order: four interleaved running sums combined pairwise
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int c = 0;
  for (; c + 3 < nparts; c += 4) {
    s0 += parts[(long long)c * len + j];
    s1 += parts[(long long)(c + 1) * len + j];
    s2 += parts[(long long)(c + 2) * len + j];
    s3 += parts[(long long)(c + 3) * len + j];
  }
  for (; c < nparts; ++c) s0 += parts[(long long)c * len + j];
  double v = (s0 + s1) + (s2 + s3);
  if (n_mat > 0 && diag_add && (j % (n_mat + 1)) == 0) v += diag_add[j / (n_mat + 1)] + dw;
  if (sub_vec) v -= sub_vec[j];
  out[j] = v;
  if (sym_n > 0 && row != col) out[row * sym_n + col] = v;
}

__global__ void affine_mix_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  double t, long long len, double* out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < len) out[j] = a[j] + t * (b[j] - a[j]);
}

// ------------------------------------------------------ single-RHS kernels
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) reduce_rhs_kernel(RhsLaunch a, double* scratch,
                                                           int in_smem) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  const int n_x = a.n_x;
  const DevLu& P = a.lu;
  double* X = in_smem ? sm : scratch + size_t(s) * 2 * n_x;
  double* Z = X + n_x;
  const FactorView F = factor_of(P, a.F, a.FT, a.D, s);
  const double* __restrict__ gu = a.gu_v + size_t(s) * a.gu.nnz;
  const double* __restrict__ kxx = a.kxx_v + size_t(s) * a.kxx.nnz;
  const double* __restrict__ kxu = a.kxu_v + size_t(s) * a.kxu.nnz;
  const double* __restrict__ sig = a.sigma_x + size_t(s) * n_x;
  const double* __restrict__ r1 = a.rhat1 + size_t(s) * n_x;
  const double* __restrict__ r3 = a.rhat3 + size_t(s) * n_x;

  // debug: clock64 after each phase, CTA 0 (RhsLaunch::phase)
  int np = 0;
  auto mark = [&] {
    if (a.phase && s == 0 && threadIdx.x == 0) a.phase[np++] = clock64();
  };
  mark();
  for (int p = threadIdx.x; p < n_x; p += BLOCK) X[p] = r3[P.perm[p]];
  __syncthreads();
  mark();
  // X = P a
  level_sweep<BLOCK, 1, false>(P.sL, F.F, X);
  mark();
  tail_gather<BLOCK, 1, false>(P.sL, F.F, X);
  dense_tail_gemm<BLOCK, 1>(P, dense_block(P, F, 0), X);
  mark();
  level_sweep<BLOCK, 1, true>(P.sU, F.F + P.nnz_l, X);
  mark();
  // Z = P (rhat1 - K~ a)
  for (int p = threadIdx.x; p < n_x; p += BLOCK) {
    const int i = P.perm[p];
    double acc = 0.0;
    for (int t = a.kxx.ptr[i]; t < a.kxx.ptr[i + 1]; ++t) acc += kxx[t] * X[P.iperm[a.kxx.ind[t]]];
    double v = r1[i] + -1.0 * acc;
    v -= (sig[i] + a.dw) * X[p];
    Z[p] = v;
  }
  __syncthreads();
  mark();
  level_sweep<BLOCK, 1, true>(P.sUt, F.FT, Z);
  mark();
  tail_gather<BLOCK, 1, true>(P.sUt, F.FT, Z);
  dense_tail_gemm<BLOCK, 1>(P, dense_block(P, F, 1), Z);
  mark();
  level_sweep<BLOCK, 1, false>(P.sLt, F.FT + (P.nnz_f - P.nnz_l), Z);
  mark();
  double* out = a.part + size_t(s) * a.n_u;
  for (int u = threadIdx.x; u < a.n_u; u += BLOCK) {
    double v = 0.0;
    for (int q = a.gu.t_ptr[u]; q < a.gu.t_ptr[u + 1]; ++q)
      v += gu[a.gu.t_slot[q]] * Z[P.iperm[a.gu.t_row[q]]];
    for (int q = a.kxu.t_ptr[u]; q < a.kxu.t_ptr[u + 1]; ++q)
      v += kxu[a.kxu.t_slot[q]] * X[P.iperm[a.kxu.t_row[q]]];
    out[u] = v;
  }
  if (a.phase) {
    __syncthreads();
    mark();
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) recover_state_kernel(RecoverLaunch a, double* scratch,
                                                              int in_smem) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  const int n_x = a.n_x;
  const DevLu& P = a.lu;
  double* X = in_smem ? sm : scratch + size_t(s) * 2 * n_x;
  double* Z = X + n_x;
  const FactorView F = factor_of(P, a.F, a.FT, a.D, s);
  const double* __restrict__ gu = a.gu_v + size_t(s) * a.gu.nnz;
  const double* __restrict__ kxx = a.kxx_v + size_t(s) * a.kxx.nnz;
  const double* __restrict__ kxu = a.kxu_v + size_t(s) * a.kxu.nnz;
  const double* __restrict__ sig = a.sigma_x + size_t(s) * n_x;
  const double* __restrict__ r1 = a.rhat1 + size_t(s) * n_x;
  const double* __restrict__ r3 = a.rhat3 + size_t(s) * n_x;
  double* px = a.px + size_t(s) * n_x;
  double* py = a.py + size_t(s) * n_x;

  // p_x = -G_x^{-1} (rhat3 + G_u p_u)
  for (int p = threadIdx.x; p < n_x; p += BLOCK) {
    const int i = P.perm[p];
    double acc = 0.0;
    for (int t = a.gu.ptr[i]; t < a.gu.ptr[i + 1]; ++t) acc += gu[t] * a.pu[a.gu.ind[t]];
    X[p] = r3[i] + 1.0 * acc;
  }
  __syncthreads();
  solve_LU<BLOCK, 1>(P, F, X);
  for (int p = threadIdx.x; p < n_x; p += BLOCK) {
    X[p] = -X[p];
    px[P.perm[p]] = X[p];
  }
  __syncthreads();
  // p_y = -G_x^{-T} (rhat1 + K~ p_x + K_xu p_u)
  for (int p = threadIdx.x; p < n_x; p += BLOCK) {
    const int i = P.perm[p];
    double acc = 0.0;
    for (int t = a.kxx.ptr[i]; t < a.kxx.ptr[i + 1]; ++t) acc += kxx[t] * X[P.iperm[a.kxx.ind[t]]];
    double v = r1[i] + 1.0 * acc;
    v += (sig[i] + a.dw) * X[p];
    double au = 0.0;
    for (int t = a.kxu.ptr[i]; t < a.kxu.ptr[i + 1]; ++t) au += kxu[t] * a.pu[a.kxu.ind[t]];
    Z[p] = v + 1.0 * au;
  }
  __syncthreads();
  solve_LUt<BLOCK, 1>(P, F, Z);
  for (int p = threadIdx.x; p < n_x; p += BLOCK) py[P.perm[p]] = -Z[p];
}

__global__ void recover_slack_kernel(DevCsr hx, DevCsr hu, int m, int n_x, int M,
                                     const double* __restrict__ hxv, const double* __restrict__ huv,
                                     const double* __restrict__ px, const double* __restrict__ pu,
                                     const double* __restrict__ sigma_s,
                                     const double* __restrict__ r2, const double* __restrict__ r4,
                                     double* pz, double* ps) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)m * M) return;
  const int s = int(id / m), i = int(id % m);
  const double* hxs = hxv + size_t(s) * hx.nnz;
  const double* hus = huv + size_t(s) * hu.nnz;
  const double* pxs = px + size_t(s) * n_x;
  // row i of H_x p_x in order, four entries' loads in flight
  double a = 0.0;
  int t = hx.ptr[i];
  const int t1 = hx.ptr[i + 1];
  for (; t + 4 <= t1; t += 4) {
    int ci[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ci[u] = hx.ind[t + u];
    double hv[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      hv[u] = hxs[t + u];
      xv[u] = pxs[ci[u]];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) a += hv[u] * xv[u];
  }
  for (; t < t1; ++t) a += hxs[t] * pxs[hx.ind[t]];
  double hp = 0.0 + 1.0 * a;
  double b = 0.0;
  for (int t = hu.ptr[i]; t < hu.ptr[i + 1]; ++t) b += hus[t] * pu[hu.ind[t]];
  hp += 1.0 * b;
  const double sg = sigma_s[id], rr2 = r2[id];
  const double z = sg * (hp + r4[id]) - rr2;
  pz[id] = z;
  ps[id] = -(rr2 + z) / sg;
}

__global__ void condense_kernel(CondenseDev c, int M, const double* __restrict__ W, int ldw,
                                const double* __restrict__ A, int lda,
                                const double* __restrict__ B, int ldb,
                                const double* __restrict__ sigma, int lds, double* out) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)c.nout * M) return;
  const int s = int(id / c.nout), o = int(id % c.nout);
  const double* Ws = W + size_t(s) * ldw;
  const double* As = A + size_t(s) * lda;
  const double* Bs = B + size_t(s) * ldb;
  const double* Ss = sigma + size_t(s) * lds;
  double v = 0.0;
  if (c.w_of[o] >= 0) v = __dadd_rn(v, Ws[c.w_of[o]]);
  for (int t = c.ptr[o]; t < c.ptr[o + 1]; ++t)
    v = __dadd_rn(v, __dmul_rn(__dmul_rn(As[c.ka[t]], Ss[c.r[t]]), Bs[c.kb[t]]));
  out[size_t(s) * c.nout + o] = v;
}

// ------------------------------------------------ dense Cholesky, n <= 150
// The whole matrix in shared memory; right-looking by columns (LAPACK dpotrf
// semantics: fail at the first pivot that is not > 0 or is NaN).
constexpr int kSmallChol = 150;

__global__ void __launch_bounds__(kDenseBlock) shift_cholesky_small_kernel(double* K, int n,
                                                                          int* info) {
  extern __shared__ double A[];  // n x n column-major
  __shared__ int fail;
  double mx = 0.0;
  for (int i = threadIdx.x; i < n * n; i += kDenseBlock) {
    const double v = K[i];
    A[i] = v;
    mx = fmax(mx, fabs(v));
  }
  mx = block_reduce<kDenseBlock>(mx, true);
  const double shift = 1e-13 * fmax(1.0, mx);
  for (int i = threadIdx.x; i < n; i += kDenseBlock) A[i * n + i] += shift;
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double ajj = A[j * n + j];
      if (!(ajj > 0.0) || isnan(ajj)) {
        fail = j + 1;
        reinterpret_cast<double*>(info)[2] = ajj;  // the rejected pivot (factor_khat)
      } else {
        A[j * n + j] = sqrt(ajj);
      }
    }
    __syncthreads();
    if (fail) break;
    const double ljj = A[j * n + j];
    for (int i = j + 1 + threadIdx.x; i < n; i += kDenseBlock) A[j * n + i] /= ljj;
    __syncthreads();
    // trailing update of the lower triangle: A(i,k) -= L(i,j) L(k,j), j < k <= i
    const int m = n - j - 1;
    for (int t = threadIdx.x; t < m * m; t += kDenseBlock) {
      const int kk = t / m, ii = t - kk * m;  // column kk, row ii of the trailing block
      if (ii < kk) continue;
      const int k = j + 1 + kk, i = j + 1 + ii;
      A[k * n + i] -= A[j * n + i] * A[j * n + k];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n * n; i += kDenseBlock) K[i] = A[i];
  if (threadIdx.x == 0) {
    *info = fail;
    reinterpret_cast<double*>(info)[1] = mx;  // |K|_inf
  }
}

// L L' x = b for column-major lower L: one warp, x in registers (row i on
// lane i % 32), pivot broadcast by shuffle.
template <int NQ>
__global__ void cholesky_solve_warp_kernel(const double* __restrict__ L, int n, double* b) {
  const int lane = threadIdx.x & 31;
  double x[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) x[q] = (q * 32 + lane < n) ? b[q * 32 + lane] : 0.0;
  // forward: L y = b
#pragma unroll
  for (int qj = 0; qj < NQ; ++qj) {
    for (int jj = 0; jj < 32; ++jj) {
      const int j = qj * 32 + jj;
      if (j >= n) break;
      const double* __restrict__ col = L + size_t(j) * n;
      if (lane == jj) x[qj] /= col[j];
      const double xj = __shfl_sync(0xffffffffu, x[qj], jj);
#pragma unroll
      for (int q = qj; q < NQ; ++q) {
        const int i = q * 32 + lane;
        if (i > j && i < n) x[q] -= col[i] * xj;
      }
    }
  }
  // backward: L' x = y, column-oriented over rows of L
#pragma unroll
  for (int qj = NQ - 1; qj >= 0; --qj) {
    for (int jj = 31; jj >= 0; --jj) {
      const int j = qj * 32 + jj;
      if (j >= n) continue;
      if (lane == jj) x[qj] /= L[size_t(j) * n + j];
      const double xj = __shfl_sync(0xffffffffu, x[qj], jj);
#pragma unroll
      for (int q = 0; q <= qj; ++q) {
        const int i = q * 32 + lane;
        if (i < j) x[q] -= L[size_t(i) * n + j] * xj;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (q * 32 + lane < n) b[q * 32 + lane] = x[q];
}

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// (the level sweeps add their static level-pointer buffers, sweeps.cuh)
constexpr int kSingleRhsSmemCap = 200 * 1024;
size_t single_rhs_smem(int n_x) {
  const size_t b = size_t(2) * n_x * sizeof(double);
  return b <= size_t(kSingleRhsSmemCap) ? b : 0;
}

// the cluster-resident Gauss-Jordan (opt-in) when a cluster of <= 16 CTAs
// holds the tail (rb = 48 or 32 rows per CTA); false: the global-memory kernel
static bool cgj_launch(const DevLu& P, int M, double* F, double* D, const double* scale,
                       int* status, double piv_tol, cudaStream_t st) {
  static const int resident = [] {
    const char* e = std::getenv("BIPM_GJ_CLUSTER_RESIDENT");
    return e ? std::atoi(e) : 0;
  }();
  if (!resident || P.tl <= 0) return false;
  int rb = 0;
  for (int cand : {48, 32})
    if (cgj_smem_bytes(P.tl, cand) <= 227 * 1024 && (P.tl + cand - 1) / cand <= 16) {
      rb = cand;
      break;
    }
  if (rb == 0) return false;
  const int R = (P.tl + rb - 1) / rb;
  const size_t smem = cgj_smem_bytes(P.tl, rb);
  cudaFuncSetAttribute(refactor_tail_cgj_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  if (R > 8)
    cudaFuncSetAttribute(refactor_tail_cgj_kernel<512>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr{};
  cfg.gridDim = dim3(M * R);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = R;
  attr.val.clusterDim.y = attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, refactor_tail_cgj_kernel<512>, P, F, D, scale, status, piv_tol,
                         rb) != cudaSuccess) {
    cudaGetLastError();  // cluster shape not launchable here: the global-memory kernel
    return false;
  }
  note_launch();
  check_launch("refactor_tail_cgj");
  return true;
}

void launch_lu_refactor(const DevLu& P, int M, const double* gx, int nnz_gx, double* F,
                        double* FT, double* D, int* status, double piv_tol, const int* vs_src,
                        int nnz_vs, double* VS, double* Dp, double* scale, cudaStream_t st,
                        int dp_slot, cudaEvent_t after_levels) {
  if (M <= 0) return;
  bool padded = false;  // Dp written by transpose_w_kernel
  // up to one scenario per SM: 1024 threads per scenario shorten each
  // level's pass (measured refactor: 1354/32 0.84 -> 0.74 ms, 1354/148 1.46
  // -> 1.36, 9241/128 33.9 -> 27.5; BIPM_LEVELS_BLOCK=512|1024 for experiments)
  static const int levels_env = [] {
    const char* e = std::getenv("BIPM_LEVELS_BLOCK");
    return e ? std::atoi(e) : 0;
  }();
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const bool wide = levels_env ? levels_env == 1024 : M <= sms;
  if (wide)
    refactor_levels_kernel<1024><<<M, 1024, 0, st>>>(P, gx, nnz_gx, F, scale);
  else
    refactor_levels_kernel<512><<<M, 512, 0, st>>>(P, gx, nnz_gx, F, scale);
  note_launch();
  check_launch("refactor_levels");
  if (after_levels) cudaEventRecord(after_levels, st);
  const size_t smem = size_t(2) * P.tl * P.tl * sizeof(double);
  if (smem <= 200 * 1024) {
    cudaFuncSetAttribute(refactor_tail_kernel<kLuBlock>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    refactor_tail_kernel<kLuBlock><<<M, kLuBlock, smem, st>>>(P, F, FT, D, scale, status,
                                                              piv_tol, vs_src, nnz_vs, VS);
  } else if (cgj_launch(P, M, F, D, scale, status, piv_tol, st)) {
    if (P.tl > 0) {
      const int nb = (P.tl + 31) / 32;
      transpose_w_kernel<<<dim3(nb, nb, M), 256, 0, st>>>(D, P.tl, Dp, (P.tl + 15) & ~15,
                                                         dp_slot);
      note_launch();
      padded = true;
    }
    refactor_layouts_kernel<<<4 * 148, 512, 0, st>>>(P, F, FT, D, vs_src, VS ? nnz_vs : 0, VS,
                                                     M);
  } else {
    const size_t gsm = gj_smem_bytes(P.tl);
    cudaFuncSetAttribute(refactor_tail_gj_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(gsm));
    // small M: a cluster of CL CTAs per scenario so the grid covers the GPU
    static int max_cl = -1;
    if (max_cl < 0) {
      max_cl = 1;
      for (int c = 8; c > 1 && max_cl == 1; c /= 2) {
        cudaLaunchConfig_t q{};
        cudaLaunchAttribute qa{};
        q.gridDim = dim3(c);
        q.blockDim = dim3(512);
        q.dynamicSmemBytes = gsm;
        qa.id = cudaLaunchAttributeClusterDimension;
        qa.val.clusterDim.x = c;
        qa.val.clusterDim.y = qa.val.clusterDim.z = 1;
        q.attrs = &qa;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, refactor_tail_gj_kernel<512>, &q) == cudaSuccess &&
            n > 0)
          max_cl = c;
      }
      cudaGetLastError();
      if (const char* e = std::getenv("BIPM_GJ_CLUSTER")) max_cl = std::max(1, std::atoi(e));
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int cl = 1;
    while (cl * 2 <= max_cl && M * cl * 2 <= sms) cl *= 2;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr{};
    cfg.gridDim = dim3(M * cl);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = gsm;
    cfg.stream = st;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    auto gj = [&](int blk0, int blkn, int gather, int guard) {
      cudaLaunchKernelEx(&cfg, refactor_tail_gj_kernel<512>, P, F, FT, D,
                         static_cast<const double*>(scale), status, piv_tol, vs_src, nnz_vs, VS,
                         blk0, blkn, gather, guard);
      note_launch();
      check_launch("refactor_tail_gj");
    };
    // 2 x 2 block inversion (BIPM_GJ_BLOCK=0: one Gauss-Jordan over the whole
    // tail): S = [A B; C E], Ai = A^{-1} and Zi = (E - C Ai B)^{-1} by the
    // Gauss-Jordan kernel on the diagonal blocks in place (their pivots are
    // U_TT's diagonal in order), the rest by six DMMA GEMMs:
    //   T1 = Ai B, T2 = C Ai, E -= C T1 (= Z), W12 = -T1 Zi, W21 = -Zi T2,
    //   W11 = Ai - T1 W21;  T1, T2 live in the W' slot until the layouts
    static const int block_env = [] {  // recursion depth of the block inversion
      const char* e = std::getenv("BIPM_GJ_BLOCK");
      return e ? std::atoi(e) : 2;
    }();
    const int tl = P.tl;
    const long long tt = (long long)tl * tl, sw = 2 * tt;
    auto nn = [&](int m, int n, int k, double alpha, double beta, const double* A, long long lda,
                  const double* B, long long ldb, double* C, long long ldc) {
      launch_gemm_nn(GemmNN{m, n, k, M, alpha, beta, A, lda, sw, B, ldb, sw, C, ldc, sw}, st);
    };
    // invert the diagonal block [b0, b0 + n) of W in place; temporaries in the
    // W' slot from `off` on (the outer level's T1, T2 stay live while its
    // second half recurses)
    std::function<void(int, int, int, int, int, long long)> inv =
        [&](int b0, int n, int gather, int guard, int depth, long long off) {
          const int h = (n / 2) & ~15, r = n - h;
          if (depth <= 0 || h < 64 || cl != 1) {
            gj(b0, n, gather, guard);
            return;
          }
          double* Wb = D + (long long)b0 * tl + b0;  // block origin, stride tl
          double* T1 = D + tt + off;                  // h x r
          double* T2 = T1 + (long long)h * r;          // r x h
          double* Cb = Wb + (long long)h * tl;         // C, then W21
          double* Eb = Cb + h;                         // E, then Z, then Zi
          inv(b0, h, gather, 0, depth - 1, off);                    // A -> Ai
          nn(h, r, h, 1.0, 0.0, Wb, tl, Wb + h, tl, T1, r);          // T1 = Ai B
          nn(r, h, h, 1.0, 0.0, Cb, tl, Wb, tl, T2, h);              // T2 = C Ai
          nn(r, r, h, -1.0, 1.0, Cb, tl, T1, r, Eb, tl);             // E -= C T1
          inv(b0 + h, r, 0, guard, depth - 1, off + 2LL * h * r);   // Z -> Zi
          nn(h, r, r, -1.0, 0.0, T1, r, Eb, tl, Wb + h, tl);         // W12 = -T1 Zi
          nn(r, h, r, -1.0, 0.0, Eb, tl, T2, h, Cb, tl);             // W21 = -Zi T2
          nn(h, h, r, -1.0, 1.0, T1, r, Cb, tl, Wb, tl);             // W11 = Ai - T1 W21
        };
    inv(0, tl, 1, 1, block_env, 0);
    if (P.tl > 0) {
      const int nb = (P.tl + 31) / 32;
      transpose_w_kernel<<<dim3(nb, nb, M), 256, 0, st>>>(D, P.tl, Dp, (P.tl + 15) & ~15,
                                                         dp_slot);
      note_launch();
      padded = true;
    }
    refactor_layouts_kernel<<<4 * 148, 512, 0, st>>>(P, F, FT, D, vs_src, VS ? nnz_vs : 0, VS,
                                                     M);
  }
  note_launch();
  check_launch("refactor_tail");
  if (Dp && P.tl > 0 && !padded) {
    const int ldw = (P.tl + 15) & ~15;
    const long long n = (long long)M * (dp_slot >= 0 ? 1 : 2) * P.tl * ldw;
    pad_dense_kernel<<<int(std::min<long long>((n + 255) / 256, 8 * 148)), 256, 0, st>>>(
        D, Dp, P.tl, ldw, n, dp_slot);
    note_launch();
    check_launch("pad_dense");
  }
}

void plan_reduce_launch(ReduceLaunch& a, int smem_budget, int sm_count) {
  // widest tile (<= 32 columns) whose accumulator and panel fit on chip
  // widest power-of-two tile (<= 32 columns, <= n_u rounded up) whose
  // accumulator and panel fit on chip
  int cap = 1;
  while (cap < 32 && cap < a.n_u) cap *= 2;
  int kc = cap;
  while (kc > 1 && size_t(a.n_x + a.n_u) * kc * sizeof(double) > size_t(smem_budget)) kc /= 2;
  a.panel_in_smem = size_t(a.n_x + a.n_u) * kc * sizeof(double) <= size_t(smem_budget);
  if (!a.panel_in_smem) {
    kc = cap;
    while (kc > 1 && size_t(a.n_u) * kc * sizeof(double) > size_t(smem_budget)) kc /= 2;
  }
  a.kc = kc;
  const int tiles = (a.n_u + a.kc - 1) / a.kc;
  const int per_sm = std::max(1, int(smem_budget / std::max<size_t>(1, reduce_smem_bytes(a))));
  int nchunks = std::max(1, (4 * sm_count * std::min(per_sm, 4) + tiles - 1) / tiles);
  nchunks = std::min(nchunks, a.M);
  a.chunk = (a.M + nchunks - 1) / nchunks;
  a.nchunks = (a.M + a.chunk - 1) / a.chunk;
}

size_t reduce_smem_bytes(const ReduceLaunch& a) {
  return size_t(a.n_u + (a.panel_in_smem ? a.n_x : 0)) * a.kc * sizeof(double);
}

size_t reduce_scratch_doubles(const ReduceLaunch& a) {
  const int tiles = (a.n_u + a.kc - 1) / a.kc;
  return size_t(tiles) * a.nchunks * a.n_x * a.kc * (a.panel_in_smem ? 1 : 2);
}

template <int K>
void launch_reduce_k(const ReduceLaunch& a, cudaStream_t st) {
  const int tiles = (a.n_u + K - 1) / K;
  const size_t smem = reduce_smem_bytes(a);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(reduce_tiles_kernel<kReduceBlock, K>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr_set = true;
  }
  reduce_tiles_kernel<kReduceBlock, K><<<dim3(tiles, a.nchunks), kReduceBlock, smem, st>>>(a);
  note_launch();
}

void launch_reduce_tiles(const ReduceLaunch& a, cudaStream_t st) {
  if (a.M <= 0) return;
  switch (a.kc) {
    case 1: launch_reduce_k<1>(a, st); break;
    case 2: launch_reduce_k<2>(a, st); break;
    case 4: launch_reduce_k<4>(a, st); break;
    case 8: launch_reduce_k<8>(a, st); break;
    case 16: launch_reduce_k<16>(a, st); break;
    default: launch_reduce_k<32>(a, st); break;
  }
  check_launch("reduce_tiles");
}

void launch_sum_parts(const double* parts, int nparts, long long len, double* out,
                      const double* diag_add, double dw, int n_mat, const double* sub_vec,
                      cudaStream_t st, int sym_n) {
  if (len <= 0) return;
  const int B = 256;
  sum_parts_kernel<<<int((len + B - 1) / B), B, 0, st>>>(parts, nparts, len, out, diag_add, dw,
                                                          n_mat, sub_vec, sym_n);
  note_launch();
  check_launch("sum_parts");
}

void launch_affine_mix(const double* a, const double* b, double t, long long len, double* out,
                       cudaStream_t st) {
  if (len <= 0) return;
  affine_mix_kernel<<<int((len + 255) / 256), 256, 0, st>>>(a, b, t, len, out);
  note_launch();
  check_launch("affine_mix");
}

// 1024 threads per scenario while there is at most one scenario per SM
// (measured: 9241/128 rhs 3.85 -> 2.57 ms, recovery 3.70 -> 2.50 ms against
// 512 threads; 1354/128 0.25 -> 0.22 ms; BIPM_RHS_WIDE_M overrides the limit)
static bool wide_single_rhs(int M) {
  static const int lim = [] {
    const char* e = std::getenv("BIPM_RHS_WIDE_M");
    if (e) return std::atoi(e);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return M <= lim;
}

void launch_reduce_rhs(const RhsLaunch& a, cudaStream_t st) {
  if (a.M <= 0) return;
  const size_t smem = single_rhs_smem(a.n_x);
  double* scratch = a.scratch;
  if (!smem && !scratch) throw std::runtime_error("single-RHS kernels: scratch [M][2 n_x] required");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(reduce_rhs_kernel<kSolveBlock>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSingleRhsSmemCap);
    cudaFuncSetAttribute(reduce_rhs_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSingleRhsSmemCap);
    attr_set = true;
  }
  // latency-bound level sweeps: more threads per scenario while the scenarios
  // leave SMs free (measured at 1354: 256 -> 512 threads 0.44 -> 0.35 ms;
  // 1024 threads 0.29 ms at 32 scenarios, 0.56 ms at 256; wide_single_rhs)
  if (wide_single_rhs(a.M))
    reduce_rhs_kernel<1024><<<a.M, 1024, smem, st>>>(a, scratch, smem ? 1 : 0);
  else
    reduce_rhs_kernel<kSolveBlock><<<a.M, kSolveBlock, smem, st>>>(a, scratch, smem ? 1 : 0);
  note_launch();
  check_launch("reduce_rhs");
}

void launch_recover_state(const RecoverLaunch& a, cudaStream_t st) {
  if (a.M <= 0) return;
  const size_t smem = single_rhs_smem(a.n_x);
  double* scratch = a.scratch;
  if (!smem && !scratch) throw std::runtime_error("single-RHS kernels: scratch [M][2 n_x] required");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(recover_state_kernel<kSolveBlock>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSingleRhsSmemCap);
    cudaFuncSetAttribute(recover_state_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSingleRhsSmemCap);
    attr_set = true;
  }
  // latency-bound level sweeps: more threads per scenario while the scenarios
  // leave SMs free (measured at 1354: 256 -> 512 threads 0.44 -> 0.35 ms;
  // 1024 threads 0.29 ms at 32 scenarios, 0.56 ms at 256; wide_single_rhs)
  if (wide_single_rhs(a.M))
    recover_state_kernel<1024><<<a.M, 1024, smem, st>>>(a, scratch, smem ? 1 : 0);
  else
    recover_state_kernel<kSolveBlock><<<a.M, kSolveBlock, smem, st>>>(a, scratch, smem ? 1 : 0);
  note_launch();
  check_launch("recover_state");
}

void launch_recover_slack(const DevCsr& hx, const DevCsr& hu, int m, int n_x, int M,
                          const double* hx_v, const double* hu_v, const double* px,
                          const double* pu, const double* sigma_s, const double* r2,
                          const double* r4, double* pz, double* ps, cudaStream_t st) {
  const long long n = (long long)m * M;
  if (n <= 0) return;
  recover_slack_kernel<<<int((n + 255) / 256), 256, 0, st>>>(hx, hu, m, n_x, M, hx_v, hu_v, px,
                                                              pu, sigma_s, r2, r4, pz, ps);
  note_launch();
  check_launch("recover_slack");
}

void launch_condense(const CondenseDev& c, int M, const double* W, int ldw, const double* A,
                     int lda, const double* B, int ldb, const double* sigma, int lds, double* out,
                     cudaStream_t st) {
  const long long n = (long long)c.nout * M;
  if (n <= 0) return;
  condense_kernel<<<int((n + 255) / 256), 256, 0, st>>>(c, M, W, ldw, A, lda, B, ldb, sigma, lds,
                                                         out);
  note_launch();
  check_launch("condense");
}

void launch_shift_cholesky(double* K, int n, int* info, double*, cudaStream_t st) {
  if (n <= kSmallChol) {
    cudaFuncSetAttribute(shift_cholesky_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(size_t(n) * n * sizeof(double)));
    shift_cholesky_small_kernel<<<1, kDenseBlock, size_t(n) * n * sizeof(double), st>>>(K, n, info);
    note_launch();
    check_launch("shift_cholesky");
  } else {
    launch_blocked_cholesky(K, n, info, st);  // DMMA trailing updates (dense_chol.cu)
  }
}

void launch_cholesky_solve(const double* L, int n, double* b, cudaStream_t st) {
  if (n <= 64)
    cholesky_solve_warp_kernel<2><<<1, 32, 0, st>>>(L, n, b);
  else if (n <= 128)
    cholesky_solve_warp_kernel<4><<<1, 32, 0, st>>>(L, n, b);
  else if (n <= 256)
    cholesky_solve_warp_kernel<8><<<1, 32, 0, st>>>(L, n, b);
  else {
    launch_blocked_solve(L, n, b, st);
    return;
  }
  note_launch();
  check_launch("cholesky_solve");
}

}  // namespace bipm
