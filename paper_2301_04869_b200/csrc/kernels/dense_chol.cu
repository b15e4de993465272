// Blocked dense Cholesky of the reduced matrix K_hat (n_u x n_u, column-major,
// lower) for n_u above the shared-memory kernel's range, with the trailing
// update on the FP64 tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA; tcgen05 has
// no f64 kind).
//
// Reference: factor_dense_sym -> LAPACKE_dpotrf('L') (linalg.cpp:129-145,
// lapack.cpp:26-31) after the 1e-13 max(1,|K|_inf) diagonal shift
// (kkt.cpp:965-968); a pivot that is not > 0 (or NaN) fails the factor, which
// is exactly when the reference's attempt is rejected (kkt.cpp:970-971).
//
// Per panel of kNb = 32 columns: (1) factor the diagonal block in shared
// memory, (2) L21 = A21 L11^{-T} row-parallel, (3) A22 -= L21 L21' on the lower
// triangle in 64 x 64 tiles, four warps of 32 x 32 DMMA fragments each.
#include <cooperative_groups.h>

#include <cmath>
#include <algorithm>
#include <stdexcept>
#include <string>

#include "kkt_kernels.hpp"
#include "stats.hpp"

namespace bipm {

namespace {

constexpr int kNb = 32;
constexpr int kTile = 64;

void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// |K|_inf then the diagonal shift; info reset
__global__ void shift_kernel(double* K, int n, int* info) {
  __shared__ double red[32];
  double mx = 0.0;
  for (long long i = threadIdx.x; i < (long long)n * n; i += blockDim.x) mx = fmax(mx, fabs(K[i]));
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double shift = 1e-13 * fmax(1.0, red[0]);
  for (int i = threadIdx.x; i < n; i += blockDim.x) K[size_t(i) * n + i] += shift;
  if (threadIdx.x == 0) {
    *info = 0;
    reinterpret_cast<double*>(info)[1] = red[0];  // |K|_inf
  }
}

// Cholesky of the w x w diagonal block held in one warp's registers (lane r
// holds row r, a[c] = A(r, c) for c <= r); each pivot's column L(:, j) is
// broadcast through a 32-double shared buffer (shuffles of a whole column
// would keep 31 doubles live per step and spill).  Padded to 32 x 32 with the
// identity so the loop is branch-free.  Returns 0, or 1 + the first failing
// column (pivot not > 0 or NaN).
__device__ __forceinline__ int warp_chol32(double (&a)[kNb], int w, int lane, double* colbuf,
                                           double* fail_pivot = nullptr) {
  if (lane >= w) {
#pragma unroll
    for (int c = 0; c < kNb; ++c) a[c] = (c == lane) ? 1.0 : 0.0;
  }
  int fail = 0;
#pragma unroll
  for (int j = 0; j < kNb; ++j) {
    const double ajj = __shfl_sync(0xffffffffu, a[j], j);
    const bool bad = !(ajj > 0.0) || isnan(ajj);
    if (fail == 0 && bad && fail_pivot) *fail_pivot = ajj;  // the value dpotrf rejects
    fail = (fail == 0 && bad) ? j + 1 : fail;
    // rsqrt (MUFU seed + Newton, ~1 ulp) instead of the IEEE sqrt and
    // division subroutines: they were ~2/3 of the serial per-column chain
    const double rd = rsqrt(bad ? 1.0 : ajj);
    const double d = (bad ? 1.0 : ajj) * rd;
    a[j] = lane == j ? d : (lane > j ? a[j] * rd : a[j]);  // L(r, j)
    colbuf[lane] = a[j];
    __syncwarp();
    // fixed trip count so both loops unroll completely and a[] stays in
    // registers (a j-dependent bound was unrolled by 8 only: a[] went to
    // local memory, ~900 cycles per column)
#pragma unroll
    for (int k = 0; k < kNb; ++k)
      if (k > j) a[k] = lane >= k ? a[k] - a[j] * colbuf[k] : a[k];
    __syncwarp();
  }
  return fail;
}

// (1) diagonal block [c0, c0+w), one warp, lane = row
__global__ void diag_factor_kernel(double* K, int n, int c0, int* info) {
  if (*info) return;
  const int w = min(kNb, n - c0), r = threadIdx.x;
  __shared__ double colbuf[kNb];
  double a[kNb];
#pragma unroll
  for (int c = 0; c < kNb; ++c)
    a[c] = (c < w && r < w && c <= r) ? K[size_t(c0 + c) * n + c0 + r] : 0.0;
  double piv = 0.0;
  const int fail = warp_chol32(a, w, r, colbuf, &piv);
  if (fail) {
    if (r == 0) {
      *info = c0 + fail;
      reinterpret_cast<double*>(info)[2] = piv;
    }
    return;
  }
#pragma unroll
  for (int c = 0; c < kNb; ++c)
    if (c < w && r < w && c <= r) K[size_t(c0 + c) * n + c0 + r] = a[c];
}

// (2) L21 = A21 L11^{-T}: one thread per row below the panel
__global__ void panel_trsm_kernel(double* K, int n, int c0, const int* info) {
  __shared__ double L[kNb][kNb + 1];
  if (*info) return;
  const int w = min(kNb, n - c0);
  for (int q = threadIdx.x; q < w * w; q += blockDim.x) {
    const int rr = q / w, cc = q % w;
    L[rr][cc] = cc <= rr ? K[size_t(c0 + cc) * n + c0 + rr] : 0.0;
  }
  __syncthreads();
  const int r = c0 + w + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[kNb];
#pragma unroll
  for (int j = 0; j < kNb; ++j) x[j] = j < w ? K[size_t(c0 + j) * n + r] : 0.0;
#pragma unroll
  for (int j = 0; j < kNb; ++j) {
    if (j >= w) break;
    double v = x[j];
#pragma unroll
    for (int k = 0; k < j; ++k) v -= x[k] * L[j][k];
    x[j] = v / L[j][j];
  }
#pragma unroll
  for (int j = 0; j < kNb; ++j)
    if (j < w) K[size_t(c0 + j) * n + r] = x[j];
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// (3) A22 -= L21 L21' on lower tiles (I >= J) of the trailing matrix
__global__ void __launch_bounds__(128) panel_update_kernel(double* K, int n, int c0,
                                                           const int* info) {
  __shared__ double sa[kTile][kNb + 1];
  __shared__ double sb[kTile][kNb + 1];
  if (*info) return;
  const int t0 = c0 + kNb;  // trailing start
  // lower-triangle tile enumeration: blockIdx.x -> (I, J), I >= J
  int I = int((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) / 2.0);
  while ((I + 1) * (I + 2) / 2 <= int(blockIdx.x)) ++I;
  while (I * (I + 1) / 2 > int(blockIdx.x)) --I;
  const int J = int(blockIdx.x) - I * (I + 1) / 2;
  const int r0 = t0 + I * kTile, s0 = t0 + J * kTile;
  for (int q = threadIdx.x; q < kTile * kNb; q += 128) {
    const int rr = q % kTile, kk = q / kTile;  // coalesced along rows
    const int ra = r0 + rr, rb = s0 + rr;
    sa[rr][kk] = ra < n ? K[size_t(c0 + kk) * n + ra] : 0.0;
    sb[rr][kk] = rb < n ? K[size_t(c0 + kk) * n + rb] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;  // warp sub-tile
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 4; ++b2) acc[a][b2][0] = acc[a][b2][1] = 0.0;
  const int gm = lane >> 2, gk = lane & 3;
#pragma unroll
  for (int k = 0; k < kNb; k += 4) {
    double af[4], bf[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) af[a] = sa[wm + a * 8 + gm][k + gk];
#pragma unroll
    for (int b2 = 0; b2 < 4; ++b2) bf[b2] = sb[wn + b2 * 8 + gm][k + gk];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2) dmma(acc[a][b2][0], acc[a][b2][1], af[a], bf[b2]);
  }
  // C fragment: row gm, cols 2*gk + {0,1}
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int r = r0 + wm + a * 8 + gm, c = s0 + wn + b2 * 8 + 2 * gk + v;
        if (r < n && c < n && c <= r) K[size_t(c) * n + r] -= acc[a][b2][v];
      }
}

// The whole blocked factorisation in one cooperative launch (no per-panel
// launch gaps): per panel, CTA 0 factors the diagonal block, the grid solves
// the panel rows, the grid updates the trailing lower tiles on DMMA; grid-wide
// barriers between the phases.  A failed pivot stops every CTA consistently.
__device__ long long* g_chol_stamps = nullptr;  // debug: per-panel phase clocks of CTA 0

__global__ void __launch_bounds__(128) cholesky_coop_kernel(double* K, int n, int* info) {
  namespace cg = cooperative_groups;
  long long* stamps = (blockIdx.x == 0 && threadIdx.x == 0) ? g_chol_stamps : nullptr;
  int ns = 0;
  auto stamp = [&] {
    if (stamps && ns < 256) stamps[ns++] = clock64();
  };
  cg::grid_group grid = cg::this_grid();
  __shared__ double buf[2 * kTile * (kNb + 1)];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // shift (kkt.cpp:965-968): |K|_inf over the grid, CTA 0 applies it
  {
    double mx = 0.0;
    for (long long i = blockIdx.x * 128LL + tid; i < (long long)n * n; i += gridDim.x * 128LL)
      mx = fmax(mx, fabs(K[i]));
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane == 0) buf[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double v = fmax(fmax(buf[0], buf[1]), fmax(buf[2], buf[3]));
      // max of non-negative doubles: compare as integers
      atomicMax(reinterpret_cast<unsigned long long*>(info) + 1,
                static_cast<unsigned long long>(__double_as_longlong(v)));
    }
  }
  grid.sync();
  if (blockIdx.x == 0) {
    const double kinf = __longlong_as_double(
        static_cast<long long>(reinterpret_cast<unsigned long long*>(info)[1]));
    const double shift = 1e-13 * fmax(1.0, kinf);
    for (int i = tid; i < n; i += 128) K[size_t(i) * n + i] += shift;
    if (tid == 0) info[0] = 0;
  }
  grid.sync();
  for (int c0 = 0; c0 < n; c0 += kNb) {
    const int w = min(kNb, n - c0);
    stamp();
    // (1) every CTA factors the diagonal block itself (warp 0; identical
    // inputs give an identical factor) into its shared-memory copy for the
    // panel solve, CTA 0 writes it back: no grid barrier between the factor
    // and the panel solve, and no reload of L11
    double(*L)[kNb + 1] = reinterpret_cast<double(*)[kNb + 1]>(buf);
    double* rdiag = buf + kNb * (kNb + 1);  // reciprocals of the diagonal
    __shared__ int fail_s;
    if (warp == 0) {
      const int r = lane;
      double a[kNb];
#pragma unroll
      for (int c = 0; c < kNb; ++c)
        a[c] = (c < w && r < w && c <= r) ? K[size_t(c0 + c) * n + c0 + r] : 0.0;
      stamp();
      double piv = 0.0;
      const int f = warp_chol32(a, w, r, rdiag + kNb, &piv);
      if (r == 0) fail_s = f;
      if (f) {
        if (blockIdx.x == 0 && r == 0) {
          info[0] = c0 + f;
          reinterpret_cast<double*>(info)[2] = piv;
        }
      } else {
#pragma unroll
        for (int c = 0; c < kNb; ++c) {
          const bool in = c < w && r < w && c <= r;
          L[r][c] = in ? a[c] : 0.0;
          if (in && blockIdx.x == 0) K[size_t(c0 + c) * n + c0 + r] = a[c];
        }
      }
    }
    stamp();
    __syncthreads();
    stamp();
    if (fail_s) return;  // every CTA reached the same verdict
    const int rows = n - c0 - w;
    if (rows <= 0) break;
    // (2) L21 = A21 L11^{-T}, one thread per row
    {
      if (tid < kNb) rdiag[tid] = tid < w ? 1.0 / L[tid][tid] : 1.0;
      __syncthreads();
      for (int rb = blockIdx.x * 128; rb < rows; rb += gridDim.x * 128) {
        const int r = c0 + w + rb + tid;
        if (r < n) {
          double x[kNb];
#pragma unroll
          for (int j = 0; j < kNb; ++j) x[j] = j < w ? K[size_t(c0 + j) * n + r] : 0.0;
          // column-oriented substitution: after x_j is final, every later
          // x_k is updated independently (one multiply-add deep per step);
          // L is zero-padded beyond w, rdiag to 1
#pragma unroll
          for (int j = 0; j < kNb; ++j) {
            x[j] *= rdiag[j];
#pragma unroll
            for (int k = 0; k < kNb; ++k)  // fixed trip count: full unroll, x in registers
              if (k > j) x[k] -= L[k][j] * x[j];
          }
#pragma unroll
          for (int j = 0; j < kNb; ++j)
            if (j < w) K[size_t(c0 + j) * n + r] = x[j];
        }
      }
    }
    stamp();
    grid.sync();
    stamp();
    // (3) A22 -= L21 L21' on the lower 64 x 64 tiles
    {
      double(*sa)[kNb + 1] = reinterpret_cast<double(*)[kNb + 1]>(buf);
      double(*sb)[kNb + 1] = reinterpret_cast<double(*)[kNb + 1]>(buf + kTile * (kNb + 1));
      const int t0 = c0 + kNb;
      const int nt = (rows + kTile - 1) / kTile;
      for (int tile = blockIdx.x; tile < nt * (nt + 1) / 2; tile += gridDim.x) {
        int I = int((sqrt(8.0 * tile + 1.0) - 1.0) / 2.0);
        while ((I + 1) * (I + 2) / 2 <= tile) ++I;
        while (I * (I + 1) / 2 > tile) --I;
        const int J = tile - I * (I + 1) / 2;
        const int r0 = t0 + I * kTile, s0 = t0 + J * kTile;
        __syncthreads();
        {
          // all 32 loads of this thread in flight, then the shared-memory stores
          constexpr int kPer = kTile * kNb / 128;
          double va[kPer], vb[kPer];
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            const int q = tid + u * 128, rr = q % kTile, kk = q / kTile;
            const int ra = r0 + rr, rb = s0 + rr;
            va[u] = ra < n ? K[size_t(c0 + kk) * n + ra] : 0.0;
            vb[u] = rb < n ? K[size_t(c0 + kk) * n + rb] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            const int q = tid + u * 128, rr = q % kTile, kk = q / kTile;
            sa[rr][kk] = va[u];
            sb[rr][kk] = vb[u];
          }
        }
        __syncthreads();
        const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
        double acc[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) acc[a][b2][0] = acc[a][b2][1] = 0.0;
        const int gm = lane >> 2, gk = lane & 3;
#pragma unroll
        for (int k = 0; k < kNb; k += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) af[a] = sa[wm + a * 8 + gm][k + gk];
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) bf[b2] = sb[wn + b2 * 8 + gm][k + gk];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) dmma(acc[a][b2][0], acc[a][b2][1], af[a], bf[b2]);
        }
        // read-modify-write of the tile: all 32 loads in flight first
        double old[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int r = r0 + wm + a * 8 + gm, c = s0 + wn + b2 * 8 + 2 * gk + v;
              old[a][b2][v] = (r < n && c < n && c <= r) ? K[size_t(c) * n + r] : 0.0;
            }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int r = r0 + wm + a * 8 + gm, c = s0 + wn + b2 * 8 + 2 * gk + v;
              if (r < n && c < n && c <= r) K[size_t(c) * n + r] = old[a][b2][v] - acc[a][b2][v];
            }
      }
    }
    stamp();
    grid.sync();
  }
}

// L L' x = b, blocked by 32 rows.  Per block: one warp solves the 32 x 32
// diagonal block by shuffles (rows / columns in registers, reciprocal pivots),
// then the CTA updates the remaining rows.  Nothing the CTA loads from L
// depends on x, so each thread issues its row's 32 loads of the coming update
// and the next diagonal block's entries (double-buffered in shared memory)
// before the warp solve: the L2 latency hides behind the solve and each block
// costs a solve plus two barriers.  L is L2-resident after the factorisation.
template <int B>
__global__ void __launch_bounds__(B) blocked_solve_kernel(const double* __restrict__ L, int n,
                                                         double* b) {
  extern __shared__ double x[];     // n + 32 (zero padding for the last block)
  __shared__ double Dg[2][32][33];  // diagonal blocks, Dg[.][r][c] = L(c0 + r, c0 + c)
  constexpr int kDg = (1024 + B - 1) / B;  // block entries per thread
  for (int i = threadIdx.x; i < n + 32; i += B) x[i] = i < n ? b[i] : 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (n + 31) / 32;
  // entry e = (r, c) of block k: L(c0 + r, c0 + c), identity padding
  auto dg_load = [&](int k, double (&v)[kDg]) {
#pragma unroll
    for (int q = 0; q < kDg; ++q) {
      const int e = threadIdx.x + q * B, r = e & 31, c = e >> 5, c0 = 32 * k;
      const int w = min(32, n - c0);
      v[q] = (e < 1024 && k >= 0 && k < nb) ? ((r < w && c < w) ? L[size_t(c0 + c) * n + c0 + r]
                                                                 : (r == c ? 1.0 : 0.0))
                                            : 0.0;
    }
  };
  auto dg_store = [&](int buf, const double (&v)[kDg]) {
#pragma unroll
    for (int q = 0; q < kDg; ++q) {
      const int e = threadIdx.x + q * B;
      if (e < 1024) Dg[buf][e & 31][e >> 5] = v[q];
    }
  };
  double v[kDg];
  dg_load(0, v);
  dg_store(0, v);
  __syncthreads();
  for (int k = 0; k < nb; ++k) {  // forward: L y = b
    const int c0 = 32 * k, w = min(32, n - c0), buf = k & 1;
    const int i0 = c0 + w + threadIdx.x;  // first row of the update, prefetched
    double l[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) l[j] = (i0 < n && j < w) ? L[size_t(c0 + j) * n + i0] : 0.0;
    dg_load(k + 1, v);
    if (warp == 0) {
      const double* row = Dg[buf][lane];
      const double rd = 1.0 / Dg[buf][lane][lane];
      double xv = x[c0 + lane];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double xj = __shfl_sync(0xffffffffu, xv * rd, j);
        if (lane == j) xv = xj;
        if (lane > j) xv -= row[j] * xj;
      }
      if (lane < w) x[c0 + lane] = xv;
    }
    dg_store(buf ^ 1, v);
    __syncthreads();
    for (int i = i0; i < n; i += B) {
      if (i != i0)
#pragma unroll
        for (int j = 0; j < 32; ++j) l[j] = j < w ? L[size_t(c0 + j) * n + i] : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += l[j] * x[c0 + j];
      x[i] -= acc;
    }
    __syncthreads();
  }
  dg_load(nb - 1, v);
  dg_store(0, v);
  __syncthreads();
  for (int k = nb - 1, t = 0; k >= 0; --k, ++t) {  // backward: L' x = y
    const int c0 = 32 * k, w = min(32, n - c0), buf = t & 1;
    const int i0 = threadIdx.x;  // rows i < c0
    double l[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) l[j] = (i0 < c0 && j < w) ? L[size_t(i0) * n + c0 + j] : 0.0;
    dg_load(k - 1, v);
    if (warp == 0) {
      const double rd = 1.0 / Dg[buf][lane][lane];
      double xv = x[c0 + lane];
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        const double xj = __shfl_sync(0xffffffffu, xv * rd, j);
        if (lane == j) xv = xj;
        if (lane < j) xv -= Dg[buf][j][lane] * xj;
      }
      if (lane < w) x[c0 + lane] = xv;
    }
    dg_store(buf ^ 1, v);
    __syncthreads();
    for (int i = i0; i < c0; i += B) {
      if (i != i0)
#pragma unroll
        for (int j = 0; j < 32; ++j) l[j] = j < w ? L[size_t(i) * n + c0 + j] : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += l[j] * x[c0 + j];
      x[i] -= acc;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += B) b[i] = x[i];
}

}  // namespace

void launch_blocked_cholesky(double* K, int n, int* info, cudaStream_t st) {
  // one cooperative launch when the grid fits co-resident (info holds two
  // 8-byte slots: the status and the |K|_inf scratch)
  static int coop_blocks = -1;
  if (coop_blocks < 0) {
    int dev = 0, sms = 0, per = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cholesky_coop_kernel, 128, 0);
    coop_blocks = coop ? sms * per : 0;
  }
  const int rows0 = n - kNb;
  const int nt0 = (rows0 + kTile - 1) / kTile;
  const int want = std::max(nt0 * (nt0 + 1) / 2, (rows0 + 127) / 128);
  const int grid = std::min(want, coop_blocks);
  if (grid >= 1 && coop_blocks > 0) {
    cudaMemsetAsync(info, 0, 16, st);
    void* args[] = {&K, &n, &info};
    const cudaError_t e = cudaLaunchCooperativeKernel(
        reinterpret_cast<void*>(cholesky_coop_kernel), dim3(grid), dim3(128), args, 0, st);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cholesky_coop: ") + cudaGetErrorString(e));
    note_launch();
    return;
  }
  shift_kernel<<<1, 1024, 0, st>>>(K, n, info);
  note_launch();
  for (int c0 = 0; c0 < n; c0 += kNb) {
    diag_factor_kernel<<<1, kNb, 0, st>>>(K, n, c0, info);
    const int rows = n - c0 - kNb;
    if (rows > 0) {
      panel_trsm_kernel<<<(rows + 127) / 128, 128, 0, st>>>(K, n, c0, info);
      const int nt = (rows + kTile - 1) / kTile;
      panel_update_kernel<<<nt * (nt + 1) / 2, 128, 0, st>>>(K, n, c0, info);
      note_launch(3);
    } else {
      note_launch(1);
    }
  }
  check("blocked_cholesky");
}

void launch_blocked_solve(const double* L, int n, double* b, cudaStream_t st) {
  const size_t smem = size_t(n + 32) * sizeof(double);
  // 640 threads: one prefetched update row per thread up to n = 640 (more
  // rows are loaded after the barrier), <= 102 registers so l[32] stays in them
  cudaFuncSetAttribute(blocked_solve_kernel<640>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  blocked_solve_kernel<640><<<1, 640, smem, st>>>(L, n, b);
  note_launch();
  check("blocked_solve");
}

}  // namespace bipm
