// Bunch-Kaufman LDL' of the reduced matrix K_hat: the inertia half of the
// reference's DenseSymFactor (linalg.cpp:129-159).
//
// The reference factors the shifted K_hat with dpotrf and, only when that
// fails, with dsytrf (Bunch-Kaufman, lower) and accepts the attempt iff the
// D blocks report neg = 0 and zero = 0 (bunch_kaufman_inertia,
// lapack.cpp:55-97; kkt.cpp:969-971).  In exact arithmetic a failed Cholesky
// means K_hat is not positive definite, so both verdicts agree; they can
// differ only when the failing pivot is within rounding of zero.  The engine
// runs this factorisation exactly then (engine.cu, factor_khat) and solves
// with it when it reports a positive definite matrix.
//
// bk_factor_kernel follows LAPACK dsytf2 ('L') step for step (alpha =
// (1 + sqrt(17)) / 8, first-maximum pivot search, symmetric interchanges,
// rank-1 / rank-2 updates) as one cooperative launch: CTA 0 runs the pivot
// search and the interchange, the grid the trailing update, two grid barriers
// per pivot step.  bk_solve_kernel is dsytrs ('L').  Both are rare-path
// kernels (one call per borderline attempt), not tuned.
#include <cooperative_groups.h>

#include <cmath>
#include <stdexcept>
#include <string>

#include "kkt_kernels.hpp"
#include "stats.hpp"

namespace bipm {

namespace {

namespace cg = cooperative_groups;
constexpr int kBkThreads = 256;

__device__ __forceinline__ double& at(double* A, int n, int i, int j) {
  return A[size_t(j) * n + i];
}

// first index of the maximum |x| over [b, e) with stride (IDAMAX), block-wide
// (CTA 0 only); returns (index, value)
__device__ void block_argmax(const double* A, int n, int b, int e, bool row, int fixed,
                             int* out_i, double* out_v, double* sv, int* si) {
  const int tid = threadIdx.x;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int t = b + tid; t < e; t += kBkThreads) {
    const double v = fabs(row ? A[size_t(t) * n + fixed] : A[size_t(fixed) * n + t]);
    if (v > best || (v == best && t < bi)) best = v, bi = t;
  }
  sv[tid] = best;
  si[tid] = bi;
  __syncthreads();
  for (int s = kBkThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double v = sv[tid + s];
      const int i = si[tid + s];
      if (v > sv[tid] || (v == sv[tid] && i < si[tid])) sv[tid] = v, si[tid] = i;
    }
    __syncthreads();
  }
  *out_i = si[0];
  *out_v = sv[0];
  __syncthreads();
}

// state shared through global memory between the grid phases
struct BkState {
  int k, kstep, kp, skip, info;
  double kinf;
};

__global__ void __launch_bounds__(kBkThreads) bk_factor_kernel(double* A, int n, int* ipiv,
                                                              BkState* st, int* inertia) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[kBkThreads];
  __shared__ int si[kBkThreads];
  const int tid = threadIdx.x;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  // shift 1e-13 max(1, |K|_inf) (kkt.cpp:965-968), as the Cholesky path
  if (blockIdx.x == 0) {
    double mx = 0.0;
    for (long long q = tid; q < (long long)n * n; q += kBkThreads) mx = fmax(mx, fabs(A[q]));
    sv[tid] = mx;
    __syncthreads();
    for (int s = kBkThreads / 2; s > 0; s >>= 1) {
      if (tid < s) sv[tid] = fmax(sv[tid], sv[tid + s]);
      __syncthreads();
    }
    const double shift = 1e-13 * fmax(1.0, sv[0]);
    for (int i = tid; i < n; i += kBkThreads) at(A, n, i, i) += shift;
    if (tid == 0) {
      st->k = 0;
      st->info = 0;
      st->kinf = sv[0];
    }
  }
  grid.sync();
  for (;;) {
    const int k = st->k;
    if (k >= n) break;
    // ---- pivot choice and interchange (CTA 0)
    if (blockIdx.x == 0) {
      int kstep = 1, kp = k, skip = 0;
      const double absakk = fabs(at(A, n, k, k));
      int imax = k;
      double colmax = 0.0;
      if (k < n - 1) block_argmax(A, n, k + 1, n, false, k, &imax, &colmax, sv, si);
      if (fmax(absakk, colmax) == 0.0 || isnan(absakk)) {
        if (tid == 0 && st->info == 0) st->info = k + 1;
        kp = k;
        skip = 1;  // dsytf2: zero column, no interchange and no update
      } else if (absakk >= alpha * colmax) {
        kp = k;
      } else {
        int jmax;
        double rowmax;
        block_argmax(A, n, k, imax, true, imax, &jmax, &rowmax, sv, si);  // row imax, cols k..imax-1
        if (imax < n - 1) {
          double r2;
          block_argmax(A, n, imax + 1, n, false, imax, &jmax, &r2, sv, si);
          rowmax = fmax(rowmax, r2);
        }
        if (absakk >= alpha * colmax * (colmax / rowmax))
          kp = k;
        else if (fabs(at(A, n, imax, imax)) >= alpha * rowmax)
          kp = imax;
        else
          kp = imax, kstep = 2;
      }
      const int kk = k + kstep - 1;
      if (kp != kk && !skip) {
        for (int i = kp + 1 + tid; i < n; i += kBkThreads) {  // A(kp+1:n, kk) <-> A(kp+1:n, kp)
          const double t = at(A, n, i, kk);
          at(A, n, i, kk) = at(A, n, i, kp);
          at(A, n, i, kp) = t;
        }
        for (int j = kk + 1 + tid; j < kp; j += kBkThreads) {  // A(kk+1:kp-1, kk) <-> A(kp, kk+1:kp-1)
          const double t = at(A, n, j, kk);
          at(A, n, j, kk) = at(A, n, kp, j);
          at(A, n, kp, j) = t;
        }
        if (tid == 0) {
          double t = at(A, n, kk, kk);
          at(A, n, kk, kk) = at(A, n, kp, kp);
          at(A, n, kp, kp) = t;
          if (kstep == 2) {
            t = at(A, n, k + 1, k);
            at(A, n, k + 1, k) = at(A, n, kp, k);
            at(A, n, kp, k) = t;
          }
        }
      }
      if (tid == 0) {
        st->kstep = kstep;
        st->kp = kp;
        st->skip = skip;
        if (kstep == 1) {
          ipiv[k] = kp + 1;
        } else {
          ipiv[k] = -(kp + 1);
          ipiv[k + 1] = -(kp + 1);
        }
      }
    }
    grid.sync();
    // ---- trailing update (grid): columns j > k(+1), rows i >= j
    const int kstep = st->kstep;
    const bool skip = st->skip != 0;
    const int warps = gridDim.x * (kBkThreads / 32);
    const int gw = blockIdx.x * (kBkThreads / 32) + (tid >> 5), lane = tid & 31;
    if (skip) {
    } else if (kstep == 1) {
      if (k < n - 1) {
        const double d11 = 1.0 / at(A, n, k, k);
        // dsyr: A(i,j) += x(i) * (-d11 x(j)), x = A(k+1:n, k) (original)
        for (int j = k + 1 + gw; j < n; j += warps) {
          const double temp = -d11 * at(A, n, j, k);
          for (int i = j + lane; i < n; i += 32) at(A, n, i, j) += at(A, n, i, k) * temp;
        }
      }
    } else if (k < n - 2) {
      double d21 = at(A, n, k + 1, k);
      const double d11 = at(A, n, k + 1, k + 1) / d21;
      const double d22 = at(A, n, k, k) / d21;
      const double t = 1.0 / (d11 * d22 - 1.0);
      d21 = t / d21;
      for (int j = k + 2 + gw; j < n; j += warps) {
        const double wk = d21 * (d11 * at(A, n, j, k) - at(A, n, j, k + 1));
        const double wkp1 = d21 * (d22 * at(A, n, j, k + 1) - at(A, n, j, k));
        for (int i = j + lane; i < n; i += 32)
          at(A, n, i, j) = at(A, n, i, j) - at(A, n, i, k) * wk - at(A, n, i, k + 1) * wkp1;
      }
    }
    grid.sync();
    // ---- scale the pivot column(s) (grid: every update read the originals)
    if (skip) {
    } else if (kstep == 1) {
      if (k < n - 1) {
        const double d11 = 1.0 / at(A, n, k, k);
        for (int i = k + 1 + blockIdx.x * kBkThreads + tid; i < n; i += gridDim.x * kBkThreads)
          at(A, n, i, k) *= d11;
      }
    } else if (k < n - 2) {
      double d21 = at(A, n, k + 1, k);
      const double d11 = at(A, n, k + 1, k + 1) / d21;
      const double d22 = at(A, n, k, k) / d21;
      const double t = 1.0 / (d11 * d22 - 1.0);
      d21 = t / d21;
      for (int j = k + 2 + blockIdx.x * kBkThreads + tid; j < n; j += gridDim.x * kBkThreads) {
        const double ajk = at(A, n, j, k), ajk1 = at(A, n, j, k + 1);
        at(A, n, j, k) = d21 * (d11 * ajk - ajk1);
        at(A, n, j, k + 1) = d21 * (d22 * ajk1 - ajk);
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) st->k = k + kstep;
    grid.sync();
  }
  // inertia of D (bunch_kaufman_inertia, lapack.cpp:55-97)
  if (blockIdx.x == 0 && tid == 0) {
    int np = 0, nn = 0, nz = 0;
    for (int k = 0; k < n;) {
      if (ipiv[k] > 0) {
        const double d = at(A, n, k, k);
        if (d > 0)
          ++np;
        else if (d < 0)
          ++nn;
        else
          ++nz;
        ++k;
      } else {
        const double a = at(A, n, k, k), c = at(A, n, k + 1, k + 1), b = at(A, n, k + 1, k);
        const double det = a * c - b * b;
        if (det < 0) {
          ++np;
          ++nn;
        } else if (det > 0) {
          if (a + c > 0)
            np += 2;
          else
            nn += 2;
        } else {
          ++nz;
          if (a + c > 0)
            ++np;
          else if (a + c < 0)
            ++nn;
          else
            ++nz;
        }
        k += 2;
      }
    }
    // an exactly zero pivot (dsytrf info > 0): the reference throws; counted
    // as a zero eigenvalue here, which rejects the attempt
    if (st->info != 0 && nz == 0) nz = 1;
    inertia[0] = np;
    inertia[1] = nn;
    inertia[2] = nz;
  }
}

// dsytrs ('L'), one right-hand side, one CTA
__global__ void __launch_bounds__(1024) bk_solve_kernel(const double* __restrict__ A, int n,
                                                        const int* __restrict__ ipiv, double* b) {
  __shared__ double red[32];
  __shared__ double bk_s[2];
  const int tid = threadIdx.x;
  auto swap = [&](int p, int q) {
    if (tid == 0 && p != q) {
      const double t = b[p];
      b[p] = b[q];
      b[q] = t;
    }
    __syncthreads();
  };
  auto dot = [&](int col, int from) {  // sum_{i >= from} A(i, col) b(i), block-wide
    double v = 0.0;
    for (int i = from + tid; i < n; i += 1024) v += A[size_t(col) * n + i] * b[i];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (tid == 0)
      for (int w = 0; w < 32; ++w) s += red[w];
    __syncthreads();
    return s;  // valid on thread 0
  };
  // L D x = P b
  for (int k = 0; k < n;) {
    if (ipiv[k] > 0) {
      swap(k, ipiv[k] - 1);
      const double bk = b[k];
      for (int i = k + 1 + tid; i < n; i += 1024) b[i] -= A[size_t(k) * n + i] * bk;
      __syncthreads();
      if (tid == 0) b[k] /= A[size_t(k) * n + k];
      __syncthreads();
      ++k;
    } else {
      swap(k + 1, -ipiv[k] - 1);
      const double b0 = b[k], b1 = b[k + 1];
      for (int i = k + 2 + tid; i < n; i += 1024)
        b[i] -= A[size_t(k) * n + i] * b0 + A[size_t(k + 1) * n + i] * b1;
      __syncthreads();
      if (tid == 0) {
        const double akm1k = A[size_t(k) * n + k + 1];
        const double akm1 = A[size_t(k) * n + k] / akm1k;
        const double ak = A[size_t(k + 1) * n + k + 1] / akm1k;
        const double denom = akm1 * ak - 1.0;
        const double bkm1 = b0 / akm1k, bk = b1 / akm1k;
        b[k] = (ak * bkm1 - bk) / denom;
        b[k + 1] = (akm1 * bk - bkm1) / denom;
      }
      __syncthreads();
      k += 2;
    }
  }
  // L' x = y, then P'
  for (int k = n - 1; k >= 0;) {
    if (ipiv[k] > 0) {
      if (k < n - 1) {
        const double s = dot(k, k + 1);
        if (tid == 0) b[k] -= s;
        __syncthreads();
      }
      swap(k, ipiv[k] - 1);
      --k;
    } else {
      if (k < n - 1) {
        const double s1 = dot(k, k + 1);
        if (tid == 0) bk_s[0] = s1;
        __syncthreads();
        const double s0 = dot(k - 1, k + 1);
        if (tid == 0) {
          b[k] -= bk_s[0];
          b[k - 1] -= s0;
        }
        __syncthreads();
      }
      swap(k, -ipiv[k] - 1);
      k -= 2;
    }
  }
}

void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

size_t bk_work_bytes(int n) { return sizeof(BkState) + size_t(n) * sizeof(int) + 16; }

void launch_bk_factor(double* K, int n, int* ipiv, void* state, int* inertia, cudaStream_t st) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk_factor_kernel, kBkThreads, 0);
  const int want = std::max(1, (n * (n + 1) / 2 + 32 * 256 - 1) / (32 * 256));
  int grid = std::min(sms * std::max(1, per), want);
  grid = std::max(1, grid);
  BkState* s = static_cast<BkState*>(state);
  void* args[] = {&K, &n, &ipiv, &s, &inertia};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bk_factor_kernel),
                                                    dim3(grid), dim3(kBkThreads), args, 0, st);
  if (e != cudaSuccess) throw std::runtime_error(std::string("bk_factor: ") + cudaGetErrorString(e));
  note_launch();
}

void launch_bk_solve(const double* F, int n, const int* ipiv, double* b, cudaStream_t st) {
  bk_solve_kernel<<<1, 1024, 0, st>>>(F, n, ipiv, b);
  note_launch();
  check("bk_solve");
}

}  // namespace bipm
