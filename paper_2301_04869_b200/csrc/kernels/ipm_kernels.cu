// Interior-point vector kernels (see ipm_kernels.hpp for the reference map).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "ipm_kernels.hpp"

#include "stats.hpp"

namespace bipm {

namespace {

constexpr int kB = 256;
constexpr int kMaxBlocks = 592;  // 4 x 148 SMs; reductions are grid-stride

__device__ __forceinline__ double combine(int op, double a, double b) {
  return op == kSum ? a + b : (op == kMax ? fmax(a, b) : fmin(a, b));
}
__device__ __forceinline__ double ident(int op) {
  return op == kSum ? 0.0 : (op == kMax ? -INFINITY : INFINITY);
}

// Block-level reduction of K accumulators into partial[blockIdx.x][K].
template <int K>
__device__ void block_partial(double (&v)[K], const int (&op)[K], double* partial) {
  __shared__ double sh[K][kB / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int off = 16; off > 0; off >>= 1)
      v[k] = combine(op[k], v[k], __shfl_xor_sync(0xffffffffu, v[k], off));
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k][warp] = v[k];
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double a = ident(op[k]);
    for (int w = 0; w < kB / 32; ++w) a = combine(op[k], a, sh[k][w]);
    partial[size_t(blockIdx.x) * K + k] = a;
  }
}

// one warp per slot: lane-strided partials, then a fixed xor tree (deterministic)
template <int K>
__global__ void finalize_kernel(const double* partial, int nblocks, const int* ops_unused,
                                double* out, int o0, int o1, int o2, int o3, int o4, int o5,
                                int o6, int o7) {
  const int ops[8] = {o0, o1, o2, o3, o4, o5, o6, o7};
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= K) return;
  const int op = ops[k];
  double a = ident(op);
  for (int b = lane; b < nblocks; b += 32) a = combine(op, a, partial[size_t(b) * K + k]);
  for (int off = 16; off > 0; off >>= 1) a = combine(op, a, __shfl_xor_sync(0xffffffffu, a, off));
  if (lane == 0) out[k] = a;
}

// Same reduction written to dst[0..K) (single-block use).
template <int K>
__device__ void block_reduce_to(double (&v)[K], const int (&op)[K], double* dst) {
  __shared__ double sh2[K][kB / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int off = 16; off > 0; off >>= 1)
      v[k] = combine(op[k], v[k], __shfl_xor_sync(0xffffffffu, v[k], off));
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh2[k][warp] = v[k];
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double a = ident(op[k]);
    for (int w = 0; w < kB / 32; ++w) a = combine(op[k], a, sh2[k][w]);
    dst[k] = a;
  }
}

template <int K>
void finalize(const double* partial, int nblocks, const int (&op)[K], double* out,
              cudaStream_t st) {
  int o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < K; ++k) o[k] = op[k];
  finalize_kernel<K><<<1, 32 * K, 0, st>>>(partial, nblocks, nullptr, out, o[0], o[1], o[2], o[3],
                                       o[4], o[5], o[6], o[7]);
  note_launch();
}

int red_blocks(long long n) {
  long long b = (n + kB - 1) / kB;
  if (b < 1) b = 1;
  return int(b < kMaxBlocks ? b : kMaxBlocks);
}
int ew_blocks(long long n) { return int((n + kB - 1) / kB > 0 ? (n + kB - 1) / kB : 1); }

void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// -------------------------------------------------------------- residuals
__global__ void __launch_bounds__(kB) kkt_error_xs_kernel(IpmDims d, DevIter it, DevBounds b,
                                                          const double* grad, const double* g,
                                                          const double* h, double mu,
                                                          double* partial) {
  constexpr int ops[6] = {kMax, kMax, kMax, kMax, kMax, kSum};
  double v[6] = {0, 0, 0, 0, 0, 0};
  const long long nx = (long long)d.M * d.n_x, ns = (long long)d.M * d.m;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < nx + ns;
       id += (long long)gridDim.x * kB) {
    if (id < nx) {
      const int s = int(id / d.n_x), i = int(id % d.n_x);
      const double lo = b.xlo[i], up = b.xup[i], xv = it.x[id];
      const double sx = grad[size_t(s) * d.n_d + i] - it.klo[id] + it.kup[id];
      v[0] = fmax(v[0], fabs(sx));
      v[2] = fmax(v[2], fabs(g[id]));
      if (isfinite(lo)) v[4] = fmax(v[4], fabs((xv - lo) * it.klo[id] - mu));
      if (isfinite(up)) v[4] = fmax(v[4], fabs((up - xv) * it.kup[id] - mu));
      v[5] += fabs(it.y[id]);
      if (isfinite(lo)) v[5] += fabs(it.klo[id]);
      if (isfinite(up)) v[5] += fabs(it.kup[id]);
    } else {
      const long long k = id - nx;
      const int i = int(k % d.m);
      const double lo = b.slo[i], up = b.sup[i], sv = it.s[k];
      v[1] = fmax(v[1], fabs(it.z[k] - it.nlo[k] + it.nup[k]));
      v[3] = fmax(v[3], fabs(h[k] + sv));
      if (isfinite(lo)) v[4] = fmax(v[4], fabs((sv - lo) * it.nlo[k] - mu));
      if (isfinite(up)) v[4] = fmax(v[4], fabs((up - sv) * it.nup[k] - mu));
      v[5] += fabs(it.z[k]);
      if (isfinite(lo)) v[5] += fabs(it.nlo[k]);
      if (isfinite(up)) v[5] += fabs(it.nup[k]);
    }
  }
  block_partial<6>(v, ops, partial);
}

constexpr int kEvalXs = 11;
__global__ void __launch_bounds__(kB) kkt_eval_kernel(IpmDims d, DevIter it, DevBounds b,
                                                      const double* grad, const double* g,
                                                      const double* h, const double* f,
                                                      const int* bad, int lo,
                                                      const double* gsum, double mu0, double mu1,
                                                      double mu2, double mu3, double* partial,
                                                      unsigned int* counter, double* out) {
  constexpr int ops[kEvalXs] = {kMax, kMax, kMax, kMax, kMax, kMax, kMax, kMax, kSum, kSum, kMin};
  const double mus[4] = {mu0, mu1, mu2, mu3};
  double v[kEvalXs] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1e300};
  const long long nx = (long long)d.M * d.n_x, ns = (long long)d.M * d.m;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < nx + ns + d.M;
       id += (long long)gridDim.x * kB) {
    if (id < nx) {
      const int s = int(id / d.n_x), i = int(id % d.n_x);
      const double lo_ = b.xlo[i], up = b.xup[i], xv = it.x[id];
      v[0] = fmax(v[0], fabs(grad[size_t(s) * d.n_d + i] - it.klo[id] + it.kup[id]));
      v[2] = fmax(v[2], fabs(g[id]));
      v[8] += fabs(it.y[id]);
      if (isfinite(lo_)) {
        const double p = (xv - lo_) * it.klo[id];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[4 + k] = fmax(v[4 + k], fabs(p - mus[k]));
        v[8] += fabs(it.klo[id]);
      }
      if (isfinite(up)) {
        const double p = (up - xv) * it.kup[id];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[4 + k] = fmax(v[4 + k], fabs(p - mus[k]));
        v[8] += fabs(it.kup[id]);
      }
    } else if (id < nx + ns) {
      const long long q = id - nx;
      const int i = int(q % d.m);
      const double lo_ = b.slo[i], up = b.sup[i], sv = it.s[q];
      v[1] = fmax(v[1], fabs(it.z[q] - it.nlo[q] + it.nup[q]));
      v[3] = fmax(v[3], fabs(h[q] + sv));
      v[8] += fabs(it.z[q]);
      if (isfinite(lo_)) {
        const double p = (sv - lo_) * it.nlo[q];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[4 + k] = fmax(v[4 + k], fabs(p - mus[k]));
        v[8] += fabs(it.nlo[q]);
      }
      if (isfinite(up)) {
        const double p = (up - sv) * it.nup[q];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[4 + k] = fmax(v[4 + k], fabs(p - mus[k]));
        v[8] += fabs(it.nup[q]);
      }
    } else {
      const int s = int(id - nx - ns);
      v[9] += f[s];
      if (bad && bad[s]) v[10] = fmin(v[10], double(lo + s));
    }
  }
  block_partial<kEvalXs>(v, ops, partial);
  // last block: fixed-order combination of the partials, then the u part
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < kEvalXs; k += kB / 32) {
    const int op = ops[k];
    double a = ident(op);
    for (int blk = lane; blk < int(gridDim.x); blk += 32)
      a = combine(op, a, ((volatile double*)partial)[size_t(blk) * kEvalXs + k]);
    for (int off = 16; off > 0; off >>= 1) a = combine(op, a, __shfl_xor_sync(0xffffffffu, a, off));
    if (lane == 0) out[k] = a;
  }
  constexpr int uops[6] = {kMax, kMax, kMax, kMax, kMax, kSum};
  double u[6] = {0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < d.n_u; i += kB) {
    const double lo_ = b.ulo[i], up = b.uup[i], uv = it.u[i];
    u[0] = fmax(u[0], fabs(gsum[i] + (-it.llo[i] + it.lup[i])));
    if (isfinite(lo_)) {
      const double p = (uv - lo_) * it.llo[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[1 + k] = fmax(u[1 + k], fabs(p - mus[k]));
      u[5] += fabs(it.llo[i]);
    }
    if (isfinite(up)) {
      const double p = (up - uv) * it.lup[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[1 + k] = fmax(u[1 + k], fabs(p - mus[k]));
      u[5] += fabs(it.lup[i]);
    }
  }
  __syncthreads();
  block_reduce_to<6>(u, uops, out + 11);
  if (threadIdx.x == 0) *counter = 0u;  // reusable
}

// a + x[0] + x[ld] + ... + x[(M-1) ld], added in scenario order (the
// reference's sequential sums), with 32 loads in flight: the plain loop kept
// four in flight and waited ~8 memory latencies per 32 scenarios (1354/256:
// 30 us per 519-control sum, three a step)
__device__ __forceinline__ double ordered_scenario_sum(const double* __restrict__ x, long long ld,
                                                       int M, double a) {
  int s = 0;
  for (; s + 32 <= M; s += 32) {
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = x[size_t(s + k) * ld];
#pragma unroll
    for (int k = 0; k < 32; ++k) a += v[k];
  }
  for (; s < M; ++s) a += x[size_t(s) * ld];
  return a;
}

__global__ void grad_u_sum_kernel(IpmDims d, const double* grad, double* gsum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n_u) return;
  gsum[i] = ordered_scenario_sum(grad + d.n_x + i, d.n_d, d.M, 0.0);
}

__global__ void __launch_bounds__(kB) kkt_error_u_kernel(IpmDims d, DevIter it, DevBounds b,
                                                         const double* gsum, double mu,
                                                         double* out) {
  constexpr int ops[3] = {kMax, kMax, kSum};
  double v[3] = {0, 0, 0};
  for (int i = threadIdx.x; i < d.n_u; i += kB) {
    const double lo = b.ulo[i], up = b.uup[i], uv = it.u[i];
    v[0] = fmax(v[0], fabs(gsum[i] + (-it.llo[i] + it.lup[i])));
    if (isfinite(lo)) {
      v[1] = fmax(v[1], fabs((uv - lo) * it.llo[i] - mu));
      v[2] += fabs(it.llo[i]);
    }
    if (isfinite(up)) {
      v[1] = fmax(v[1], fabs((up - uv) * it.lup[i] - mu));
      v[2] += fabs(it.lup[i]);
    }
  }
  block_partial<3>(v, ops, out);
}

// ------------------------------------------------------ augmented system
__device__ __forceinline__ bool bound_terms(double v, double lo, double up, double mlo,
                                            double mup, double mu, double& sig, double& r) {
  bool ok = true;
  if (isfinite(lo)) {
    const double sl = v - lo;
    if (!(sl > 0)) ok = false;
    sig += mlo / sl;
    r -= mu / sl;
  }
  if (isfinite(up)) {
    const double su = up - v;
    if (!(su > 0)) ok = false;
    sig += mup / su;
    r += mu / su;
  }
  return ok;
}

__global__ void assemble_xs_kernel(IpmDims d, DevIter it, DevBounds b, const double* grad,
                                   const double* h, double mu, double* sigma_x, double* r1x,
                                   double* sigma_s, double* r2, double* r4, int* flag) {
  const long long nx = (long long)d.M * d.n_x, ns = (long long)d.M * d.m;
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id >= nx + ns) return;
  if (id < nx) {
    const int s = int(id / d.n_x), i = int(id % d.n_x);
    double sig = 0.0, r = grad[size_t(s) * d.n_d + i];
    if (!bound_terms(it.x[id], b.xlo[i], b.xup[i], it.klo[id], it.kup[id], mu, sig, r)) *flag = 1;
    sigma_x[id] = sig;
    r1x[id] = r;
  } else {
    const long long k = id - nx;
    const int i = int(k % d.m);
    double sig = 0.0, r = it.z[k];
    if (!bound_terms(it.s[k], b.slo[i], b.sup[i], it.nlo[k], it.nup[k], mu, sig, r)) *flag = 1;
    if (!(sig > 0)) *flag = 1;  // condense: Sigma_s must be positive (kkt.cpp:140-143)
    sigma_s[k] = sig;
    r2[k] = r;
    r4[k] = h[k] + it.s[k];
  }
}

__global__ void assemble_u_kernel(IpmDims d, DevIter it, DevBounds b, const double* gsum,
                                  double mu, double* sigma_u, double* r1u, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n_u) return;
  double sig = 0.0, r = 0.0;
  if (!bound_terms(it.u[i], b.ulo[i], b.uup[i], it.llo[i], it.lup[i], mu, sig, r)) *flag = 1;
  sigma_u[i] = 0.0 + sig;
  r1u[i] = gsum[i] + r;
}

__global__ void condensed_rhs_kernel(IpmDims d, DevCsr hx, DevCsr hu, const double* hxv,
                                     const double* huv, const double* sigma_s, const double* r4,
                                     const double* r2, const double* r1x, double* rhat1,
                                     double* part_u) {
  const int per = d.n_x + d.n_u;
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id >= (long long)d.M * per) return;
  const int s = int(id / per), c = int(id % per);
  const size_t so = size_t(s) * d.m;
  // y += H'(sigma_s r4 - r2) over the column's entries in order; four
  // entries' index and value loads in flight before their (unchanged) sums
  auto column = [&](const DevCsr& H, const double* v, int col, double y) {
    int q = H.t_ptr[col];
    const int q1 = H.t_ptr[col + 1];
    for (; q + 4 <= q1; q += 4) {
      int rr[4], sl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rr[u] = H.t_row[q + u];
        sl[u] = H.t_slot[q + u];
      }
      double sg[4], a4[4], b2[4], hv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sg[u] = sigma_s[so + rr[u]];
        a4[u] = r4[so + rr[u]];
        b2[u] = r2[so + rr[u]];
        hv[u] = v[sl[u]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double t = sg[u] * a4[u] - b2[u];
        y += hv[u] * (1.0 * t);
      }
    }
    for (; q < q1; ++q) {
      const int r = H.t_row[q];
      const double t = sigma_s[so + r] * r4[so + r] - r2[so + r];
      y += v[H.t_slot[q]] * (1.0 * t);
    }
    return y;
  };
  if (c < d.n_x) {
    rhat1[size_t(s) * d.n_x + c] =
        column(hx, hxv + size_t(s) * hx.nnz, c, r1x[size_t(s) * d.n_x + c]);
  } else {
    const int cu = c - d.n_x;
    part_u[size_t(s) * d.n_u + cu] = column(hu, huv + size_t(s) * hu.nnz, cu, 0.0);
  }
}

__global__ void scenario_sum_kernel(int M, int n, const double* part, const double* base,
                                    double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = ordered_scenario_sum(part + i, n, M, base ? base[i] : 0.0);
}

// ------------------------------------------- double-double accumulation
struct dd_pair {
  double hi, lo;
};
__device__ __forceinline__ dd_pair two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd_pair dd_add(dd_pair a, dd_pair b) {
  dd_pair s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd_pair dd_add_prod(dd_pair a, double x, double y) {
  const double p = x * y;
  const double e = fma(x, y, -p);
  return dd_add(a, dd_pair{p, e});
}
__device__ __forceinline__ dd_pair dd_add_d(dd_pair a, double x) { return dd_add(a, dd_pair{x, 0.0}); }

__global__ void __launch_bounds__(kB) aug_residual_kernel(AugResidualArgs a, double* partial) {
  constexpr int ops[1] = {kMax};
  double vmax[1] = {0.0};
  const IpmDims& d = a.d;
  const long long per = (long long)d.n_x + d.m + d.n_x + d.m + d.n_u;
  const long long total = (long long)d.M * per;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < total;
       id += (long long)gridDim.x * kB) {
    const int s = int(id / per);
    int r = int(id % per);
    const double* px = a.p.px + size_t(s) * d.n_x;
    const double* py = a.p.py + size_t(s) * d.n_x;
    const double* pz = a.p.pz + size_t(s) * d.m;
    const double* ps = a.p.ps + size_t(s) * d.m;
    const double* pu = a.p.pu;
    if (r < d.n_x) {  // row 1 (x block)
      const int i = r;
      dd_pair t{0.0, 0.0};
      const double* w = a.wxx_v + size_t(s) * a.wxx.nnz;
      for (int q = a.wxx.ptr[i]; q < a.wxx.ptr[i + 1]; ++q) t = dd_add_prod(t, w[q], px[a.wxx.ind[q]]);
      const double* wu = a.wxu_v + size_t(s) * a.wxu.nnz;
      for (int q = a.wxu.ptr[i]; q < a.wxu.ptr[i + 1]; ++q) t = dd_add_prod(t, wu[q], pu[a.wxu.ind[q]]);
      const double* gx = a.gx_v + size_t(s) * a.gx.nnz;
      for (int q = a.gx.t_ptr[i]; q < a.gx.t_ptr[i + 1]; ++q)
        t = dd_add_prod(t, gx[a.gx.t_slot[q]], py[a.gx.t_row[q]]);
      const double* hx = a.hx_v + size_t(s) * a.hx.nnz;
      for (int q = a.hx.t_ptr[i]; q < a.hx.t_ptr[i + 1]; ++q)
        t = dd_add_prod(t, hx[a.hx.t_slot[q]], pz[a.hx.t_row[q]]);
      const size_t k = size_t(s) * d.n_x + i;
      t = dd_add_d(t, (a.sigma_x[k] + a.dw) * px[i]);
      t = dd_add_d(t, a.r1x[k]);
      const double o = t.hi + t.lo;
      a.o1x[k] = o;
      vmax[0] = fmax(vmax[0], fabs(o));
      continue;
    }
    r -= d.n_x;
    if (r < d.m) {  // row 2
      const size_t k = size_t(s) * d.m + r;
      dd_pair t{0.0, 0.0};
      t = dd_add_prod(t, a.sigma_s[k], ps[r]);
      t = dd_add_d(t, pz[r]);
      t = dd_add_d(t, a.r2[k]);
      const double o = t.hi + t.lo;
      a.o2[k] = o;
      vmax[0] = fmax(vmax[0], fabs(o));
      continue;
    }
    r -= d.m;
    if (r < d.n_x) {  // row 3: G p_d + r3 (delta_c = 0 on the reduced path)
      const int i = r;
      dd_pair t{0.0, 0.0};
      const double* gx = a.gx_v + size_t(s) * a.gx.nnz;
      for (int q = a.gx.ptr[i]; q < a.gx.ptr[i + 1]; ++q) t = dd_add_prod(t, gx[q], px[a.gx.ind[q]]);
      const double* gu = a.gu_v + size_t(s) * a.gu.nnz;
      for (int q = a.gu.ptr[i]; q < a.gu.ptr[i + 1]; ++q) t = dd_add_prod(t, gu[q], pu[a.gu.ind[q]]);
      const size_t k = size_t(s) * d.n_x + i;
      t = dd_add_d(t, a.r3[k]);
      const double o = t.hi + t.lo;
      a.o3[k] = o;
      vmax[0] = fmax(vmax[0], fabs(o));
      continue;
    }
    r -= d.n_x;
    if (r < d.m) {  // row 4: H p_d + p_s + r4
      const int i = r;
      dd_pair t{0.0, 0.0};
      const double* hx = a.hx_v + size_t(s) * a.hx.nnz;
      for (int q = a.hx.ptr[i]; q < a.hx.ptr[i + 1]; ++q) t = dd_add_prod(t, hx[q], px[a.hx.ind[q]]);
      const double* hu = a.hu_v + size_t(s) * a.hu.nnz;
      for (int q = a.hu.ptr[i]; q < a.hu.ptr[i + 1]; ++q) t = dd_add_prod(t, hu[q], pu[a.hu.ind[q]]);
      const size_t k = size_t(s) * d.m + i;
      t = dd_add_d(t, ps[i]);
      t = dd_add_d(t, a.r4[k]);
      const double o = t.hi + t.lo;
      a.o4[k] = o;
      vmax[0] = fmax(vmax[0], fabs(o));
      continue;
    }
    r -= d.m;  // u row partial of this scenario: W_xu' p_x + W_uu p_u + G_u' p_y + H_u' p_z
    {
      const int i = r;
      dd_pair t{0.0, 0.0};
      const double* wu = a.wxu_v + size_t(s) * a.wxu.nnz;
      for (int q = a.wxu.t_ptr[i]; q < a.wxu.t_ptr[i + 1]; ++q)
        t = dd_add_prod(t, wu[a.wxu.t_slot[q]], px[a.wxu.t_row[q]]);
      const double* wuu = a.wuu_v + size_t(s) * a.wuu.nnz;
      for (int q = a.wuu.ptr[i]; q < a.wuu.ptr[i + 1]; ++q) t = dd_add_prod(t, wuu[q], pu[a.wuu.ind[q]]);
      const double* gu = a.gu_v + size_t(s) * a.gu.nnz;
      for (int q = a.gu.t_ptr[i]; q < a.gu.t_ptr[i + 1]; ++q)
        t = dd_add_prod(t, gu[a.gu.t_slot[q]], py[a.gu.t_row[q]]);
      const double* hu = a.hu_v + size_t(s) * a.hu.nnz;
      for (int q = a.hu.t_ptr[i]; q < a.hu.t_ptr[i + 1]; ++q)
        t = dd_add_prod(t, hu[a.hu.t_slot[q]], pz[a.hu.t_row[q]]);
      a.o1u_part[(size_t(s) * d.n_u + i) * 2] = t.hi;
      a.o1u_part[(size_t(s) * d.n_u + i) * 2 + 1] = t.lo;
    }
  }
  block_partial<1>(vmax, ops, partial);
}

// per control: the double-double sum over the scenarios, one warp per
// control, lanes over scenarios, then a fixed xor tree (deterministic order)
__global__ void aug_residual_u_local_kernel(AugResidualArgs a, double* dd) {
  const IpmDims& d = a.d;
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * kB + threadIdx.x) >> 5;
  if (i >= d.n_u) return;  // whole warps exit together
  dd_pair t{0.0, 0.0};
  for (int s = lane; s < d.M; s += 32) {
    const size_t k = (size_t(s) * d.n_u + i) * 2;
    t = dd_add(t, dd_pair{a.o1u_part[k], a.o1u_part[k + 1]});
  }
  for (int off = 16; off > 0; off >>= 1) {
    const dd_pair o{__shfl_xor_sync(0xffffffffu, t.hi, off), __shfl_xor_sync(0xffffffffu, t.lo, off)};
    t = (lane & off) ? dd_add(o, t) : dd_add(t, o);  // same operand order on both lanes
  }
  if (lane == 0) {
    dd[2 * i] = t.hi;
    dd[2 * i + 1] = t.lo;
  }
}

__global__ void aug_residual_u_finish_kernel(AugResidualArgs a, const double* dd, double* o1u,
                                             double* out) {
  constexpr int ops[1] = {kMax};
  double vmax[1] = {0.0};
  const IpmDims& d = a.d;
  for (int i = threadIdx.x; i < d.n_u; i += kB) {
    dd_pair t{a.r1u[i], 0.0};
    t = dd_add_d(t, (a.sigma_u[i] + a.dw) * a.p.pu[i]);
    t = dd_add(t, dd_pair{dd[2 * i], dd[2 * i + 1]});
    const double o = t.hi + t.lo;
    o1u[i] = o;
    vmax[0] = fmax(vmax[0], fabs(o));
  }
  block_partial<1>(vmax, ops, out);
}

__global__ void __launch_bounds__(kB) rhs_scale_kernel(IpmDims d, const double* r1x,
                                                       const double* r1u, const double* r2,
                                                       const double* r3, const double* r4,
                                                       double* partial) {
  constexpr int ops[1] = {kMax};
  double v[1] = {1.0};
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  const long long total = 2 * nx + 2 * nm + d.n_u;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < total;
       id += (long long)gridDim.x * kB) {
    double x;
    if (id < nx)
      x = r1x[id];
    else if (id < 2 * nx)
      x = r3[id - nx];
    else if (id < 2 * nx + nm)
      x = r2[id - 2 * nx];
    else if (id < 2 * nx + 2 * nm)
      x = r4[id - 2 * nx - nm];
    else
      x = r1u[id - 2 * nx - 2 * nm];
    v[0] = fmax(v[0], fabs(x));
  }
  block_partial<1>(v, ops, partial);
}

__global__ void axpy_step_kernel(IpmDims d, DevStep a, DevStep q) {
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id < nx) {
    a.px[id] += 1.0 * q.px[id];
    a.py[id] += 1.0 * q.py[id];
  } else if (id < nx + nm) {
    const long long k = id - nx;
    a.ps[k] += 1.0 * q.ps[k];
    a.pz[k] += 1.0 * q.pz[k];
  } else if (id < nx + nm + d.n_u) {
    const long long k = id - nx - nm;
    a.pu[k] += 1.0 * q.pu[k];
  }
}

// ---------------------------------------------------- bound steps / alpha
__device__ __forceinline__ void pair_steps(double v, double pv, double lo, double up, double mlo,
                                           double mup, double mu, double& olo, double& oup) {
  olo = isfinite(lo) ? mu / (v - lo) - mlo - mlo / (v - lo) * pv : 0.0;
  oup = isfinite(up) ? mu / (up - v) - mup + mup / (up - v) * pv : 0.0;
}
__device__ __forceinline__ void cap_primal(double v, double pv, double lo, double up, double tau,
                                           double& a) {
  if (isfinite(lo) && pv < 0) a = fmin(a, -tau * (v - lo) / pv);
  if (isfinite(up) && pv > 0) a = fmin(a, tau * (up - v) / pv);
}
__device__ __forceinline__ void cap_dual(double m, double pm, double tau, double& a) {
  if (pm < 0 && m > 0) a = fmin(a, -tau * m / pm);
}

__global__ void __launch_bounds__(kB) bound_steps_kernel(IpmDims d, DevIter it, DevBounds b,
                                                         DevStep p, double mu, double tau,
                                                         DevBoundStep bs, double* partial) {
  constexpr int ops[2] = {kMin, kMin};
  double v[2] = {1.0, 1.0};
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  const long long total = nx + nm + d.n_u;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < total;
       id += (long long)gridDim.x * kB) {
    if (id < nx) {
      const int i = int(id % d.n_x);
      double lo_s, up_s;
      pair_steps(it.x[id], p.px[id], b.xlo[i], b.xup[i], it.klo[id], it.kup[id], mu, lo_s, up_s);
      bs.klo[id] = lo_s;
      bs.kup[id] = up_s;
      cap_primal(it.x[id], p.px[id], b.xlo[i], b.xup[i], tau, v[0]);
      cap_dual(it.klo[id], lo_s, tau, v[1]);
      cap_dual(it.kup[id], up_s, tau, v[1]);
    } else if (id < nx + nm) {
      const long long k = id - nx;
      const int i = int(k % d.m);
      double lo_s, up_s;
      pair_steps(it.s[k], p.ps[k], b.slo[i], b.sup[i], it.nlo[k], it.nup[k], mu, lo_s, up_s);
      bs.nlo[k] = lo_s;
      bs.nup[k] = up_s;
      cap_primal(it.s[k], p.ps[k], b.slo[i], b.sup[i], tau, v[0]);
      cap_dual(it.nlo[k], lo_s, tau, v[1]);
      cap_dual(it.nup[k], up_s, tau, v[1]);
    } else {
      const int i = int(id - nx - nm);
      double lo_s, up_s;
      pair_steps(it.u[i], p.pu[i], b.ulo[i], b.uup[i], it.llo[i], it.lup[i], mu, lo_s, up_s);
      bs.llo[i] = lo_s;
      bs.lup[i] = up_s;
      cap_primal(it.u[i], p.pu[i], b.ulo[i], b.uup[i], tau, v[0]);
      cap_dual(it.llo[i], lo_s, tau, v[1]);
      cap_dual(it.lup[i], up_s, tau, v[1]);
    }
  }
  block_partial<2>(v, ops, partial);
}

__device__ __forceinline__ void clip(double v, double lo, double up, double mu, double& mlo,
                                     double& mup) {
  const double ks = 1e10;
  if (isfinite(lo)) {
    const double c = mu / (v - lo);
    mlo = fmin(fmax(mlo, c / ks), c * ks);
  }
  if (isfinite(up)) {
    const double c = mu / (up - v);
    mup = fmin(fmax(mup, c / ks), c * ks);
  }
}

__global__ void apply_step_kernel(IpmDims d, DevIter it, DevIter tr, DevBounds b, DevStep p,
                                  DevBoundStep bs, double ap, double ad, double mu) {
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id < nx) {
    const int i = int(id % d.n_x);
    const double x = it.x[id] + ap * p.px[id];
    double klo = it.klo[id] + ad * bs.klo[id], kup = it.kup[id] + ad * bs.kup[id];
    tr.x[id] = x;
    tr.y[id] = it.y[id] + ad * p.py[id];
    clip(x, b.xlo[i], b.xup[i], mu, klo, kup);
    tr.klo[id] = klo;
    tr.kup[id] = kup;
  } else if (id < nx + nm) {
    const long long k = id - nx;
    const int i = int(k % d.m);
    const double s = it.s[k] + ap * p.ps[k];
    double nlo = it.nlo[k] + ad * bs.nlo[k], nup = it.nup[k] + ad * bs.nup[k];
    tr.s[k] = s;
    tr.z[k] = it.z[k] + ad * p.pz[k];
    clip(s, b.slo[i], b.sup[i], mu, nlo, nup);
    tr.nlo[k] = nlo;
    tr.nup[k] = nup;
  } else if (id < nx + nm + d.n_u) {
    const int i = int(id - nx - nm);
    const double u = it.u[i] + ap * p.pu[i];
    double llo = it.llo[i] + ad * bs.llo[i], lup = it.lup[i] + ad * bs.lup[i];
    tr.u[i] = u;
    clip(u, b.ulo[i], b.uup[i], mu, llo, lup);
    tr.llo[i] = llo;
    tr.lup[i] = lup;
  }
}

__global__ void primal_trial_kernel(IpmDims d, DevIter it, DevIter tr, DevStep p, double alpha) {
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id < nx)
    tr.x[id] = it.x[id] + alpha * p.px[id];
  else if (id < nx + nm)
    tr.s[id - nx] = it.s[id - nx] + alpha * p.ps[id - nx];
  else if (id < nx + nm + d.n_u)
    tr.u[id - nx - nm] = it.u[id - nx - nm] + alpha * p.pu[id - nx - nm];
}

// ------------------------------------------------------------- merit terms
__device__ __forceinline__ void barrier_add(double v, double pv, double lo, double up, double mu,
                                            double& logs, double& dir) {
  if (isfinite(lo)) {
    logs -= log(v - lo);
    dir -= mu * pv / (v - lo);
  }
  if (isfinite(up)) {
    logs -= log(up - v);
    dir += mu * pv / (up - v);
  }
}

__global__ void __launch_bounds__(kB) merit_kernel(IpmDims d, DevIter it, DevBounds b, DevStep p,
                                                   const double* grad, const double* f,
                                                   const double* g, const double* h, DevCsr gx,
                                                   DevCsr gu, DevCsr hx, DevCsr hu,
                                                   const double* gxv, const double* guv,
                                                   const double* hxv, const double* huv,
                                                   double mu, double* partial) {
  constexpr int ops[8] = {kSum, kMax, kMax, kSum, kSum, kSum, kSum, kSum};
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long nd = (long long)d.M * (d.n_x + d.n_u), nm = (long long)d.M * d.m;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < nd + nm + d.M;
       id += (long long)gridDim.x * kB) {
    if (id < nd) {
      const int per = d.n_x + d.n_u;
      const int s = int(id / per), c = int(id % per);
      const double* y = it.y + size_t(s) * d.n_x;
      const double* z = it.z + size_t(s) * d.m;
      double gf = grad[size_t(s) * d.n_d + c];
      double pv;
      if (c < d.n_x) {
        const double* gv = gxv + size_t(s) * gx.nnz;
        for (int q = gx.t_ptr[c]; q < gx.t_ptr[c + 1]; ++q) gf -= gv[gx.t_slot[q]] * y[gx.t_row[q]];
        const double* hv = hxv + size_t(s) * hx.nnz;
        for (int q = hx.t_ptr[c]; q < hx.t_ptr[c + 1]; ++q) gf -= hv[hx.t_slot[q]] * z[hx.t_row[q]];
        const size_t k = size_t(s) * d.n_x + c;
        pv = p.px[k];
        v[0] += fabs(g[k]);
        v[1] = fmax(v[1], fabs(it.y[k] + p.py[k]));
        barrier_add(it.x[k], pv, b.xlo[c], b.xup[c], mu, v[3], v[4]);
      } else {
        const int cu = c - d.n_x;
        const double* gv = guv + size_t(s) * gu.nnz;
        for (int q = gu.t_ptr[cu]; q < gu.t_ptr[cu + 1]; ++q) gf -= gv[gu.t_slot[q]] * y[gu.t_row[q]];
        const double* hv = huv + size_t(s) * hu.nnz;
        for (int q = hu.t_ptr[cu]; q < hu.t_ptr[cu + 1]; ++q) gf -= hv[hu.t_slot[q]] * z[hu.t_row[q]];
        pv = p.pu[cu];
      }
      v[5] += gf * pv;
    } else if (id < nd + nm) {
      const long long k = id - nd;
      const int i = int(k % d.m);
      v[0] += fabs(h[k] + it.s[k]);
      v[2] = fmax(v[2], fabs(it.z[k] + p.pz[k]));
      barrier_add(it.s[k], p.ps[k], b.slo[i], b.sup[i], mu, v[3], v[4]);
    } else {
      const int s = int(id - nd - nm);
      v[6] += f[s];
      v[7] += fabs(f[s]);
    }
  }
  block_partial<8>(v, ops, partial);
}

__global__ void merit_u_kernel(IpmDims d, DevIter it, DevBounds b, const double* pu, double mu,
                               double* out) {
  constexpr int ops[2] = {kSum, kSum};
  double v[2] = {0, 0};
  for (int i = threadIdx.x; i < d.n_u; i += kB)
    barrier_add(it.u[i], pu ? pu[i] : 0.0, b.ulo[i], b.uup[i], mu, v[0], v[1]);
  block_partial<2>(v, ops, out);
}

__global__ void __launch_bounds__(kB) ls_values_kernel(IpmDims d, DevIter tr, DevBounds b,
                                                       const double* f, const double* g,
                                                       const double* h, double* partial) {
  constexpr int ops[3] = {kSum, kSum, kSum};
  double v[3] = {0, 0, 0};
  const long long nx = (long long)d.M * d.n_x, nm = (long long)d.M * d.m;
  for (long long id = blockIdx.x * (long long)kB + threadIdx.x; id < nx + nm + d.M;
       id += (long long)gridDim.x * kB) {
    double dummy = 0.0;
    if (id < nx) {
      const int i = int(id % d.n_x);
      v[2] += fabs(g[id]);
      barrier_add(tr.x[id], 0.0, b.xlo[i], b.xup[i], 0.0, v[1], dummy);
    } else if (id < nx + nm) {
      const long long k = id - nx;
      const int i = int(k % d.m);
      v[2] += fabs(h[k] + tr.s[k]);
      barrier_add(tr.s[k], 0.0, b.slo[i], b.sup[i], 0.0, v[1], dummy);
    } else {
      v[0] += f[id - nx - nm];
    }
  }
  block_partial<3>(v, ops, partial);
}

// ----------------------------------------------------------- start point
__device__ __forceinline__ double project_slack(double target, double lo, double up) {
  double mlo = isfinite(lo) ? 1e-2 * fmax(1.0, fabs(lo)) : 0.0;
  double mup = isfinite(up) ? 1e-2 * fmax(1.0, fabs(up)) : 0.0;
  if (isfinite(lo) && isfinite(up)) {
    const double span = up - lo;
    mlo = fmin(mlo, 0.45 * span);
    mup = fmin(mup, 0.45 * span);
  }
  double v = target;
  if (isfinite(up)) v = fmin(v, up - mup);
  if (isfinite(lo)) v = fmax(v, lo + mlo);
  return v;
}

__global__ void init_slacks_kernel(IpmDims d, DevIter it, DevBounds b, const double* h,
                                   double mu0) {
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id >= (long long)d.M * d.m) return;
  const int i = int(id % d.m);
  const double lo = b.slo[i], up = b.sup[i];
  const double s = project_slack(-h[id], lo, up);
  it.s[id] = s;
  it.nlo[id] = isfinite(lo) ? mu0 / (s - lo) : 0.0;
  it.nup[id] = isfinite(up) ? mu0 / (up - s) : 0.0;
  it.z[id] = 0.0;
}

__global__ void init_x_kernel(IpmDims d, DevIter it, DevBounds b, const double* x0, double mu0) {
  const long long id = blockIdx.x * (long long)kB + threadIdx.x;
  if (id >= (long long)d.M * d.n_x) return;
  const int i = int(id % d.n_x);
  const double lo = b.xlo[i], up = b.xup[i], x = x0[i];
  it.x[id] = x;
  it.y[id] = 0.0;
  it.klo[id] = isfinite(lo) ? mu0 / (x - lo) : 0.0;
  it.kup[id] = isfinite(up) ? mu0 / (up - x) : 0.0;
}

__global__ void pu_rhs_kernel(int n, const double* S, const double* r, double* pu, int first) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (first) {
    const double red = S[i] - r[i];   // finish_reduce: rhs -= rhat2
    const double fs = red + r[i];     // first_sum += rhat2
    pu[i] = fs - r[i];                // solve_with: pu -= rhat2
  } else {
    pu[i] = S[i] - r[i];
  }
}

}  // namespace

void launch_pu_rhs(int n, const double* S, const double* r, double* pu, bool first,
                   cudaStream_t st) {
  pu_rhs_kernel<<<ew_blocks(n), kB, 0, st>>>(n, S, r, pu, first ? 1 : 0);
  note_launch();
  check("pu_rhs");
}

void launch_kkt_error_xs(const IpmDims& d, const DevIter& it, const DevBounds& b,
                         const double* grad, const double* g, const double* h, double mu,
                         double* partial, double* out6, cudaStream_t st) {
  const int nb = red_blocks((long long)d.M * (d.n_x + d.m));
  kkt_error_xs_kernel<<<nb, kB, 0, st>>>(d, it, b, grad, g, h, mu, partial);
  note_launch();
  const int ops[6] = {kMax, kMax, kMax, kMax, kMax, kSum};
  finalize<6>(partial, nb, ops, out6, st);
  check("kkt_error_xs");
}

void launch_kkt_eval(const IpmDims& d, const DevIter& it, const DevBounds& b, const double* grad,
                     const double* g, const double* h, const double* f, const int* bad, int lo,
                     const double* gsum_u, const double mus[4], double* partial,
                     unsigned int* counter, double* out, cudaStream_t st) {
  const int nb = red_blocks((long long)d.M * (d.n_x + d.m + 1));
  kkt_eval_kernel<<<nb, kB, 0, st>>>(d, it, b, grad, g, h, f, bad, lo, gsum_u, mus[0], mus[1],
                                     mus[2], mus[3], partial, counter, out);
  note_launch();
  check("kkt_eval");
}

void launch_grad_u_sum(const IpmDims& d, const double* grad, double* gsum, cudaStream_t st) {
  grad_u_sum_kernel<<<ew_blocks(d.n_u), kB, 0, st>>>(d, grad, gsum);
  note_launch();
  check("grad_u_sum");
}

void launch_kkt_error_u(const IpmDims& d, const DevIter& it, const DevBounds& b,
                        const double* gsum, double mu, double* out3, cudaStream_t st) {
  kkt_error_u_kernel<<<1, kB, 0, st>>>(d, it, b, gsum, mu, out3);
  note_launch();
  check("kkt_error_u");
}

void launch_assemble_xs(const IpmDims& d, const DevIter& it, const DevBounds& b,
                        const double* grad, const double* h, double mu, double* sigma_x,
                        double* r1x, double* sigma_s, double* r2, double* r4, int* flag,
                        cudaStream_t st) {
  assemble_xs_kernel<<<ew_blocks((long long)d.M * (d.n_x + d.m)), kB, 0, st>>>(
      d, it, b, grad, h, mu, sigma_x, r1x, sigma_s, r2, r4, flag);
  note_launch();
  check("assemble_xs");
}

void launch_assemble_u(const IpmDims& d, const DevIter& it, const DevBounds& b,
                       const double* gsum, double mu, double* sigma_u, double* r1u, int* flag,
                       cudaStream_t st) {
  assemble_u_kernel<<<ew_blocks(d.n_u), kB, 0, st>>>(d, it, b, gsum, mu, sigma_u, r1u, flag);
  note_launch();
  check("assemble_u");
}

void launch_condensed_rhs(const IpmDims& d, const DevCsr& hx, const DevCsr& hu,
                          const double* hx_v, const double* hu_v, const double* sigma_s,
                          const double* r4, const double* r2, const double* r1x, double* rhat1,
                          double* part_u, cudaStream_t st) {
  condensed_rhs_kernel<<<ew_blocks((long long)d.M * (d.n_x + d.n_u)), kB, 0, st>>>(
      d, hx, hu, hx_v, hu_v, sigma_s, r4, r2, r1x, rhat1, part_u);
  note_launch();
  check("condensed_rhs");
}

void launch_scenario_sum(int M, int n, const double* part, const double* base, double* out,
                         cudaStream_t st) {
  scenario_sum_kernel<<<ew_blocks(n), kB, 0, st>>>(M, n, part, base, out);
  note_launch();
  check("scenario_sum");
}

void launch_aug_residual(const AugResidualArgs& a, double* partial, double* out1,
                         cudaStream_t st) {
  const IpmDims& d = a.d;
  // one item per thread up to the partial buffer's 9,600 slots (one max
  // each, order-free): the dependent double-double chains of a row are
  // latency-bound, so more rows in flight rather than the grid-stride cap
  const long long items = (long long)d.M * (2 * d.n_x + 2 * d.m + d.n_u);
  const int nb = int(std::max(1LL, std::min((items + kB - 1) / kB, 9600LL)));
  aug_residual_kernel<<<nb, kB, 0, st>>>(a, partial);
  note_launch();
  const int ops[1] = {kMax};
  finalize<1>(partial, nb, ops, out1, st);
  check("aug_residual");
}

void launch_aug_residual_u_local(const AugResidualArgs& a, double* dd, cudaStream_t st) {
  const long long threads = (long long)a.d.n_u * 32;
  aug_residual_u_local_kernel<<<int((threads + kB - 1) / kB), kB, 0, st>>>(a, dd);
  note_launch();
  check("aug_residual_u_local");
}

void launch_aug_residual_u_finish(const AugResidualArgs& a, const double* dd, double* o1u,
                                  double* out1, cudaStream_t st) {
  aug_residual_u_finish_kernel<<<1, kB, 0, st>>>(a, dd, o1u, out1);
  note_launch();
  check("aug_residual_u_finish");
}

// the scenario sums spread over the GPU (warp per control), then one CTA
// adds r1u + (sigma_u + dw) p_u and reduces the max
void launch_aug_residual_u(const AugResidualArgs& a, double* dd, double* o1u, double* out1,
                           cudaStream_t st) {
  launch_aug_residual_u_local(a, dd, st);
  launch_aug_residual_u_finish(a, dd, o1u, out1, st);
}


void launch_rhs_scale(const IpmDims& d, const double* r1x, const double* r1u, const double* r2,
                      const double* r3, const double* r4, double* partial, double* out1,
                      cudaStream_t st) {
  const int nb = red_blocks(2LL * d.M * (d.n_x + d.m) + d.n_u);
  rhs_scale_kernel<<<nb, kB, 0, st>>>(d, r1x, r1u, r2, r3, r4, partial);
  note_launch();
  const int ops[1] = {kMax};
  finalize<1>(partial, nb, ops, out1, st);
  check("rhs_scale");
}

void launch_axpy_step(const IpmDims& d, DevStep a, DevStep q, cudaStream_t st) {
  axpy_step_kernel<<<ew_blocks((long long)d.M * (d.n_x + d.m) + d.n_u), kB, 0, st>>>(d, a, q);
  note_launch();
  check("axpy_step");
}

void launch_bound_steps(const IpmDims& d, const DevIter& it, const DevBounds& b, const DevStep& p,
                        double mu, double tau, DevBoundStep bs, double* partial, double* out2,
                        cudaStream_t st) {
  const int nb = red_blocks((long long)d.M * (d.n_x + d.m) + d.n_u);
  bound_steps_kernel<<<nb, kB, 0, st>>>(d, it, b, p, mu, tau, bs, partial);
  note_launch();
  const int ops[2] = {kMin, kMin};
  finalize<2>(partial, nb, ops, out2, st);
  check("bound_steps");
}

void launch_apply_step(const IpmDims& d, const DevIter& it, DevIter trial, const DevBounds& b,
                       const DevStep& p, const DevBoundStep& bs, double ap, double ad, double mu,
                       cudaStream_t st) {
  apply_step_kernel<<<ew_blocks((long long)d.M * (d.n_x + d.m) + d.n_u), kB, 0, st>>>(
      d, it, trial, b, p, bs, ap, ad, mu);
  note_launch();
  check("apply_step");
}

void launch_primal_trial(const IpmDims& d, const DevIter& it, DevIter trial, const DevStep& p,
                         double alpha, cudaStream_t st) {
  primal_trial_kernel<<<ew_blocks((long long)d.M * (d.n_x + d.m) + d.n_u), kB, 0, st>>>(
      d, it, trial, p, alpha);
  note_launch();
  check("primal_trial");
}

void launch_merit(const IpmDims& d, const DevIter& it, const DevBounds& b, const DevStep& p,
                  const double* grad, const double* f, const double* g, const double* h,
                  const DevCsr& gx, const DevCsr& gu, const DevCsr& hx, const DevCsr& hu,
                  const double* gx_v, const double* gu_v, const double* hx_v,
                  const double* hu_v, double mu, double* partial, double* out8,
                  cudaStream_t st) {
  const int nb = red_blocks((long long)d.M * (d.n_x + d.n_u + d.m + 1));
  merit_kernel<<<nb, kB, 0, st>>>(d, it, b, p, grad, f, g, h, gx, gu, hx, hu, gx_v, gu_v, hx_v,
                                  hu_v, mu, partial);
  note_launch();
  const int ops[8] = {kSum, kMax, kMax, kSum, kSum, kSum, kSum, kSum};
  finalize<8>(partial, nb, ops, out8, st);
  check("merit");
}

void launch_merit_u(const IpmDims& d, const DevIter& it, const DevBounds& b, const double* pu,
                    double mu, double* out2, cudaStream_t st) {
  merit_u_kernel<<<1, kB, 0, st>>>(d, it, b, pu, mu, out2);
  note_launch();
  check("merit_u");
}

void launch_ls_values(const IpmDims& d, const DevIter& trial, const DevBounds& b,
                      const double* f, const double* g, const double* h, double* partial,
                      double* out3, cudaStream_t st) {
  const int nb = red_blocks((long long)d.M * (d.n_x + d.m + 1));
  ls_values_kernel<<<nb, kB, 0, st>>>(d, trial, b, f, g, h, partial);
  note_launch();
  const int ops[3] = {kSum, kSum, kSum};
  finalize<3>(partial, nb, ops, out3, st);
  check("ls_values");
}

void launch_init_slacks(const IpmDims& d, DevIter it, const DevBounds& b, const double* h,
                        double mu0, cudaStream_t st) {
  init_slacks_kernel<<<ew_blocks((long long)d.M * d.m), kB, 0, st>>>(d, it, b, h, mu0);
  note_launch();
  check("init_slacks");
}

void launch_init_x(const IpmDims& d, DevIter it, const DevBounds& b, const double* x0,
                   double mu0, cudaStream_t st) {
  init_x_kernel<<<ew_blocks((long long)d.M * d.n_x), kB, 0, st>>>(d, it, b, x0, mu0);
  note_launch();
  check("init_x");
}

}  // namespace bipm
