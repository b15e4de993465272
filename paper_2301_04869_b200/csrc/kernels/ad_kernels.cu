// Batched analytic AD of the polar power-flow basis (subsystem 1).
//
// Replaces batch_eval / batch_jacobian / batch_hessian
// (proj/core/src/autodiff.cpp:256-415) and PolarBasisKernel::eval/adjoint
// (proj/core/src/opf_model.cpp:199-576).  One thread per (basis element,
// scenario) with the scenario index fastest: a warp evaluates one bus /
// branch / generator (or one output slot) for 32 consecutive scenarios, so
// the shared pattern and program loads are warp-uniform broadcasts and every
// per-scenario access of the element-major scratch (psi, dp, w, c: [lane][M])
// is one coalesced 256-byte line.  The reference-layout outputs ([M][nnz],
// scenario-major) are written through 32 x 32 shared-memory tiles so the
// stores are row-contiguous too; the inputs X, y, z are transposed to
// element-major first.  First derivatives replay the reference's
// dual-number operation order, and this file is compiled with -fmad=false
// (the reference builds with -ffp-contract=off), so f, g, h, G and H match the
// reference bit for bit; the Lagrangian Hessian and gradient are analytic
// (equal to rounding, exactly symmetric by construction).
#include <cmath>
#include <stdexcept>
#include <string>

#include "ad_kernels.cuh"
#include "ad_launch.hpp"

#include "stats.hpp"

namespace bipm {

namespace {

constexpr int kB = 256;

__device__ __forceinline__ double in_val(const AdBuffers& b, const DevAd& A, int s, int d) {
  return d < A.n_x ? b.Xt[size_t(d) * A.M + s] : b.u[d - A.n_x];
}

// element-major scratch: lane / slot e of scenario s
__device__ __forceinline__ size_t em(const DevAd& A, int e, int s) {
  return size_t(e) * A.M + s;
}

// [M][cols] -> [cols][M] through a 32 x 32 shared tile (grid: column tiles x
// scenario tiles, 32 x 8 threads)
__global__ void transpose_in_kernel(const double* __restrict__ in, int M, int cols,
                                    double* __restrict__ out) {
  __shared__ double t[32][33];
  const int c0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
  for (int r = y; r < 32; r += 8) {
    const int s = s0 + r, c = c0 + x;
    t[r][x] = (s < M && c < cols) ? in[size_t(s) * cols + c] : 0.0;
  }
  __syncthreads();
  for (int r = y; r < 32; r += 8) {
    const int c = c0 + r, s = s0 + x;
    if (c < cols && s < M) out[size_t(c) * M + s] = t[x][r];
  }
}

// Output tile writer: rows [r0, r0+32) x scenarios [s0, s0+32) computed with
// the scenario fastest (coalesced element-major reads), stored scenario-major
// with the row fastest.  put(r, s, v) routes row r of scenario s to its array.
template <typename Val, typename Put>
__device__ __forceinline__ void tile_rows(int n_rows, int M, Val val, Put put) {
  __shared__ double t[32][33];
  const int r0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
  for (int rr = y; rr < 32; rr += 8) {
    const int r = r0 + rr, s = s0 + x;
    t[rr][x] = (r < n_rows && s < M) ? val(r, s) : 0.0;
  }
  __syncthreads();
  for (int ss = y; ss < 32; ss += 8) {
    const int s = s0 + ss, r = r0 + x;
    if (r < n_rows && s < M) put(r, s, t[x][ss]);
  }
}

__device__ __forceinline__ void flag_bad(const AdBuffers& b, int s, double v) {
  if (!isfinite(v)) b.bad[s] = 1;
}

// Forward pass: basis values (and first partials) of buses, branches, gens.
template <bool kPartials>
__global__ void __launch_bounds__(kB) ad_forward_kernel(DevAd A, AdBuffers b) {
  const int E = A.nbus + A.nbr + A.ngen;
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)E * A.M) return;
  const int e = int(id / A.M), s = int(id % A.M);
  // element-major views: psi[lane] / dp[k] of this scenario
  auto psi = [&](int lane) -> double& { return b.psi[em(A, lane, s)]; };
  auto dp = [&](int k) -> double& { return b.dp[em(A, k, s)]; };
  if (e < A.nbus) {
    const int bus = e;
    const double v = in_val(b, A, s, A.vmag_in[bus]);
    const double vv = v * v;
    psi(A.vv + bus) = vv;
    psi(A.pd + bus) = A.pd_v[em(A, bus, s)];
    psi(A.qd + bus) = A.qd_v[em(A, bus, s)];
    if (bus == 0) psi(0) = 1.0;
    flag_bad(b, s, vv);
    if (kPartials) dp(A.dp_off[A.vv + bus]) = 2.0 * v * 1.0;
    return;
  }
  if (e < A.nbus + A.nbr) {
    const int l = e - A.nbus;
    const double* c = A.brc + 8 * l;
    const double gff = c[0], bff = c[1], gft = c[2], bft = c[3], gtf = c[4], btf = c[5],
                 gtt = c[6], btt = c[7];
    const int thf = A.br_th[2 * l], tht = A.br_th[2 * l + 1];
    const int ivf = A.br_v[2 * l], ivt = A.br_v[2 * l + 1];
    const double vf = in_val(b, A, s, ivf), vt = in_val(b, A, s, ivt);
    double dth;
    if (thf >= 0 && tht >= 0)
      dth = in_val(b, A, s, thf) - in_val(b, A, s, tht);
    else if (thf >= 0)
      dth = in_val(b, A, s, thf);
    else if (tht >= 0)
      dth = in_val(b, A, s, tht) * -1.0;
    else
      dth = 0.0;
    const double sn = sin(dth), cs = cos(dth);
    const double vv = vf * vt;
    const double st = A.status[em(A, l, s)];
    const double cff = (vf * vf) * st, ctt = (vt * vt) * st;
    const double wc = (cs * vv) * st, ws = (sn * vv) * st;
    const double Pf = gff * cff + gft * wc + bft * ws;
    const double Qf = -bff * cff + -bft * wc + gft * ws;
    const double Pt = gtt * ctt + gtf * wc + -btf * ws;
    const double Qt = -btt * ctt + -btf * wc + -gtf * ws;
    const double sqf = Pf * Pf + Qf * Qf, sqt = Pt * Pt + Qt * Qt;
    psi(A.br + 4 * l) = cff;
    psi(A.br + 4 * l + 1) = ctt;
    psi(A.br + 4 * l + 2) = wc;
    psi(A.br + 4 * l + 3) = ws;
    psi(A.sq + 2 * l) = sqf;
    psi(A.sq + 2 * l + 1) = sqt;
    flag_bad(b, s, sqf + sqt + wc + ws + cff + ctt);
    if (kPartials) {
      dp(A.dp_off[A.br + 4 * l]) = 2.0 * vf * 1.0 * st;
      dp(A.dp_off[A.br + 4 * l + 1]) = 2.0 * vt * 1.0 * st;
      // support order: [theta_f?, theta_t?, v_f, v_t]
      int k = 0;
      const int o_wc = A.dp_off[A.br + 4 * l + 2], o_ws = A.dp_off[A.br + 4 * l + 3];
      const int o_sf = A.dp_off[A.sq + 2 * l], o_st = A.dp_off[A.sq + 2 * l + 1];
      for (int q = 0; q < 4; ++q) {
        double tdl, tvf, tvt;
        if (q == 0) {
          if (thf < 0) continue;
          tdl = 1.0, tvf = 0.0, tvt = 0.0;
        } else if (q == 1) {
          if (tht < 0) continue;
          tdl = -1.0;
          tvf = 0.0, tvt = 0.0;
        } else if (q == 2) {
          tdl = 0.0, tvf = 1.0, tvt = 0.0;
        } else {
          tdl = 0.0, tvf = 0.0, tvt = 1.0;
        }
        const double vvt = vf * tvt + tvf * vt;
        const double wct = (cs * vvt + (-sn * tdl) * vv) * st;
        const double wst = (sn * vvt + (cs * tdl) * vv) * st;
        const double cft = (2.0 * vf * tvf) * st;
        const double ctt_t = (2.0 * vt * tvt) * st;
        const double Pft = gff * cft + gft * wct + bft * wst;
        const double Qft = -bff * cft + -bft * wct + gft * wst;
        const double Ptt = gtt * ctt_t + gtf * wct + -btf * wst;
        const double Qtt = -btt * ctt_t + -btf * wct + -gtf * wst;
        const double dsf = 2.0 * (Pf * Pft + Qf * Qft), dst = 2.0 * (Pt * Ptt + Qt * Qtt);
        dp(o_wc + k) = wct;
        dp(o_ws + k) = wst;
        dp(o_sf + k) = dsf;
        dp(o_st + k) = dst;
        flag_bad(b, s, wct + wst + dsf + dst);
        ++k;
      }
    }
    return;
  }
  const int g = e - A.nbus - A.nbr;
  if (g == A.slack_gen) return;
  const double p = in_val(b, A, s, A.pgen_in[g]);
  psi(A.pg + g) = p;
  psi(A.pg2 + g) = p * p;
  flag_bad(b, s, p * p);
  if (kPartials) {
    dp(A.dp_off[A.pg + g]) = 1.0;
    dp(A.dp_off[A.pg2 + g]) = 2.0 * p * 1.0;
  }
}

// Dependent slack generation p = Pd_ref + gs vv_ref + ref flows - other gens.
template <bool kPartials>
__global__ void ad_slack_kernel(DevAd A, AdBuffers b) {
  const int per = A.nsd + 1;
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)per * A.M) return;
  const int j = int(id / A.M), s = int(id % A.M);
  double v = b.psi[em(A, A.pd + A.ref_bus, s)];
  for (int q = A.slack_val.ptr[0]; q < A.slack_val.ptr[1]; ++q)
    v += A.slack_val.coef[q] * b.psi[em(A, A.slack_val.src[q], s)];
  if (j == A.nsd) {
    b.psi[em(A, A.pg + A.slack_gen, s)] = v;
    b.psi[em(A, A.pg2 + A.slack_gen, s)] = v * v;
    flag_bad(b, s, v * v);
    return;
  }
  if (!kPartials) return;
  double t = 0.0;
  for (int q = A.slack_grad.ptr[j]; q < A.slack_grad.ptr[j + 1]; ++q)
    t += A.slack_grad.coef[q] * b.dp[em(A, A.slack_grad.src[q], s)];
  b.dp[em(A, A.dp_off[A.pg + A.slack_gen] + j, s)] = t;
  b.dp[em(A, A.dp_off[A.pg2 + A.slack_gen] + j, s)] = 2.0 * v * t;
  flag_bad(b, s, t * v);
}

// f = L_f psi, g = L_g psi, h = L_h psi
// The objective row (~2 ngen terms: 520 at 1354) as one lane's sequential
// loop was the values kernel's long pole (65 dependent rounds of loads).  Here
// a warp per scenario forms the products in parallel, 256 at a time, and one
// lane adds them in the reference's order (autodiff.cpp:265-279): the same
// rounded products, the same sequence of rounded sums (-fmad=false).
constexpr int kObjChunk = 256;
__global__ void __launch_bounds__(256) ad_objective_kernel(DevAd A, AdBuffers b) {
  __shared__ double prod[8][kObjChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * 8 + warp;
  if (s >= A.M) return;
  const int e0 = A.Lf_ptr[0], e1 = A.Lf_ptr[1];
  double v = 0.0;
  for (int c = e0; c < e1; c += kObjChunk) {
    const int n = min(kObjChunk, e1 - c);
    for (int k = lane; k < n; k += 32) prod[warp][k] = A.Lf_val[c + k] * b.psi[em(A, A.Lf_ind[c + k], s)];
    __syncwarp();
    if (lane == 0)
      for (int k = 0; k < n; ++k) v += prod[warp][k];
    __syncwarp();
  }
  if (lane == 0) b.f[s] = v;
}

__global__ void __launch_bounds__(256) ad_values_kernel(DevAd A, AdBuffers b) {
  const int R = 1 + A.n_x + A.m;
  tile_rows(
      R, A.M,
      [&](int r, int s) {
        const int *ptr, *ind;
        const double* val;
        int row;
        if (r == 0) {
          return 0.0;  // ad_objective_kernel
        } else if (r <= A.n_x) {
          row = r - 1;
          ptr = A.Lg_ptr, ind = A.Lg_ind, val = A.Lg_val;
        } else {
          row = r - 1 - A.n_x;
          ptr = A.Lh_ptr, ind = A.Lh_ind, val = A.Lh_val;
        }
        // the reference's order (autodiff.cpp:265-279), eight loads in flight
        // (the objective row has ~2 ngen terms; 16 in flight measured slower)
        double v = 0.0;
        int e = ptr[row];
        const int e1 = ptr[row + 1];
        for (; e + 8 <= e1; e += 8) {
          double a[8], x[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = val[e + k];
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] = b.psi[em(A, ind[e + k], s)];
#pragma unroll
          for (int k = 0; k < 8; ++k) v += a[k] * x[k];
        }
        for (; e < e1; ++e) v += val[e] * b.psi[em(A, ind[e], s)];
        return v;
      },
      [&](int r, int s, double v) {
        if (r == 0)
          return;
        else if (r <= A.n_x)
          b.g[size_t(s) * A.n_x + (r - 1)] = v;
        else
          b.h[size_t(s) * A.m + (r - 1 - A.n_x)] = v;
      });
}

// x element-major ([src][M]): the scenario's column; sequential sums in the
// program's order, four loads in flight
__device__ __forceinline__ double gather_coef(const DevGather& G, int k, const double* x, int M,
                                              int s) {
  double v = 0.0;
  int q = G.ptr[k];
  const int q1 = G.ptr[k + 1];
  for (; q + 4 <= q1; q += 4) {
    double c[4], y[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = G.coef[q + j];
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = x[size_t(G.src[q + j]) * M + s];
#pragma unroll
    for (int j = 0; j < 4; ++j) v += c[j] * y[j];
  }
  for (; q < q1; ++q) v += G.coef[q] * x[size_t(G.src[q]) * M + s];
  return v;
}

__device__ __forceinline__ double gather_sum(const DevGather& G, int k, const double* x, int M,
                                             int s) {
  double v = 0.0;
  int q = G.ptr[k];
  const int q1 = G.ptr[k + 1];
  for (; q + 4 <= q1; q += 4) {
    double y[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = x[size_t(G.src[q + j]) * M + s];
#pragma unroll
    for (int j = 0; j < 4; ++j) v += y[j];
  }
  for (; q < q1; ++q) v += x[size_t(G.src[q]) * M + s];
  return v;
}

// G_x, G_u, H_x, H_u from the lane partials
__global__ void __launch_bounds__(256) ad_jacobian_kernel(DevAd A, AdBuffers b) {
  const int n1 = A.gx.n, n2 = n1 + A.gu.n, n3 = n2 + A.hx.n, R = n3 + A.hu.n;
  tile_rows(
      R, A.M,
      [&](int k, int s) {
        if (k < n1) return gather_coef(A.gx, k, b.dp, A.M, s);
        if (k < n2) return gather_coef(A.gu, k - n1, b.dp, A.M, s);
        if (k < n3) return gather_coef(A.hx, k - n2, b.dp, A.M, s);
        return gather_coef(A.hu, k - n3, b.dp, A.M, s);
      },
      [&](int k, int s, double v) {
        if (k < n1)
          b.gx[size_t(s) * n1 + k] = v;
        else if (k < n2)
          b.gu[size_t(s) * A.gu.n + (k - n1)] = v;
        else if (k < n3)
          b.hx[size_t(s) * A.hx.n + (k - n2)] = v;
        else
          b.hu[size_t(s) * A.hu.n + (k - n3)] = v;
      });
}

// w = obj_w L_f' + L_g' y + L_h' z
__global__ void ad_weights_kernel(DevAd A, AdBuffers b) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)A.n_b * A.M) return;
  const int j = int(id / A.M), s = int(id % A.M);
  double v = 0.0;
  for (int q = A.w.ptr[j]; q < A.w.ptr[j + 1]; ++q) {
    const int src = A.w.src[q];
    const double c = A.w.coef[q];
    if (src < 0)
      v += b.obj_w * c;
    else if (src < A.n_x)
      v += c * b.Yt[em(A, src, s)];
    else
      v += c * b.Zt[em(A, src - A.n_x, s)];
  }
  b.w[em(A, j, s)] = v;
}

// Element-local Lagrangian gradient and Hessian contributions.
__global__ void __launch_bounds__(kB) ad_second_kernel(DevAd A, AdBuffers b) {
  const int E = A.nbus + A.nbr + A.ngen + A.nsd;
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)E * A.M) return;
  const int e = int(id / A.M), s = int(id % A.M);
  auto psi = [&](int lane) { return b.psi[em(A, lane, s)]; };
  auto w = [&](int lane) { return b.w[em(A, lane, s)]; };
  auto c = [&](int k) -> double& { return b.c[em(A, k, s)]; };
  const double psl = psi(A.pg + A.slack_gen);
  const double sv = w(A.pg + A.slack_gen) + w(A.pg2 + A.slack_gen) * 2.0 * psl;
  if (e < A.nbus) {
    const int bus = e;
    const double v = in_val(b, A, s, A.vmag_in[bus]);
    double wv = w(A.vv + bus);
    if (bus == A.ref_bus) wv += A.gs_ref * sv;
    c(A.c_bus + 2 * bus) = 2.0 * v * wv;
    c(A.c_bus + 2 * bus + 1) = 2.0 * wv;
    flag_bad(b, s, v * wv);
    return;
  }
  if (e < A.nbus + A.nbr) {
    const int l = e - A.nbus;
    const double* cf = A.brc + 8 * l;
    const double gff = cf[0], bff = cf[1], gft = cf[2], bft = cf[3], gtf = cf[4], btf = cf[5],
                 gtt = cf[6], btt = cf[7];
    const int thf = A.br_th[2 * l], tht = A.br_th[2 * l + 1];
    const int ivf = A.br_v[2 * l], ivt = A.br_v[2 * l + 1];
    const double vf = in_val(b, A, s, ivf), vt = in_val(b, A, s, ivt);
    double dth = 0.0;
    if (thf >= 0) dth += in_val(b, A, s, thf);
    if (tht >= 0) dth -= in_val(b, A, s, tht);
    const double sn = sin(dth), cs = cos(dth), st = A.status[em(A, l, s)];
    const double vv = vf * vt;
    const double cff = st * vf * vf, ctt = st * vt * vt, wc = st * vv * cs, ws = st * vv * sn;
    const double Pf = gff * cff + gft * wc + bft * ws, Qf = -bff * cff - bft * wc + gft * ws;
    const double Pt = gtt * ctt + gtf * wc - btf * ws, Qt = -btt * ctt - btf * wc - gtf * ws;
    const int rf = A.br_ref[l];
    const double wsqf = w(A.sq + 2 * l), wsqt = w(A.sq + 2 * l + 1);
    double ocff = w(A.br + 4 * l) + 2.0 * wsqf * (Pf * gff - Qf * bff);
    double octt = w(A.br + 4 * l + 1) + 2.0 * wsqt * (Pt * gtt - Qt * btt);
    double owc = w(A.br + 4 * l + 2) + 2.0 * wsqf * (Pf * gft - Qf * bft) +
                 2.0 * wsqt * (Pt * gtf - Qt * btf);
    double ows = w(A.br + 4 * l + 3) + 2.0 * wsqf * (Pf * bft + Qf * gft) +
                 2.0 * wsqt * (-Pt * btf - Qt * gtf);
    if (rf & 1) ocff += gff * sv, owc += gft * sv, ows += bft * sv;
    if (rf & 2) octt += gtt * sv, owc += gtf * sv, ows += -btf * sv;
    const double d0 = thf >= 0 ? 1.0 : 0.0, d1 = tht >= 0 ? -1.0 : 0.0;
    const double dd[4] = {d0, d1, 0.0, 0.0};
    // gradients of the monomials (local order th_f, th_t, v_f, v_t)
    const double gcf[4] = {0.0, 0.0, 2.0 * st * vf, 0.0};
    const double gct[4] = {0.0, 0.0, 0.0, 2.0 * st * vt};
    const double gwc[4] = {-st * vv * sn * d0, -st * vv * sn * d1, st * vt * cs, st * vf * cs};
    const double gws[4] = {st * vv * cs * d0, st * vv * cs * d1, st * vt * sn, st * vf * sn};
    double gPf[4], gQf[4], gPt[4], gQt[4];
    for (int a = 0; a < 4; ++a) {
      gPf[a] = gff * gcf[a] + gft * gwc[a] + bft * gws[a];
      gQf[a] = -bff * gcf[a] - bft * gwc[a] + gft * gws[a];
      gPt[a] = gtt * gct[a] + gtf * gwc[a] - btf * gws[a];
      gQt[a] = -btt * gct[a] - btf * gwc[a] - gtf * gws[a];
      c(14 * l + a) = ocff * gcf[a] + octt * gct[a] + owc * gwc[a] + ows * gws[a];
    }
    // second derivatives of wc / ws in (Delta, v_f, v_t) coordinates
    const double wc_dd = -st * vv * cs, wc_dvf = -st * vt * sn, wc_dvt = -st * vf * sn,
                 wc_ff = st * cs;
    const double ws_dd = -st * vv * sn, ws_dvf = st * vt * cs, ws_dvt = st * vf * cs,
                 ws_ff = st * sn;
    int q = 4;
    for (int a = 0; a < 4; ++a)
      for (int bb = a; bb < 4; ++bb) {
        double hwc = 0.0, hws = 0.0, hcf = 0.0, hct = 0.0;
        if (a < 2 && bb < 2) {
          hwc = dd[a] * dd[bb] * wc_dd;
          hws = dd[a] * dd[bb] * ws_dd;
        } else if (a < 2) {  // (theta, v)
          hwc = dd[a] * (bb == 2 ? wc_dvf : wc_dvt);
          hws = dd[a] * (bb == 2 ? ws_dvf : ws_dvt);
        } else if (a == 2 && bb == 3) {
          hwc = wc_ff;
          hws = ws_ff;
        } else if (a == 2 && bb == 2) {
          hcf = 2.0 * st;
        } else {
          hct = 2.0 * st;
        }
        c(14 * l + q) = ocff * hcf + octt * hct + owc * hwc + ows * hws +
                        2.0 * wsqf * (gPf[a] * gPf[bb] + gQf[a] * gQf[bb]) +
                        2.0 * wsqt * (gPt[a] * gPt[bb] + gQt[a] * gQt[bb]);
        ++q;
      }
    flag_bad(b, s, c(14 * l) + c(14 * l + 4) + c(14 * l + 13));
    return;
  }
  if (e < A.nbus + A.nbr + A.ngen) {
    const int g = e - A.nbus - A.nbr;
    if (g == A.slack_gen) return;
    const double p = in_val(b, A, s, A.pgen_in[g]);
    double wv = w(A.pg + g) + w(A.pg2 + g) * 2.0 * p;
    if (A.gen_ref_other[g]) wv -= sv;
    c(A.c_gen + 2 * g) = wv;
    c(A.c_gen + 2 * g + 1) = 2.0 * w(A.pg2 + g);
    flag_bad(b, s, wv);
    return;
  }
  // slack rank-one curvature 2 w_sl2 grad p grad p'
  const int i = e - A.nbus - A.nbr - A.ngen;
  const int off = A.dp_off[A.pg + A.slack_gen];
  const double w2 = 2.0 * w(A.pg2 + A.slack_gen);
  const double gi = b.dp[em(A, off + i, s)];
  for (int j = 0; j < A.nsd; ++j) c(A.c_slack + i * A.nsd + j) = w2 * gi * b.dp[em(A, off + j, s)];
}

// W blocks and the Lagrangian gradient
__global__ void __launch_bounds__(256) ad_hessian_kernel(DevAd A, AdBuffers b) {
  const int n1 = A.wxx.n, n2 = n1 + A.wxu.n, n3 = n2 + A.wuu.n, R = n3 + A.n_d;
  tile_rows(
      R, A.M,
      [&](int k, int s) {
        if (k < n1) return gather_sum(A.wxx, k, b.c, A.M, s);
        if (k < n2) return gather_sum(A.wxu, k - n1, b.c, A.M, s);
        if (k < n3) return gather_sum(A.wuu, k - n2, b.c, A.M, s);
        return gather_sum(A.grad, k - n3, b.c, A.M, s);
      },
      [&](int k, int s, double v) {
        if (k < n1)
          b.wxx[size_t(s) * n1 + k] = v;
        else if (k < n2)
          b.wxu[size_t(s) * A.wxu.n + (k - n1)] = v;
        else if (k < n3)
          b.wuu[size_t(s) * A.wuu.n + (k - n2)] = v;
        else
          b.grad[size_t(s) * A.n_d + (k - n3)] = v;
      });
}

int blocks(long long n) { return int((n + kB - 1) / kB); }

void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

dim3 tiles(int rows, int M) { return dim3((rows + 31) / 32, (M + 31) / 32); }

void transpose_in(const double* in, int M, int cols, double* out, cudaStream_t st) {
  if (cols <= 0 || !in) return;
  transpose_in_kernel<<<tiles(cols, M), 256, 0, st>>>(in, M, cols, out);
  note_launch();
}

}  // namespace

void launch_ad_bundle(const DevAd& A, const AdBuffers& b, cudaStream_t st) {
  const long long M = A.M;
  transpose_in(b.X, A.M, A.n_x, b.Xt, st);
  transpose_in(b.Y, A.M, A.n_x, b.Yt, st);
  transpose_in(b.Z, A.M, A.m, b.Zt, st);
  ad_forward_kernel<true><<<blocks(M * (A.nbus + A.nbr + A.ngen)), kB, 0, st>>>(A, b);
  note_launch();
  ad_slack_kernel<true><<<blocks(M * (A.nsd + 1)), kB, 0, st>>>(A, b);
  note_launch();
  ad_values_kernel<<<tiles(1 + A.n_x + A.m, A.M), 256, 0, st>>>(A, b);
  ad_objective_kernel<<<int((M + 7) / 8), 256, 0, st>>>(A, b);
  note_launch(2);
  ad_jacobian_kernel<<<tiles(A.gx.n + A.gu.n + A.hx.n + A.hu.n, A.M), 256, 0, st>>>(A, b);
  note_launch();
  ad_weights_kernel<<<blocks(M * A.n_b), kB, 0, st>>>(A, b);
  note_launch();
  ad_second_kernel<<<blocks(M * (A.nbus + A.nbr + A.ngen + A.nsd)), kB, 0, st>>>(A, b);
  note_launch();
  ad_hessian_kernel<<<tiles(A.wxx.n + A.wxu.n + A.wuu.n + A.n_d, A.M), 256, 0, st>>>(A, b);
  note_launch();
  check("ad_bundle");
}

void launch_ad_values(const DevAd& A, const AdBuffers& b, cudaStream_t st) {
  const long long M = A.M;
  transpose_in(b.X, A.M, A.n_x, b.Xt, st);
  ad_forward_kernel<false><<<blocks(M * (A.nbus + A.nbr + A.ngen)), kB, 0, st>>>(A, b);
  note_launch();
  ad_slack_kernel<false><<<blocks(M * (A.nsd + 1)), kB, 0, st>>>(A, b);
  note_launch();
  ad_values_kernel<<<tiles(1 + A.n_x + A.m, A.M), 256, 0, st>>>(A, b);
  ad_objective_kernel<<<int((M + 7) / 8), 256, 0, st>>>(A, b);
  note_launch(2);
  check("ad_values");
}

}  // namespace bipm
