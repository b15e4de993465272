// Forward half of X = G_x^{-1} P G_u for all control columns of every
// scenario (host/stream_plan.hpp ReachPlan), and the batched FP64 DMMA GEMM
// that applies the dense tail inverse W to it.
//
// The reference solves every column of every tile with the whole L factor
// (reduce_group, kkt.cpp:388-404: spsm over n_x rows per column); column u
// of L^{-1} P G_u is nonzero only on the reach of G_u's rows in the graph of
// L, a few etree paths.  reach_solve_kernel walks exactly those rows (a
// group of 4-32 lanes per (scenario, column), the column's y_N in shared
// memory, factor values staged a segment at a time with all loads in
// flight), then gathers the tail rows y_T = (P G_u)_T - L_TN y_N.  X_T = W y_T
// is then formed for all n_u columns at once -- by gemm_tn_kernel (FP64 DMMA)
// or, when y_T is sparse enough, by xt_sparse_kernel -- so W is read once per
// scenario instead of once per column tile of the reduction.  gemm_tn_kernel
// also forms the batch-sum tail product -sum_s X_T' Z_T after the tiles.
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "reach_gemm.hpp"
#include "stats.hpp"

namespace bipm {

namespace {

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kReachWarps = 4;

// One group of G lanes per (scenario, column): the column's ops run in order,
// each op's entries split over the group's lanes and summed by shuffles
// within the group; 32 / G columns per warp.  Dynamic shared memory per
// group: y_N of its column (ymax doubles), then the staged segment (SEG
// factor values + SEG source indices, SEG = 8 G) so a segment's loads are all
// in flight before its dependent ops run.
template <int G>
__global__ void __launch_bounds__(32 * kReachWarps)
    reach_solve_kernel(ReachDev p, const double* __restrict__ F, long long nnz_f,
                       const double* __restrict__ gu, long long gu_nnz, double* __restrict__ yn,
                       double* __restrict__ yt) {
  constexpr int SEG = 8 * G, NG = 32 / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (grp * G);
  const int u = (blockIdx.x * kReachWarps + warp) * NG + grp, s = blockIdx.y;
  if (u >= p.n_u) return;  // the whole group leaves together
  const int ymax = p.ymax;
  unsigned char* wb =
      smem + size_t(warp * NG + grp) * (size_t(ymax) * 8 + SEG * 12);
  double* y = reinterpret_cast<double*>(wb);
  double* fv = y + ymax;
  int* src = reinterpret_cast<int*>(fv + SEG);
  const double* Fs = F + size_t(s) * nnz_f;
  const double* gs = gu + size_t(s) * gu_nnz;
  const int ob = p.op_ptr[u], oe = p.op_ptr[u + 1];
  const int ny = p.yn_ptr[u + 1] - p.yn_ptr[u];
  // packed y_T: the column's tail ops follow its ny y_N ops in yt_row order
  double* ts = p.packed ? yt + size_t(s) * p.nnz_yt + p.yt_ptr[u] - (ob + ny)
                        : yt + (size_t(s) * p.n_u + u) * p.ldy;
  if (!p.packed)
    for (int i = gl; i < p.ldy; i += G) ts[i] = 0.0;
  for (int o = ob; o < oe;) {
    // segment: up to G ops whose entries fit the staging buffer (an op with
    // more entries than that runs alone, straight from global memory)
    const bool valid = o + gl < oe;
    const int4 rec = valid ? p.ops[o + gl] : make_int4(0, -1, 0, 0x7fffffff);
    const int e0 = __shfl_sync(gmask, rec.z, 0, G);
    // entries are contiguous and increasing over the ops: a prefix of lanes fits
    const unsigned fits =
        (__ballot_sync(gmask, valid && rec.w - e0 <= SEG) >> (grp * G)) & (gmask >> (grp * G));
    const bool staged = (fits & 1u) != 0;
    const int nseg = staged ? __popc(fits) : 1;
    const double bval = rec.y >= 0 ? gs[rec.y] : 0.0;
    const int e1 = __shfl_sync(gmask, rec.w, nseg - 1, G);
    if (staged) {
      for (int e = e0 + gl; e < e1; e += G) {
        const int2 en = p.ent[e];
        src[e - e0] = en.x;
        fv[e - e0] = Fs[en.y];
      }
      __syncwarp(gmask);
    }
    for (int i = 0; i < nseg; ++i) {
      const int dest = __shfl_sync(gmask, rec.x, i, G);
      const int eb = __shfl_sync(gmask, rec.z, i, G), ee = __shfl_sync(gmask, rec.w, i, G);
      const double b = __shfl_sync(gmask, bval, i, G);
      double a = 0.0;
      if (staged) {
        for (int e = eb - e0 + gl; e < ee - e0; e += G) a += fv[e] * y[src[e]];
      } else {
        for (int e = eb + gl; e < ee; e += G) {
          const int2 en = p.ent[e];
          a += Fs[en.y] * y[en.x];
        }
      }
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) a += __shfl_xor_sync(gmask, a, off, G);
      if (gl == 0) {
        if (dest >= 0)
          y[dest] = b - a;
        else
          ts[p.packed ? o + i : -1 - dest] = b - a;
      }
      __syncwarp(gmask);
    }
    o += nseg;
  }
  double* ys = yn + size_t(s) * p.nnz_yn + p.yn_ptr[u];
  for (int i = gl; i < ny; i += G) ys[i] = y[i];
}

// X_T = W y_T with y_T sparse (column u nonzero on yt_row[yt_ptr[u] ..], its
// values packed in the same order, [M][nnz_yt]):
// X_T[:, u] = sum_k y_T[t_k, u] W[:, t_k] = sum_k y_T[t_k, u] W'[t_k, :].
// CTA = (scenario, 32 RPL output rows): W'[:, i-block] (tl x 32 RPL) is staged
// in shared memory once, then each warp forms whole columns u, lane = RPL
// consecutive rows i.  A column's (t_k, y) pairs are read coalesced (packed
// y_T; the next chunk's loads in flight while the current one is summed) and
// written as 16-byte records to the warp's slot in shared memory, so each
// entry costs one broadcast record load plus one W' load of RPL doubles per
// lane (shuffling t and y to the lanes cost three SHFLs per entry and
// bound the kernel on the MIO queue).  RPL = 2 halves the record loads per
// FMA where the 64-row W' block fits in shared memory.
constexpr int kXtRows = 32, kXtWarps = 16;
template <int RPL>
__global__ void __launch_bounds__(32 * kXtWarps)
    xt_sparse_kernel(const double* __restrict__ WT, int ldw, long long sw,
                     const double* __restrict__ ytc, int nnz_yt, const int* __restrict__ yt_ptr,
                     const int* __restrict__ yt_row, int n_u, int tl, double* __restrict__ xt,
                     int ldy) {
  constexpr int R = kXtRows * RPL;  // rows per CTA
  extern __shared__ __align__(16) double wts[];  // [tl][R], records, then yt_ptr
  double2* rec_all = reinterpret_cast<double2*>(wts + size_t(tl) * R);
  int* ptr = reinterpret_cast<int*>(rec_all + 32 * kXtWarps);
  const int s = blockIdx.y, i0 = blockIdx.x * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* W = WT + size_t(s) * sw;
  for (int q = tid; q < tl * R; q += 32 * kXtWarps) {
    const int t = q / R, i = i0 + q % R;
    wts[q] = i < tl ? W[size_t(t) * ldw + i] : 0.0;
  }
  for (int q = tid; q <= n_u; q += 32 * kXtWarps) ptr[q] = yt_ptr[q];
  __syncthreads();
  double2* rec = rec_all + 32 * warp;
  const unsigned rec_b = static_cast<unsigned>(__cvta_generic_to_shared(rec));
  const unsigned w_b = static_cast<unsigned>(__cvta_generic_to_shared(wts)) + 8 * RPL * lane;
  const double* ys = ytc + size_t(s) * nnz_yt;
  double* xs = xt + size_t(s) * n_u * ldy;
  // chunk of up to 32 entries starting at k0 of column u (rows pre-scaled to
  // byte offsets of W' rows)
  auto fetch = [&](int k0, int ke, int& tv, double& yv) {
    const int k = k0 + lane;
    tv = k < ke ? yt_row[k] * (R * 8) : 0;
    yv = k < ke ? ys[k] : 0.0;
  };
  int u = warp;
  if (u >= n_u) return;
  int tn;
  double yn;
  fetch(ptr[u], ptr[u + 1], tn, yn);
  for (; u < n_u; u += kXtWarps) {
    const int kb = ptr[u], ke = ptr[u + 1];
    double a0[RPL], a1[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) a0[r] = a1[r] = 0.0;
    for (int k0 = kb; k0 < ke; k0 += 32) {
      __syncwarp();
      rec[lane] = make_double2(yn, __hiloint2double(0, tn));
      __syncwarp();
      // the following chunk (this column's or the next column's first) in flight
      if (k0 + 32 < ke) {
        fetch(k0 + 32, ke, tn, yn);
      } else if (u + kXtWarps < n_u) {
        fetch(ptr[u + kXtWarps], ptr[u + kXtWarps + 1], tn, yn);
      }
      const int n = min(32, ke - k0);
      int k = 0;
      for (; k + 3 < n; k += 4) {
        double2 e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                       : "=d"(e[q].x), "=d"(e[q].y)
                       : "r"(rec_b + 16 * (k + q)));
        double w[4][RPL];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const unsigned a = w_b + unsigned(__double2loint(e[q].y));
          if constexpr (RPL == 2)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w[q][0]), "=d"(w[q][1]) : "r"(a));
          else
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(w[q][0]) : "r"(a));
        }
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          a0[r] += e[0].x * w[0][r];
          a1[r] += e[1].x * w[1][r];
          a0[r] += e[2].x * w[2][r];
          a1[r] += e[3].x * w[3][r];
        }
      }
      for (; k < n; ++k) {
        double2 e;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(e.x), "=d"(e.y) : "r"(rec_b + 16 * k));
        const unsigned a = w_b + unsigned(__double2loint(e.y));
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          double w;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(w) : "r"(a + 8 * r));
          a0[r] += e.x * w;
        }
      }
    }
    if (kb == ke && u + kXtWarps < n_u)  // empty column: its successor's chunk
      fetch(ptr[u + kXtWarps], ptr[u + kXtWarps + 1], tn, yn);
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = i0 + RPL * lane + r;
      if (i < tl) xs[size_t(u) * ldy + i] = a0[r] + a1[r];
    }
  }
}

// ------------------------------------------------------------- DMMA GEMM
constexpr int kGM = 64, kGN = 64, kGK = 16, kGPad = 20;  // row stride 20 doubles: conflict-free fragments

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes)
               : "memory");
}

// 64 x 64 tile of C per CTA, four warps of 32 x 32 (4 x 4 DMMA tiles), k in
// chunks of 16 double-buffered with cp.async (zero fill past m, n, kd).
// Batched (g.splits == 0): blockIdx.z is the batch.  Batch sum (g.splits >
// 0): blockIdx.z is a split of the batches, the CTA sums its batches' products
// (fixed order) into slab z of C.
__global__ void __launch_bounds__(128) gemm_tn_kernel(GemmTN g) {
  __shared__ __align__(16) double As[2][kGM][kGPad];
  __shared__ __align__(16) double Bs[2][kGN][kGPad];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gm = lane >> 2, gk = lane & 3;
  const int m0 = blockIdx.x * kGM, n0 = blockIdx.y * kGN, z = blockIdx.z;
  if (g.lower && m0 + kGM - 1 < n0) return;  // tile entirely above the diagonal
  int b0 = z, nb = 1;
  if (g.splits > 0) {
    const int per = (g.batch + g.splits - 1) / g.splits;
    b0 = z * per;
    nb = min(g.batch, b0 + per) - b0;
  }
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int nk = (g.kd + kGK - 1) / kGK;
  auto load = [&](int c, int buf) {
    const int b = b0 + c / nk, k0 = (c % nk) * kGK;
    const double* A = g.A + size_t(b) * g.sa;
    const double* B = g.B + size_t(b) * g.sb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 128, row = e >> 3, k = k0 + 2 * (e & 7);
      const int kb = k < g.kd ? (g.kd - k >= 2 ? 16 : 8) : 0;
      {
        const int i = m0 + row;
        const int bytes = i < g.m ? kb : 0;
        cp_async16(&As[buf][row][2 * (e & 7)], bytes ? A + size_t(i) * g.lda + k : A, bytes);
      }
      {
        const int j = n0 + row;
        const int bytes = j < g.n ? kb : 0;
        cp_async16(&Bs[buf][row][2 * (e & 7)], bytes ? B + size_t(j) * g.ldb + k : B, bytes);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nc = nb * nk;
  if (nc > 0) load(0, 0);
  for (int c = 0; c < nc; ++c) {
    const int buf = c & 1;
    if (c + 1 < nc) {
      load(c + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGK / 4; ++ks) {
      const int kk = ks * 4 + gk;
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][wm + i * 8 + gm][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[buf][wn + j * 8 + gm][kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
    __syncthreads();
  }
  double* C = g.C + size_t(z) * g.sc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + gm;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = n0 + wn + j * 8 + 2 * gk + v;
        if (col < g.n) C[size_t(col) * g.ldc + r] = g.alpha * acc[i][j][v];
      }
  }
}

// Row-major batched C = alpha A B + beta C (the tail's 2 x 2 block inversion,
// kkt_kernels.cu): 64 x 64 C tiles, four warps of 32 x 32, k chunks of 16,
// 8-byte cp.async staging (the tail's rows need not be 16-byte aligned).
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes)
               : "memory");
}
constexpr int kNnPadB = 4;  // Bs row stride 64 + 4 doubles: conflict-free fragments

__global__ void __launch_bounds__(128) gemm_nn_kernel(GemmNN g) {
  __shared__ __align__(16) double As[2][kGM][kGPad];
  __shared__ __align__(16) double Bs[2][kGK][kGN + kNnPadB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gm = lane >> 2, gk = lane & 3;
  const int m0 = blockIdx.x * kGM, n0 = blockIdx.y * kGN, b = blockIdx.z;
  const double* A = g.A + size_t(b) * g.sa;
  const double* B = g.B + size_t(b) * g.sb;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  auto load = [&](int k0, int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * 128;  // 1024 elements of each tile
      {
        const int row = e >> 4, k = k0 + (e & 15), i = m0 + row;
        const bool ok = i < g.m && k < g.kd;
        cp_async8(&As[buf][row][e & 15], ok ? A + size_t(i) * g.lda + k : A, ok ? 8 : 0);
      }
      {
        const int kr = e >> 6, j = n0 + (e & 63), k = k0 + kr;
        const bool ok = j < g.n && k < g.kd;
        cp_async8(&Bs[buf][kr][e & 63], ok ? B + size_t(k) * g.ldb + j : B, ok ? 8 : 0);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (g.kd + kGK - 1) / kGK;
  if (nk > 0) load(0, 0);
  for (int c = 0; c < nk; ++c) {
    const int buf = c & 1;
    if (c + 1 < nk) {
      load((c + 1) * kGK, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGK / 4; ++ks) {
      const int kk = ks * 4 + gk;
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][wm + i * 8 + gm][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[buf][kk][wn + j * 8 + gm];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
    __syncthreads();
  }
  double* C = g.C + size_t(b) * g.sc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + gm;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = n0 + wn + j * 8 + 2 * gk + v;
        if (col < g.n) {
          double* cp = C + size_t(r) * g.ldc + col;
          *cp = g.alpha * acc[i][j][v] + (g.beta != 0.0 ? g.beta * *cp : 0.0);
        }
      }
  }
}

}  // namespace

template <int G>
static void launch_reach_g(const ReachDev& p, int M, const double* F, long long nnz_f,
                           const double* gu, long long gu_nnz, double* yn, double* yt,
                           cudaStream_t st) {
  constexpr int NG = 32 / G, SEG = 8 * G;
  const size_t smem = size_t(kReachWarps) * NG * (size_t(p.ymax) * 8 + SEG * 12);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reach_solve_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  const int cols_per_cta = kReachWarps * NG;
  reach_solve_kernel<G><<<dim3((p.n_u + cols_per_cta - 1) / cols_per_cta, M), 32 * kReachWarps,
                          smem, st>>>(p, F, nnz_f, gu, gu_nnz, yn, yt);
}

void launch_reach_solve(const ReachDev& p, int M, const double* F, long long nnz_f,
                        const double* gu, long long gu_nnz, double* yn, double* yt,
                        cudaStream_t st) {
  if (M <= 0 || p.n_u <= 0) return;
  switch (p.group) {
    case 4: launch_reach_g<4>(p, M, F, nnz_f, gu, gu_nnz, yn, yt, st); break;
    case 8: launch_reach_g<8>(p, M, F, nnz_f, gu, gu_nnz, yn, yt, st); break;
    case 16: launch_reach_g<16>(p, M, F, nnz_f, gu, gu_nnz, yn, yt, st); break;
    default: launch_reach_g<32>(p, M, F, nnz_f, gu, gu_nnz, yn, yt, st); break;
  }
  note_launch();
  check_launch("reach_solve");
}

void launch_xt_sparse(const double* WT, int ldw, long long sw, const double* ytc, int nnz_yt,
                      const int* yt_ptr, const int* yt_row, int n_u, int tl, int M, double* xt,
                      int ldy, cudaStream_t st) {
  if (M <= 0 || n_u <= 0 || tl <= 0) return;
  auto smem_of = [&](int rpl) {
    return size_t(tl) * kXtRows * rpl * sizeof(double) + 32 * kXtWarps * sizeof(double2) +
           size_t(n_u + 1) * sizeof(int);
  };
  // two rows per lane where the 64-row W' block fits (1354/256, tl 272:
  // reduce_pre 1.01 -> 0.95 ms against one row per lane; BIPM_XT_RPL=1|2)
  int rpl = 2;
  if (const char* e = std::getenv("BIPM_XT_RPL")) rpl = std::atoi(e) == 2 ? 2 : 1;
  if (smem_of(rpl) > 227 * 1024) rpl = 1;
  const size_t smem = smem_of(rpl);
  const int R = kXtRows * rpl;
  if (rpl == 2) {
    cudaFuncSetAttribute(xt_sparse_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    xt_sparse_kernel<2><<<dim3((tl + R - 1) / R, M), 32 * kXtWarps, smem, st>>>(
        WT, ldw, sw, ytc, nnz_yt, yt_ptr, yt_row, n_u, tl, xt, ldy);
  } else {
    cudaFuncSetAttribute(xt_sparse_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    xt_sparse_kernel<1><<<dim3((tl + R - 1) / R, M), 32 * kXtWarps, smem, st>>>(
        WT, ldw, sw, ytc, nnz_yt, yt_ptr, yt_row, n_u, tl, xt, ldy);
  }
  note_launch();
  check_launch("xt_sparse");
}

void launch_gemm_nn(const GemmNN& g, cudaStream_t st) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
  gemm_nn_kernel<<<dim3((g.m + kGM - 1) / kGM, (g.n + kGN - 1) / kGN, g.batch), 128, 0, st>>>(g);
  note_launch();
  check_launch("gemm_nn");
}

void launch_gemm_tn(const GemmTN& g, cudaStream_t st) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
  gemm_tn_kernel<<<dim3((g.m + kGM - 1) / kGM, (g.n + kGN - 1) / kGN,
                       g.splits > 0 ? g.splits : g.batch),
                   128, 0, st>>>(g);
  note_launch();
  check_launch("gemm_tn");
}

}  // namespace bipm
