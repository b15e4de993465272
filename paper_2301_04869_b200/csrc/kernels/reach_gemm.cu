// Forward half of X = G_x^{-1} P G_u for all control columns of every
// scenario (host/stream_plan.hpp ReachPlan), and the batched FP64 DMMA GEMM
// that applies the dense tail inverse W to it.
//
// The reference solves every column of every tile with the whole L factor
// (reduce_group, kkt.cpp:388-404: spsm over n_x rows per column); column u
// of L^{-1} P G_u is nonzero only on the reach of G_u's rows in the graph of
// L, a few etree paths.  reach_solve_kernel walks exactly those rows (one
// warp per (scenario, column), the column's y_N in shared memory, factor
// values staged a segment at a time with all loads in flight), then gathers
// the tail rows y_T = (P G_u)_T - L_TN y_N.  gemm_tn_kernel then forms
// X_T = W y_T for all n_u columns at once (W read once per scenario instead
// of once per column tile of the reduction).
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

constexpr int kReachWarps = 8;
constexpr int kReachSeg = 256;  // staged entries per warp

// dynamic shared memory per warp: y_N of its column (ymax doubles), then the
// staged segment (kReachSeg factor values + kReachSeg source indices)
__global__ void __launch_bounds__(32 * kReachWarps)
    reach_solve_kernel(ReachDev p, const double* __restrict__ F, long long nnz_f,
                       const double* __restrict__ gu, long long gu_nnz, double* __restrict__ yn,
                       double* __restrict__ yt) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * kReachWarps + warp, s = blockIdx.y;
  if (u >= p.n_u) return;
  const int ymax = p.ymax;
  unsigned char* wb = smem + size_t(warp) * (size_t(ymax) * 8 + kReachSeg * 12);
  double* y = reinterpret_cast<double*>(wb);
  double* fv = y + ymax;
  int* src = reinterpret_cast<int*>(fv + kReachSeg);
  const double* Fs = F + size_t(s) * nnz_f;
  const double* gs = gu + size_t(s) * gu_nnz;
  double* ts = yt + (size_t(s) * p.n_u + u) * p.ldy;
  for (int i = lane; i < p.ldy; i += 32) ts[i] = 0.0;
  const int ob = p.op_ptr[u], oe = p.op_ptr[u + 1];
  for (int o = ob; o < oe;) {
    // segment: up to 32 ops whose entries fit the staging buffer (an op with
    // more entries than that runs alone, straight from global memory)
    const int4 rec = o + lane < oe ? p.ops[o + lane] : make_int4(0, -1, 0, 0x7fffffff);
    const int e0 = __shfl_sync(0xffffffffu, rec.z, 0);
    // entries are contiguous and increasing over the ops: a prefix of lanes fits
    const unsigned fits = __ballot_sync(0xffffffffu, o + lane < oe && rec.w - e0 <= kReachSeg);
    const bool staged = (fits & 1u) != 0;
    const int nseg = staged ? __popc(fits) : 1;
    const double bval = rec.y >= 0 ? gs[rec.y] : 0.0;
    const int e1 = __shfl_sync(0xffffffffu, rec.w, nseg - 1);
    if (staged) {
      for (int e = e0 + lane; e < e1; e += 32) {
        const int2 en = p.ent[e];
        src[e - e0] = en.x;
        fv[e - e0] = Fs[en.y];
      }
      __syncwarp();
    }
    for (int i = 0; i < nseg; ++i) {
      const int dest = __shfl_sync(0xffffffffu, rec.x, i);
      const int eb = __shfl_sync(0xffffffffu, rec.z, i), ee = __shfl_sync(0xffffffffu, rec.w, i);
      const double b = __shfl_sync(0xffffffffu, bval, i);
      double a = 0.0;
      if (staged) {
        for (int e = eb - e0 + lane; e < ee - e0; e += 32) a += fv[e] * y[src[e]];
      } else {
        for (int e = eb + lane; e < ee; e += 32) {
          const int2 en = p.ent[e];
          a += Fs[en.y] * y[en.x];
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) {
        if (dest >= 0)
          y[dest] = b - a;
        else
          ts[-1 - dest] = b - a;
      }
      __syncwarp();
    }
    o += nseg;
  }
  double* ys = yn + size_t(s) * p.nnz_yn + p.yn_ptr[u];
  const int ny = p.yn_ptr[u + 1] - p.yn_ptr[u];
  for (int i = lane; i < ny; i += 32) ys[i] = y[i];
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
// chunks of 16 double-buffered with cp.async (zero fill past m, n, kd)
__global__ void __launch_bounds__(128) gemm_tn_kernel(GemmTN g) {
  __shared__ __align__(16) double As[2][kGM][kGPad];
  __shared__ __align__(16) double Bs[2][kGN][kGPad];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gm = lane >> 2, gk = lane & 3;
  const int m0 = blockIdx.x * kGM, n0 = blockIdx.y * kGN, b = blockIdx.z;
  const double* A = g.A + size_t(b) * g.sa;
  const double* B = g.B + size_t(b) * g.sb;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  auto load = [&](int k0, int buf) {
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
  const int nk = (g.kd + kGK - 1) / kGK;
  load(0, 0);
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
      for (int j = 0; j < 4; ++j) bb[j] = Bs[buf][wn + j * 8 + gm][kk];
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
        if (col < g.n) C[size_t(col) * g.ldc + r] = acc[i][j][v];
      }
  }
}

}  // namespace

void launch_reach_solve(const ReachDev& p, int M, const double* F, long long nnz_f,
                        const double* gu, long long gu_nnz, double* yn, double* yt,
                        cudaStream_t st) {
  if (M <= 0 || p.n_u <= 0) return;
  const size_t smem = size_t(kReachWarps) * (size_t(p.ymax) * 8 + kReachSeg * 12);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reach_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  reach_solve_kernel<<<dim3((p.n_u + kReachWarps - 1) / kReachWarps, M), 32 * kReachWarps, smem,
                       st>>>(p, F, nnz_f, gu, gu_nnz, yn, yt);
  note_launch();
  check_launch("reach_solve");
}

void launch_gemm_tn(const GemmTN& g, cudaStream_t st) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
  gemm_tn_kernel<<<dim3((g.m + kGM - 1) / kGM, (g.n + kGN - 1) / kGN, g.batch), 128, 0, st>>>(g);
  note_launch();
  check_launch("gemm_tn");
}

}  // namespace bipm
