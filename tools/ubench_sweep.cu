// Microbenchmark of one sweep level of the streamed reduction, in isolation:
// a synthetic level of `units` rows x `ent` entries on a K = 8 panel held in
// shared memory, run by a team of T warps; reports cycles per level.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2301_04869_b200/csrc \
//   -o tools/ubench_sweep_bin tools/ubench_sweep.cu
#include <cstdio>

#include "kernels/reduce_stream.cu"

namespace bipm {
namespace {

constexpr int K = 8, C = 512;

// instrumented copy of step_sweep's unit loop (one level, team T)
__device__ long long g_ph[8];
__device__ void sweep_timed(int e_x, int e_y, int lg, int T, unsigned items, unsigned col,
                            unsigned v, unsigned xb, int tid, int variant) {
  using Pn = Panel<K>;
  const int warp = tid >> 5, lane = tid & 31;
  if (warp >= T) return;
  const int g = 1 << lg, upw = 32 >> lg;
  const int nch = (e_y - e_x + upw - 1) >> (5 - lg);
  const int sub = lane & (g - 1);
  long long ph[5] = {0, 0, 0, 0, 0};
  for (int c = warp; c < nch; c += T) {
    long long t0 = clock64();
    const int unit = e_x + c * upw + (lane >> lg);
    const bool active = unit < e_y;
    double a[Pn::CW];
#pragma unroll
    for (int q = 0; q < Pn::CW; ++q) a[q] = 0.0;
    int4 m = make_int4(0, 0, 0, 0);
    if (active) m = ldsi4(items + 16 * unit);
    long long t1 = clock64();
    if (active) {
      int t = m.y + sub;
      if (variant == 1) {
        for (; t + 3 * g < m.z; t += 4 * g) {
          int w[4];
          double vv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) w[u] = colw<K>(col, t + u * g);
#pragma unroll
          for (int u = 0; u < 4; ++u) vv[u] = lds1(v + 8 * (t + u * g));
#pragma unroll
          for (int u = 0; u < 4; ++u) Pn::fma(a, vv[u], xb, w[u], 0);
        }
      }
      for (; t + g < m.z; t += 2 * g) {
        const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
        const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
        Pn::fma(a, v0, xb, w0, 0);
        Pn::fma(a, v1, xb, w1, 0);
      }
      if (t < m.z) Pn::fma(a, lds1(v + 8 * t), xb, colw<K>(col, t), 0);
    }
    // consume a[] so the timing includes the FMAs
    double sum = 0;
#pragma unroll
    for (int q = 0; q < Pn::CW; ++q) sum += a[q];
    if (sum == 12345.0) a[0] = 1;
    long long t2 = clock64();
    reduce_lanes<Pn::CW>(a, g);
    long long t3 = clock64();
    if (active && sub == 0) {
      double x[Pn::CW];
      Pn::load(x, xb, m.x, 0);
#pragma unroll
      for (int q = 0; q < Pn::CW; ++q) x[q] -= a[q];
      Pn::store(x, xb, m.x, 0);
    }
    __syncwarp();
    long long t4 = clock64();
    ph[0] += t1 - t0;
    ph[1] += t2 - t1;
    ph[2] += t3 - t2;
    ph[3] += t4 - t3;
    ph[4] += 1;
  }
  if (tid == 0)
    for (int i = 0; i < 5; ++i) g_ph[i] = ph[i];
}

__global__ void __launch_bounds__(C) level_bench(int n_x, int units, int ent, int lg, int T,
                                                 int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* X = reinterpret_cast<double*>(sm);
  unsigned char* ring = sm + size_t(n_x) * K * 8;
  // step layout: level record | items | col | values
  int4* levr = reinterpret_cast<int4*>(ring);
  int4* items = levr + 1;
  unsigned short* col = reinterpret_cast<unsigned short*>(items + units);  // 16-bit panel rows
  double* v = reinterpret_cast<double*>(col + ((units * ent + 7) & ~7));
  const int tid = threadIdx.x;
  for (int i = tid; i < n_x * K; i += C) X[i] = 1e-3 * (i % 97);
  for (int u = tid; u < units; u += C)
    items[u] = make_int4(Panel<K>::word((u * 37) % n_x), u * ent, (u + 1) * ent, 0);
  for (int t = tid; t < units * ent; t += C) {
    col[t] = (unsigned short)((t * 7919 + 13) % n_x);
    v[t] = 1e-6 * (t % 31);
  }
  if (tid == 0) levr[0] = make_int4(0, units, lg, 1);
  __syncthreads();
  Hdr h{};
  h.aux0 = T;
  h.n_lev = 1;
  h.flags = 0;
  Tracer tr;
  const unsigned xb = smem_u32(X);
  const unsigned lev = smem_u32(levr), it = smem_u32(items), cl = smem_u32(col),
                 vv = smem_u32(v);
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) step_sweep<K, C>(h, lev, it, cl, vv, xb, tid, tr, 0);
  __syncthreads();
  const long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / reps;
  for (int variant = 0; variant < 2; ++variant) {
    __syncthreads();
    sweep_timed(0, units, lg, T, it, cl, vv, xb, tid, variant);
    __syncthreads();
    if (tid == 0)
      for (int i = 0; i < 5; ++i) out[1 + variant * 5 + i] = g_ph[i];
  }
}

}  // namespace
}  // namespace bipm

int main() {
  using namespace bipm;
  long long* d;
  cudaMalloc(&d, 128);
  const int n_x = 2447;
  const size_t smem = size_t(n_x) * K * 8 + 60 * 1024;
  cudaFuncSetAttribute(level_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  struct Cfg { int units, ent, lg, T; };
  const Cfg cfgs[] = {{5, 40, 2, 1},  {5, 40, 3, 2},  {5, 40, 4, 4},  {5, 40, 5, 8},
                      {8, 10, 1, 1},  {8, 10, 2, 1},  {8, 10, 3, 2},  {8, 10, 4, 4},
                      {64, 3, 0, 2},  {64, 3, 1, 4},  {64, 3, 2, 8},
                      {244, 3, 0, 8}, {244, 3, 1, 16}, {100, 10, 1, 8}, {100, 10, 2, 16}};
  for (const Cfg& c : cfgs) {
    level_bench<<<1, C, smem>>>(n_x, c.units, c.ent, c.lg, c.T, 200, d);
    long long h[11] = {0};
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("units %4d ent %3d lg %d T %2d : %6lld cycles/level | warp0 per chunk: item %lld loop %lld "
           "reduce %lld store %lld (chunks %lld) | unroll4 loop %lld\n",
           c.units, c.ent, c.lg, c.T, h[0], h[1] / h[5], h[2] / h[5], h[3] / h[5], h[4] / h[5],
           h[5], h[7] / h[10]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
