// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one SM and on all SMs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_dmma_bin tools/ubench_dmma.cu
#include <cstdio>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NA>
__global__ void k_dmma(double* out, long long* cyc, int n) {
  double acc[NA][2];
  for (int a = 0; a < NA; ++a) acc[a][0] = acc[a][1] = 0.0;
  const double x = threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int a = 0; a < NA; ++a) dmma(acc[a][0], acc[a][1], x, y);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < NA; ++a) s += acc[a][0] + acc[a][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(double* out, long long* cyc, int n) {
  double a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int q = 0; q < 8; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  long long h[4];
  const int n = 2048;
  for (int w : {1, 4, 16, 32}) {
    k_dmma<1><<<1, 32 * w>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA 1 chain/warp, %2d warps: %6.2f cycles per DMMA per warp, %6.2f FMA/clk/SM\n", w,
           double(h[0]) / n, 256.0 * n * w / double(h[0]));
    k_dmma<4><<<1, 32 * w>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA 4 chains/warp, %2d warps: %6.2f cycles per DMMA per warp, %6.2f FMA/clk/SM\n", w,
           double(h[0]) / (4.0 * n), 4.0 * 256.0 * n * w / double(h[0]));
    k_dfma<<<1, 32 * w>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains/thread, %2d warps: %6.2f FMA/clk/SM\n", w, 8.0 * 32 * n * w / double(h[0]));
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
