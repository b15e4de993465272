// Shared-memory gather bandwidth of 64-byte panel rows (K = 8 doubles):
//   lane-per-row  : each lane reads a whole random row (4 x LDS.128)
//   quad-per-row  : the 4 lanes of a quad read the 4 chunks of one random row
//                   (1 x LDS.128 per lane, 8 rows per warp instruction)
// bytes per clock per SM with 16 warps.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubq tools/ubench_quad.cu
#include <cstdio>

__global__ void k_lane(double* out, long long* cyc, int n) {
  extern __shared__ double X[];
  const int rows = 2448;
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) X[i] = i * 1e-6;
  __syncthreads();
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned r = (threadIdx.x + 7) * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    r = r * 1664525u + 1013904223u;
    const int row = (r >> 8) % rows;
    const int s = (row >> 1) & 3;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 x = reinterpret_cast<const double2*>(X + row * 8)[q ^ s];
      a[2 * q] += x.x;
      a[2 * q + 1] += x.y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double sum = 0;
  for (int q = 0; q < 8; ++q) sum += a[q];
  out[threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int U>
__global__ void k_quad(double* out, long long* cyc, int n) {
  extern __shared__ double X[];
  const int rows = 2448;
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) X[i] = i * 1e-6;
  __syncthreads();
  double a0 = 0, a1 = 0;
  const int quad = threadIdx.x >> 2, ql = threadIdx.x & 3;
  unsigned r = (quad + 7) * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < n; i += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      r = r * 1664525u + 1013904223u;
      const int row = (r >> 8) % rows;
      const int s = (row >> 1) & 3;
      const double2 x = reinterpret_cast<const double2*>(X + row * 8)[ql ^ s];
      a0 += x.x;
      a1 += x.y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  long long h[4];
  const int n = 4096, smem = 2448 * 64;
  cudaFuncSetAttribute(k_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_quad<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int w : {4, 8, 16}) {
    k_lane<<<1, 32 * w, smem>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("lane-per-row %2d warps: %.1f B/clk\n", w, 64.0 * 32 * w * n / h[0]);
    k_quad<4><<<1, 32 * w, smem>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("quad-per-row %2d warps: %.1f B/clk\n", w, 64.0 * 8 * w * n / h[0]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
