// Latency / throughput calibration of the instructions the streamed reduction
// is built from (one CTA, one or more warps): dependent DFMA, independent DFMA,
// SHFL of a double, LDS.64, LDS.128 gathers, bar.sync.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench tools/ubench.cu
#include <cstdio>

__global__ void k_dfma_dep(double* out, long long* cyc, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_dfma_ind(double* out, long long* cyc, int n) {
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

__global__ void k_shfl(double* out, long long* cyc, int n) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1 + (i & 15));
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds_dep(double* out, long long* cyc, int n) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 97 + 13) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// 32 lanes gather random 64-byte rows (4 x LDS.128) and FMA them
__global__ void k_gather(double* out, long long* cyc, int n, int swz) {
  extern __shared__ double X[];
  const int rows = 2048;
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) X[i] = i * 1e-6;
  __syncthreads();
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned r = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    r = r * 1664525u + 1013904223u;
    const int row = (r >> 8) % rows;
    const int s = swz ? ((row >> 1) & 3) : 0;
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

__global__ void k_bar(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  long long h[256];
  const int n = 4096;
  auto rep = [&](const char* name, double per) { printf("%-40s %8.2f cycles\n", name, per); };

  k_dfma_dep<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  rep("dependent DFMA latency (1 warp)", double(h[0]) / n);
  for (int w : {1, 4, 16, 32}) {
    k_dfma_ind<<<1, 32 * w>>>(out, cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    char buf[64];
    snprintf(buf, 64, "DFMA warp-instr/cycle/SM (%d warps)", w);
    rep(buf, 8.0 * n * w / double(h[0]));
  }
  k_dfma_ind<<<148, 1024>>>(out, cyc, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  rep("DFMA warp-instr/cycle/SM (148x32 warps)", 8.0 * n * 32 / double(h[0]));
  k_shfl<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  rep("dependent SHFL(double)+DADD (1 warp)", double(h[0]) / n);
  k_lds_dep<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  rep("dependent LDS latency (1 warp)", double(h[0]) / n);
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 64);
  for (int swz : {0, 1})
    for (int w : {1, 4, 16}) {
      k_gather<<<1, 32 * w, 2048 * 64>>>(out, cyc, n, swz);
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      char buf[80];
      snprintf(buf, 80, "row gather 4xLDS.128 swz=%d (%d warps) cyc/iter", swz, w);
      rep(buf, double(h[0]) / n);
    }
  for (int w : {4, 16}) {
    k_bar<<<1, 32 * w>>>(cyc, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    char buf[64];
    snprintf(buf, 64, "__syncthreads (%d warps)", w);
    rep(buf, double(h[0]) / n);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
}
