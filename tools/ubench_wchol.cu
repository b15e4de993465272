// warp_chol32 in isolation.  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a \
//   -I paper_2301_04869_b200/csrc -o tools/ubench_wchol_bin tools/ubench_wchol.cu
#include <cstdio>
#include "kernels/dense_chol.cu"
namespace bipm {
__global__ void wchol(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  __shared__ double colbuf[kNb];
  double a[kNb];
  long long t0 = 0, t1 = 0;
  int f = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < kNb; ++c) a[c] = c <= lane ? (c == lane ? 40.0 + r : 1.0 / (1 + c + lane)) : 0.0;
    __syncwarp();
    if (r == 1) t0 = clock64();
    f += warp_chol32(a, 32, lane, colbuf);
    __syncwarp();
    if (r == reps - 1) t1 = clock64();
  }
  double s = f;
#pragma unroll
  for (int c = 0; c < kNb; ++c) s += a[c];
  out[lane] = s;
  if (lane == 0) cyc[0] = (t1 - t0) / (reps - 2);
}
}  // namespace bipm
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 256);
  cudaMalloc(&c, 8);
  bipm::wchol<<<1, 32>>>(o, c, 20);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("warp_chol32: %lld cycles per call; %s\n", h, cudaGetErrorString(cudaDeviceSynchronize()));
}
