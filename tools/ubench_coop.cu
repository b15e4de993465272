// Cost of the cooperative Cholesky's pieces: grid.sync() alone vs the full
// factorisation.  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a \
//   -I paper_2301_04869_b200/csrc -o tools/ubench_coop_bin tools/ubench_coop.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>

#include "kernels/dense_chol.cu"

namespace bipm {
__global__ void syncs_only(int n_sync) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  for (int i = 0; i < n_sync; ++i) g.sync();
}
}  // namespace bipm

int main() {
  using namespace bipm;
  for (int grid : {8, 36, 148}) {
    int ns = 51;
    void* args[] = {&ns};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)syncs_only, dim3(grid), dim3(128), args, 0, 0);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) cudaLaunchCooperativeKernel((void*)syncs_only, dim3(grid), dim3(128), args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid %3d: 51 grid syncs %.1f us per launch\n", grid, ms * 100);
  }
  for (int n : {519, 1019}) {
    std::vector<double> h(size_t(n) * n);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) h[size_t(j) * n + i] = (i == j ? n + 1.0 : 1.0 / (1 + i + j));
    double* K;
    int* info;
    cudaMalloc(&K, h.size() * 8);
    cudaMalloc(&info, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < 6; ++r) {
      cudaMemcpy(K, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(a);
      launch_blocked_cholesky(K, n, info, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) tot += ms;
    }
    printf("n %d: cooperative factor %.1f us\n", n, tot / 5 * 1000);
    long long* st;
    cudaMalloc(&st, 256 * 8);
    cudaMemcpyToSymbol(g_chol_stamps, &st, sizeof(st));
    cudaMemcpy(K, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    launch_blocked_cholesky(K, n, info, 0);
    cudaDeviceSynchronize();
    std::vector<long long> hs(256);
    cudaMemcpy(hs.data(), st, 256 * 8, cudaMemcpyDeviceToHost);
    long long nulls = 0;
    cudaMemcpyToSymbol(g_chol_stamps, &nulls, sizeof(st));
    // per panel: [start, diag done, after sync, trsm done, after sync, update done]
    double d = 0, s1 = 0, t = 0, s2 = 0, u = 0;
    int np = 0;
    double dl = 0;
    for (int k = 0; k + 6 < 256 && hs[k + 6] > 0; k += 7, ++np) {
      dl += hs[k + 1] - hs[k]; d += hs[k + 2] - hs[k + 1]; s1 += hs[k + 3] - hs[k + 2];
      t += hs[k + 4] - hs[k + 3]; s2 += hs[k + 5] - hs[k + 4]; u += hs[k + 6] - hs[k + 5];
    }
    printf("  per panel (cycles, %d panels): diag load %.0f factor %.0f sync %.0f trsm %.0f sync %.0f "
           "update %.0f\n", np, dl / np, d / np, s1 / np, t / np, s2 / np, u / np);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
