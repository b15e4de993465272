// Per-panel phase clocks of the cooperative K_hat Cholesky (CTA 0's view):
// diagonal-block load, warp factor, grid barrier, L21 solve, barrier, trailing
// DMMA update + barrier.  Random SPD matrix of order n (default 519).
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2301_04869_b200/csrc \
//   -o tools/ubench_chol_bin tools/ubench_chol.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <algorithm>
#include <vector>

#include "kernels/dense_chol.cu"

namespace bipm {
void note_launch() {}
}  // namespace bipm

int main(int argc, char** argv) {
  using namespace bipm;
  const int n = argc > 1 ? std::atoi(argv[1]) : 519;
  std::vector<double> A(size_t(n) * n);
  srand(1);
  std::vector<double> B(size_t(n) * n);
  for (auto& b : B) b = rand() / double(RAND_MAX) - 0.5;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = (i == j) ? n : 0.0;
      for (int k = 0; k < 16; ++k) s += B[size_t(k) * n + i] * B[size_t(k) * n + j];
      A[size_t(j) * n + i] = s;
    }
  double* dK;
  int* info;
  long long* st;
  cudaMalloc(&dK, A.size() * 8);
  cudaMalloc(&info, 16);
  cudaMalloc(&st, 256 * 8);
  cudaMemcpyToSymbol(g_chol_stamps, &st, sizeof(st));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dK, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(st, 0, 256 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    launch_blocked_cholesky(dK, n, info, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(256);
    cudaMemcpy(h.data(), st, 256 * 8, cudaMemcpyDeviceToHost);
    int hi[2];
    cudaMemcpy(hi, info, 8, cudaMemcpyDeviceToHost);
    printf("rep %d: %.3f ms info %d\n", rep, ms, hi[0]);
    if (rep == 2) {
      // 7 stamps per panel: s0 load s1 chol s2 sync s3 trsm s4 sync s5 update s6 (sync)
      long long tot[7] = {0};
      int np = 0;
      for (int p = 0; 7 * p + 6 < 256 && h[7 * p]; ++p, ++np) {
        for (int k = 0; k < 6; ++k) tot[k] += h[7 * p + k + 1] - h[7 * p + k];
        if (h[7 * p + 7]) tot[6] += h[7 * p + 7] - h[7 * p + 6];
      }
      const char* nm[7] = {"load", "warp_chol", "sync1", "trsm", "sync2", "update", "sync3"};
      printf("panels %d, cycles per panel:", np);
      for (int k = 0; k < 7; ++k) printf(" %s %lld", nm[k], tot[k] / (np ? np : 1));
      printf("\n");
    }
  }
  {
    // residual of L L' against A (lower triangle; the shift is <= 1e-13 |A|)
    std::vector<double> L(A.size());
    cudaMemcpy(L.data(), dK, A.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0.0, amax = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = j; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k <= j; ++k) s += L[size_t(k) * n + i] * L[size_t(k) * n + j];
        err = std::max(err, std::fabs(s - A[size_t(j) * n + i]));
        amax = std::max(amax, std::fabs(A[size_t(j) * n + i]));
      }
    printf("residual max|LL'-A|/max|A| = %.3e\n", err / amax);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
