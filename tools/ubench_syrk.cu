// cuBLAS FP64 SYRKX / GEMM rate for the reduction's T'(K~T) shape:
// n = n_u, k = scenarios * n_x.   nvcc -O3 -o tools/ubench_syrk_bin tools/ubench_syrk.cu -lcublas
#include <cublas_v2.h>
#include <cstdio>
#include <vector>
int main() {
  const int cfg[][2] = {{519, 256 * 2447}, {519, 32 * 2447}, {1019, 64 * 5227}};
  cublasHandle_t h;
  cublasCreate(&h);
  for (auto& c : cfg) {
    const int n = c[0];
    const long long k = c[1];
    double *A, *B, *C;
    cudaMalloc(&A, sizeof(double) * n * k);
    cudaMalloc(&B, sizeof(double) * n * k);
    cudaMalloc(&C, sizeof(double) * n * n);
    cudaMemset(A, 0, sizeof(double) * n * k);
    cudaMemset(B, 0, sizeof(double) * n * k);
    const double al = -1.0, be = 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
      for (int it = 0; it < 4; ++it) {
        if (it == 1) cudaEventRecord(e0);
        if (mode == 0)
          cublasDsyrkx(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n, int(k), &al, A, int(k), B, int(k), &be, C, n);
        else
          cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, n, n, int(k), &al, A, int(k), B, int(k), &be, C, n);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      const double fl = (mode == 0 ? 1.0 : 2.0) * double(n) * n * k;
      printf("%s n %d k %lld: %.3f ms  %.1f TFLOP/s\n", mode == 0 ? "syrkx" : "gemm ", n, k, ms,
             fl / ms * 1e-9);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
