// Batched 100x100 fp64 symmetric eigensolves: cusolverDnXsyevBatched vs this
// repo's Jacobi kernel (sap_sym_eig_batch), 32 matrices (one lookahead batch).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <chrono>
__global__ void spin(unsigned long long ns) {
  const unsigned long long t0 = clock64();
  while (clock64() - t0 < ns * 2) {
  }
}
extern "C" int sap_sym_eig_batch(double *, int64_t, int, int, int, double *, double *, int64_t, int,
                                 int, int *, void *, size_t, void *);
int main(int argc, char **argv) {
  const int r = argc > 1 ? atoi(argv[1]) : 100, count = argc > 2 ? atoi(argv[2]) : 32;
  std::vector<double> h(size_t(count) * r * r);
  srand(1);
  std::vector<double> A(size_t(r) * (r + 3));
  for (int q = 0; q < count; ++q) {
    for (auto &x : A) x = rand() / double(RAND_MAX) - 0.5;
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) {
        double s = 0;
        for (int k = 0; k < r + 3; ++k) s += A[i * (r + 3) + k] * A[j * (r + 3) + k];
        h[size_t(q) * r * r + i * r + j] = s;
      }
  }
  double *dA, *dB, *dW, *dV;
  int *info;
  cudaMalloc(&dA, h.size() * 8); cudaMalloc(&dB, h.size() * 8); cudaMalloc(&dV, h.size() * 8);
  cudaMalloc(&dW, size_t(count) * r * 8); cudaMalloc(&info, count * 4 * 2);
  cudaMemcpy(dB, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // cuSOLVER
  cusolverDnHandle_t H; cusolverDnCreate(&H);
  cusolverDnParams_t P; cusolverDnCreateParams(&P);
  size_t wd = 0, wh = 0;
  cusolverDnXsyevBatched_bufferSize(H, P, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r,
                                    CUDA_R_64F, dA, r, CUDA_R_64F, dW, CUDA_R_64F, &wd, &wh, count);
  void *bd; cudaMalloc(&bd, wd ? wd : 8); std::vector<char> bh(wh ? wh : 8);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(dA, dB, h.size() * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    int st = cusolverDnXsyevBatched(H, P, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r,
                                    CUDA_R_64F, dA, r, CUDA_R_64F, dW, CUDA_R_64F, bd, wd,
                                    bh.data(), wh, info, count);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("cusolverDnXsyevBatched r=%d count=%d: %.3f ms (status %d, ws %zu)\n", r, count, ms, st, wd);
  }
  // does the call block the host until the work queued before it finishes?
  // (a 20 ms spin kernel ahead of it on the same stream)
  printf("host workspace %zu bytes\n", wh);
  for (int it = 0; it < 2; ++it) {
    cudaMemcpy(dA, dB, h.size() * 8, cudaMemcpyDeviceToDevice);
    cudaDeviceSynchronize();
    spin<<<1, 32>>>(20000000ull);
    auto h0 = std::chrono::steady_clock::now();
    cusolverDnXsyevBatched(H, P, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r, CUDA_R_64F,
                           dA, r, CUDA_R_64F, dW, CUDA_R_64F, bd, wd, bh.data(), wh, info, count);
    const double hms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    cudaDeviceSynchronize();
    printf("cusolverDnXsyevBatched host time behind a 20 ms kernel: %.2f ms\n", hms);
  }
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(dA, dB, h.size() * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    int rc = sap_sym_eig_batch(dA, int64_t(r) * r, r, r, count, dW, dV, int64_t(r) * r, r, 40,
                               info + count, nullptr, 0, nullptr);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    std::vector<int> sw(count);
    cudaMemcpy(sw.data(), info + count, count * 4, cudaMemcpyDeviceToHost);
    printf("sap_sym_eig_batch       r=%d count=%d: %.3f ms (rc %d, sweeps %d)\n", r, count, ms, rc, sw[0]);
  }
  return 0;
}
