// FP64 FMA throughput per SM (dependent chains x ILP), and a DMMA m8n8k4 probe.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    dfma_kernel<8><<<sms, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_kernel<8><<<sms, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fmas = double(sms) * threads * iters * 8;
    printf("DFMA %4d threads/SM: %.1f DFMA/clk/SM at 1.965 GHz (%.2f TFLOP/s)\n", threads,
           fmas / (ms * 1e-3) / sms / 1.965e9, 2 * fmas / (ms * 1e-3) / 1e12);
  }
  // latency: one dependent chain
  dfma_kernel<1><<<1, 32>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e0);
  dfma_kernel<1><<<1, 32>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA dependent latency ~%.1f cycles\n", ms * 1e-3 * 1.965e9 / iters);
  return 0;
}
