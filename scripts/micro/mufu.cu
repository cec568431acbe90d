// MUFU throughput per op on this GPU: RSQ, SQRT, EX2, LG2, and the f16x2 EX2,
// full occupancy, 8 independent chains per thread. Prints warp-instructions
// per clock per SM (a pipe of L lanes/clk/SM gives L/32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu mufu.cu && ./mufu
#include <cstdio>
#include <cuda_fp16.h>

template <int OP>
__device__ __forceinline__ float op(float x) {
  float y;
  if (OP == 0) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 1) asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 3) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 4) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 5) {
    unsigned u = __float_as_uint(x), v;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(v) : "r"(u));
    y = __uint_as_float(v);
  }
  if (OP == 6) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int OP>
__global__ void bench(float *out, int iters, long long *clk) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0f + 0.001f * (threadIdx.x + k);
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = op<OP>(a[k]);
  }
  __syncthreads();
  long long c1 = clock64();
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int OP>
void run(const char *name) {
  float *out;
  long long *clk, h[148];
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&clk, 148 * 8);
  const int threads = 1024, iters = 4096;
  bench<OP><<<148, threads>>>(out, iters, clk);
  bench<OP><<<148, threads>>>(out, iters, clk);
  cudaDeviceSynchronize();
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double warp_inst = double(threads / 32) * iters * 8;
  printf("%-10s %.3f warp-inst/clk/SM  (%.1f lanes/clk/SM)\n", name, warp_inst / h[0],
         32 * warp_inst / h[0]);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<0>("rsqrt");
  run<1>("sqrt");
  run<2>("ex2");
  run<3>("lg2");
  run<4>("rcp");
  run<5>("ex2.f16x2");
  run<6>("tanh");
  return 0;
}
