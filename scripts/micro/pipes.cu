// Per-SM instruction throughput probe (MUFU ex2/rsqrt, f32->f16 pack, HADD2.F32, FADD, FMNMX).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cstdint>

template <int OP>
__global__ void probe(float *out, int iters, unsigned long long *cyc) {
  float v[8];
  uint32_t u[8];
  double dv[8];
  for (int i = 0; i < 8; ++i) dv[i] = 0.5 + threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 8; ++i) { v[i] = 0.001f * (threadIdx.x + i); u[i] = threadIdx.x * 7 + i; }
  __syncthreads();
  unsigned long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i])); }
      if constexpr (OP == 1) { asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i])); }
      if constexpr (OP == 2) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(v[i]), "f"(__uint_as_float(u[i]))); }
      if constexpr (OP == 3) { float f; asm volatile("{.reg .b16 lo, hi; mov.b32 {lo,hi}, %1; cvt.f32.f16 %0, lo;}" : "=f"(f) : "r"(u[i])); u[i] = __float_as_uint(f); }
      if constexpr (OP == 4) { asm volatile("add.f32 %0, %0, 0f3F800001;" : "+f"(v[i])); }
      if constexpr (OP == 5) { asm volatile("max.f32 %0, %0, 0f3F800001;" : "+f"(v[i])); }
      if constexpr (OP == 6) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i])); asm volatile("add.f32 %0, %0, 0f3F800001;" : "+f"(v[(i+4)&7])); }
      if constexpr (OP == 7) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i])); asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(v[(i+3)&7]), "f"(v[(i+5)&7])); }
      if constexpr (OP == 8) { asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(v[i])); }
      if constexpr (OP == 9) { asm volatile("ex2.approx.f32 %0, %0;" : "+f"(v[i])); }
      if constexpr (OP == 10) { asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i])); }
      if constexpr (OP == 11) { asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[i])); }
      if constexpr (OP == 12) { asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i])); }
      if constexpr (OP == 13) { double dd = v[i]; asm volatile("fma.rn.f64 %0, %0, 0d3FF0000000000001, 0d3FE0000000000000;" : "+d"(dd)); v[i] = float(dd); }
      if constexpr (OP == 16) { asm volatile("and.b32 %0, %0, 0xFFFFE001;" : "+r"(u[i])); }
      if constexpr (OP == 17) { float e; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(v[i])); float h = __uint_as_float(__float_as_uint(e) & 0xFFFFE000u); float l = e - h; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(h), "f"(l)); v[i] = __uint_as_float(u[i]) + 1e-3f; }
      if constexpr (OP == 15) { asm volatile("fma.rn.f64 %0, %0, 0d3FF0000000000001, 0d3FE0000000000000;" : "+d"(dv[i])); }
      if constexpr (OP == 14) { double dd; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(dd) : "f"(v[i])); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(v[i]) : "d"(dd)); }
    }
  }
  unsigned long long c1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i] + __uint_as_float(u[i]) + float(dv[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  float *out; unsigned long long *cyc;
  const int warps = 16, iters = 4096, blocks = 148;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&cyc, blocks * 8);
  const char *names[] = {"ex2.ftz", "rsqrt", "cvt.f16x2.f32", "cvt.f32.f16", "fadd", "fmax", "ex2+fadd", "ex2+cvtpack", "ffma", "ex2(noftz)", "ex2.bf16x2", "tanh", "sqrt", "dfma(+2cvt)", "cvt f32<->f64", "dfma", "lop3", "rbf-entry-chain"};
  for (int op = 0; op < 18; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
#define L(K) case K: probe<K><<<blocks, warps * 32>>>(out, iters, cyc); break;
        L(0) L(1) L(2) L(3) L(4) L(5) L(6) L(7) L(8) L(9) L(10) L(11) L(12) L(13) L(14) L(15) L(16) L(17)
      }
    }
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int b = 0; b < blocks; ++b) c += h[b]; c /= blocks;
    const double ops = double(warps) * 32 * iters * 8;   // per SM (one block per SM)
    printf("%-14s %8.2f lanes/clk/SM  (%.0f cycles)\n", names[op], ops / c, c);
  }
  return 0;
}
