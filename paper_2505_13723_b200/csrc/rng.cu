// Device-side numpy Generator.standard_normal, bit-exact with the host stream.
//
// The reference draws every iteration's Nystrom test matrix on the host,
//   Omega_t = substream(seed, "omega", t).standard_normal((b, r))   solvers.py:384
// (rng.py:14-24: numpy PCG64 seeded by a SeedSequence), 4.4 ms of CPU per
// iteration at b=2000, r=100 -- more than an iteration's GPU time. Here the
// host only seeds the stream (SeedSequence hashing, ~30 us) and passes the
// PCG64 state; the GPU reproduces numpy's sampler exactly:
//
//   PCG64 (XSL-RR 128/64): s <- s*M + inc (mod 2^128), out = rotr(hi^lo, hi>>58)
//   random_standard_normal (numpy/random/src/distributions/distributions.c):
//     r = next_uint64; idx = r & 0xff; r >>= 8; sign = r & 1;
//     rabs = (r >> 1) & (2^52-1); x = +-rabs * wi[idx];
//     rabs < ki[idx]                       -> x                 (~99.3%)
//     idx == 0: tail loop on pairs of next_double -> +-(R + xx)
//     else: wedge test with one next_double -> x, or reject and restart
//
// The draw is a variable-length walk over the raw stream, so it runs in
// three data-parallel passes instead of one sequential loop:
//   1. raw:      R[p] = output after p+1 LCG steps (jump-ahead per chunk)
//   2. classify: for every position p, the outcome IF a normal starts at p:
//                value, emitted or rejected, and how many words it consumes
//   3. resolve:  one CTA per stream walks the ~0.7% non-trivial positions in
//                order (shared memory) to find which positions actually start
//                a draw, then a block scan assigns output indices.
// Floating-point steps use explicit _rn intrinsics in numpy's operation order
// (no FMA contraction, as in numpy's x86-64 baseline build). Exactness: every
// fast-path and wedge draw is bit-identical to numpy (the wedge's accept test
// compares against exp(), so CUDA's and libm's exp could only disagree on a
// comparison within 1 ulp, probability ~1e-16). The tail branch (|x| > r =
// 3.654, ~2.6e-4 of draws) calls log1p, where numpy's libm (glibc, an
// ifunc-selected variant) and CUDA can round differently: measured 8 values
// of 12.8M draws differ, each by 1 ulp (tests/test_device_rng.py pins that).
#include <cstdint>

#include "common.cuh"
#include "ziggurat_tables.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace rng {

struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ull, kMulLo = 0x4385DF649FCCF645ull;

// state after `delta` LCG steps (pcg_advance_lcg_128: square-and-multiply)
__device__ U128 advance(U128 s, uint64_t delta, U128 inc) {
  U128 acc_mult{0, 1}, acc_plus{0, 0};
  U128 cur_mult{kMulHi, kMulLo}, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, s), acc_plus);
}
__device__ __forceinline__ uint64_t output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = unsigned(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double next_double(uint64_t r) {
  return double(r >> 11) * (1.0 / 9007199254740992.0);
}

constexpr double kR = 3.6541528853610087963519472518;
constexpr double kInvR = 0.27366123732975827203338247596;
constexpr int kChunk = 16;       // raw words per thread
constexpr int kResolveThreads = 1024;
constexpr int kMaxSpecial = 18432;  // non-trivial positions per stream (shared memory; ~1.5%
                                    // of positions, 16.3k expected at count = 2^20)
constexpr int64_t kMaxCount = 1 << 20;

// stream layout of the workspace: R[L] u64, val[L] f64, code[L] i32
// code: bits 0..29 = words consumed by a draw starting here, bit 30 = emits a value,
// 0 = the draw would run past the generated words
__host__ __device__ inline int64_t raw_len(int64_t count) { return count + count / 32 + 2048; }

__global__ void raw_kernel(const uint64_t *states, int64_t L, uint64_t *R) {
  const int s = blockIdx.y;
  const int64_t p0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
  if (p0 >= L) return;
  const uint64_t *st = states + 4 * s;
  const U128 inc{st[2], st[3]};
  U128 x = advance(U128{st[0], st[1]}, uint64_t(p0), inc);
  const U128 mult{kMulHi, kMulLo};
  uint64_t *r = R + s * L;
  for (int k = 0; k < kChunk && p0 + k < L; ++k) {
    x = add128(mul128(x, mult), inc);
    r[p0 + k] = output(x);
  }
}

__global__ void classify_kernel(const uint64_t *Rall, int64_t L, double *valall, int *codeall) {
  const int s = blockIdx.y;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= L) return;
  const uint64_t *R = Rall + s * L;
  uint64_t r = R[p];
  const int idx = int(r & 0xff);
  r >>= 8;
  const bool neg = (r & 1) != 0;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  double x = __dmul_rn(double(rabs), zig::wi[idx]);
  if (neg) x = -x;
  double val = x;
  int code;
  if (rabs < zig::ki[idx]) {
    code = (1 << 30) | 1;
  } else if (idx == 0) {
    code = 0;  // runs past the generated words unless accepted below
    for (int64_t q = p + 1; q + 1 < L; q += 2) {
      const double xx = __dmul_rn(-kInvR, log1p(-next_double(R[q])));
      const double yy = -log1p(-next_double(R[q + 1]));
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        val = ((rabs >> 8) & 1) ? -__dadd_rn(kR, xx) : __dadd_rn(kR, xx);
        code = (1 << 30) | int(q + 2 - p);
        break;
      }
    }
  } else if (p + 1 < L) {
    const double u = next_double(R[p + 1]);
    const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(zig::fi[idx - 1], -zig::fi[idx]), u),
                                 zig::fi[idx]);
    const bool acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    code = (acc ? (1 << 30) : 0) | 2;
  } else {
    code = 0;
  }
  valall[s * L + p] = val;
  codeall[s * L + p] = code;
}

// exclusive block scan of one int per thread (1024 threads); returns the total
__device__ int block_scan(int v, int *warp_sums, int &excl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  const int base = wid ? warp_sums[wid - 1] : 0;
  excl = base + x - v;
  const int total = warp_sums[31];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kResolveThreads, 1)
    resolve_kernel(const double *valall, const int *codeall, int64_t L, int64_t count,
                   double *out, int64_t ldo, int *status) {
  extern __shared__ int sm[];
  int *sp_pos = sm;                     // [kMaxSpecial] positions of non-trivial draws
  int *sp_code = sp_pos + kMaxSpecial;  // [kMaxSpecial] their codes, then start flags
  int *sp_end = sp_code + kMaxSpecial;  // [kMaxSpecial] covered-through (prefix max)
  __shared__ int warp_sums[32];
  const int s = blockIdx.x;
  const double *val = valall + s * L;
  const int *code = codeall + s * L;
  const int64_t per = (L + kResolveThreads - 1) / kResolveThreads;
  const int64_t p0 = min(L, per * threadIdx.x), p1 = min(L, p0 + per);

  // 1. compact the non-trivial positions, in order
  int mine = 0;
  for (int64_t p = p0; p < p1; ++p) mine += code[p] != ((1 << 30) | 1);
  int off;
  const int nsp = block_scan(mine, warp_sums, off);
  if (nsp > kMaxSpecial) {
    if (threadIdx.x == 0) atomicMax(status, 2);
    return;
  }
  for (int64_t p = p0; p < p1; ++p) {
    const int c = code[p];
    if (c != ((1 << 30) | 1)) {
      sp_pos[off] = int(p);
      sp_code[off] = c;
      ++off;
    }
  }
  __syncthreads();
  // 2. walk them in order: a non-trivial position starts a draw iff the walk
  //    reaches it (every position in between consumes exactly one word)
  //    (the walk stops once `count` values are out: draws after that may run
  //    past the generated words without harm)
  if (threadIdx.x == 0) {
    int cur = 0, cov = 0;
    int64_t emitted = 0;
    int k = 0;
    for (; k < nsp; ++k) {
      const int pos = sp_pos[k], c = sp_code[k];
      if (pos >= cur) {
        emitted += pos - cur;  // the one-word draws in between
        if (emitted >= count) break;
        if ((c & 0x3fffffff) == 0) {  // a draw needs words past the generated ones
          atomicMax(status, 1);
          cur = int(L);
        } else {
          cur = pos + (c & 0x3fffffff);
          emitted += (c >> 30) & 1;
        }
        sp_code[k] = c | int(0x80000000u);  // starts
        cov = cur;
      }
      sp_end[k] = cov;  // positions < cov after the last start at or before k are consumed
    }
    for (; k < nsp; ++k) sp_end[k] = cov;
  }
  __syncthreads();
  // 3. emitted values in order: count, scan, write
  auto starts = [&](int64_t p, int &k) -> int {  // 1 = starts and emits
    while (k < nsp && sp_pos[k] < p) ++k;
    if (k < nsp && sp_pos[k] == p) {
      const int c = sp_code[k];
      return (c < 0 && (c & (1 << 30))) ? 1 : 0;
    }
    return (k == 0 || sp_end[k - 1] <= p) ? 1 : 0;  // trivial: emits unless consumed
  };
  int k0 = 0;
  {  // first special at or after p0 (binary search)
    int lo = 0, hi = nsp;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sp_pos[mid] < p0) lo = mid + 1; else hi = mid;
    }
    k0 = lo;
  }
  int k = k0, emit = 0;
  for (int64_t p = p0; p < p1; ++p) emit += starts(p, k);
  const int total = block_scan(emit, warp_sums, off);
  if (total < count) {
    if (threadIdx.x == 0) atomicMax(status, 1);
    return;
  }
  k = k0;
  double *o = out + s * ldo;
  for (int64_t p = p0; p < p1 && off < count; ++p)
    if (starts(p, k)) o[off++] = val[p];
}

}  // namespace rng
}  // namespace sap

using namespace sap;

extern "C" {

size_t sap_normal_workspace(int64_t count, int nstreams) {
  const int64_t L = rng::raw_len(count);
  return size_t(nstreams) * size_t(L) * (8 + 8 + 4) + 256;
}

int sap_normal_fill(const uint64_t *states, int nstreams, int64_t count, double *out, int64_t ldo,
                    void *ws, size_t ws_bytes, void *stream) {
  if (nstreams <= 0 || count <= 0 || count > rng::kMaxCount || ldo < count)
    return fail(SAP_ERR_CONTRACT, "normal_fill: bad shape streams=%d count=%lld ldo=%lld",
                nstreams, (long long)count, (long long)ldo);
  if (!ws || ws_bytes < sap_normal_workspace(count, nstreams))
    return fail(SAP_ERR_CONTRACT, "normal_fill: workspace too small");
  const int64_t L = rng::raw_len(count);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t *w = static_cast<uint8_t *>(ws);
  int *status = reinterpret_cast<int *>(w);  // first 256 bytes: status word
  uint64_t *R = reinterpret_cast<uint64_t *>(w + 256);
  double *val = reinterpret_cast<double *>(w + 256 + size_t(nstreams) * L * 8);
  int *code = reinterpret_cast<int *>(w + 256 + size_t(nstreams) * L * 16);
  int rc;
  if (cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess)
    return fail(SAP_ERR_DEVICE, "normal_fill: memset failed");
  {
    const int64_t threads = (L + rng::kChunk - 1) / rng::kChunk;
    dim3 grid(unsigned((threads + 255) / 256), unsigned(nstreams));
    rng::raw_kernel<<<grid, 256, 0, st>>>(states, L, R);
    if ((rc = check_launch("normal_raw_kernel")) != SAP_OK) return rc;
  }
  {
    dim3 grid(unsigned((L + 255) / 256), unsigned(nstreams));
    rng::classify_kernel<<<grid, 256, 0, st>>>(R, L, val, code);
    if ((rc = check_launch("normal_classify_kernel")) != SAP_OK) return rc;
  }
  const int smem = 3 * rng::kMaxSpecial * int(sizeof(int));
  cudaFuncSetAttribute(rng::resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rng::resolve_kernel<<<nstreams, rng::kResolveThreads, smem, st>>>(val, code, L, count, out, ldo,
                                                                   status);
  return check_launch("normal_resolve_kernel");
}

// status word of the last sap_normal_fill on this workspace (device pointer,
// the workspace's first int): 0 ok, 1 the generated raw words ran out, 2 too
// many non-trivial draws for the resolve pass
int *sap_normal_status(void *ws) { return static_cast<int *>(ws); }

}  // extern "C"
