// C-ABI entry points of libsapgp_b200.so (declared in include/sapgp_b200.h)
// plus the small HBM-bound kernels around the block-row product.
#include <cstdio>
#include <cstdarg>
#include <string>
#include <algorithm>
#include <atomic>
#include <cuda_fp16.h>

#include "common.cuh"
#include "krows_ffma.cuh"

namespace sap {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

std::atomic<long long> g_launches{0};

int check_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SAP_ERR_DEVICE, "%s: %s", what, cudaGetErrorString(e));
  return SAP_OK;
}

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// point preparation / gathers

__global__ void prepare_points_kernel(const double *X, int64_t n, int d, const double *inv_ls,
                                      float *Xs, int ldx, float *sqn) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int k = 0; k < ldx; ++k) {
    double v = 0.0;
    if (k < d) {
      v = X[j * d + k] * inv_ls[k];
      s = fma(v, v, s);
    }
    Xs[j * ldx + k] = float(v);
  }
  sqn[j] = float(s);
}

__global__ void gather_points_kernel(const float *Xs, const float *sqn, int ldx,
                                     const int64_t *idx, int64_t b, int64_t base, float *Rs,
                                     float *rsqn) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * ldx) return;
  const int64_t i = e / ldx;
  const int k = int(e % ldx);
  const int64_t j = idx[i] - base;
  Rs[e] = Xs[j * ldx + k];
  if (k == 0) rsqn[i] = sqn[j];
}

// ---------------------------------------------------------------------------
// dense tiles (kernels.py:118-143). With equal point sets and id arrays the
// result is bitwise symmetric: (rn_i + rn_j) - 2 sum_k a_k c_k is symmetric
// term by term in IEEE arithmetic.

// 32 x 32 output tile per 256-thread block: the tile's row and column points
// are staged in shared memory once (column stride ldx + 1: conflict-free),
// each thread computes four rows of one column. Same arithmetic order as the
// block product's distance (fmaf over k, then the norms): K(i, j) and K(j, i)
// are bitwise equal, so the block is exactly symmetric (kernels.py:129-136).
template <int FAM, typename T>
__global__ void __launch_bounds__(256)
    ktile_kernel(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
                 const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc, int ldx,
                 int d, float variance, T *out, int64_t ldo) {
  extern __shared__ float sh[];
  float *sA = sh;                  // [32][ldx + 1]
  float *sC = sh + 32 * (ldx + 1);  // [32][ldx + 1]
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int64_t i0 = int64_t(blockIdx.y) * 32, j0 = int64_t(blockIdx.x) * 32;
  for (int e = tid; e < 32 * ldx; e += 256) {
    const int r = e / ldx, k = e % ldx;
    sA[r * (ldx + 1) + k] = i0 + r < na ? Ra[(i0 + r) * ldx + k] : 0.0f;
    sC[r * (ldx + 1) + k] = j0 + r < nc ? Rc[(j0 + r) * ldx + k] : 0.0f;
  }
  __syncthreads();
  const int64_t j = j0 + tx;
  if (j >= nc) return;
  const float csq = rcsqn[j];
  const int64_t cid = col_ids ? col_ids[j] : -1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int li = ty + 8 * q;
    const int64_t i = i0 + li;
    if (i >= na) break;
    float v;
    if (row_ids && col_ids && row_ids[i] == cid) {
      v = variance;
    } else {
      float dot = 0.0f;
      for (int k = 0; k < d; ++k) dot = fmaf(sA[li * (ldx + 1) + k], sC[tx * (ldx + 1) + k], dot);
      const float sq = fmaf(-2.0f, dot, rasqn[i] + csq);
      v = variance * kernel_value<FAM>(sq);
    }
    out[i * ldo + j] = T(v);
  }
}


// K_BB of a batch of blocks in one launch (the lookahead's power-iteration
// input): block q's points X_q [b][ldx] (scaled fp32) against themselves,
// 64x64 outputs per CTA of 256 threads, 4x4 per thread from [k][64] staged
// coordinates (16-byte shared loads), 16-byte stores. The arithmetic is
// ktile_kernel's (same fma order, same sum of norms, the id rule on the
// diagonal: the block's ids are unique, so i == j), so the values are the
// same bit for bit; ~5x faster than the 32x32 tiles at b = 2000.
// Optionally (outh != NULL) also K / variance split into fp16 hi + lo (the
// sketch's three-pass tensor-core GEMM operand, pipeline.py): hi = fp16(k),
// lo = fp16(k - hi), k = K / variance in [0, 1].
template <int FAM>
__global__ void __launch_bounds__(256)
    ktile_batch_kernel(const float *X, int64_t strideX, const float *xsq, int64_t strideSq, int b,
                       int ldx, int d, float variance, float *out, int64_t ldo,
                       int64_t strideOut, __half *outh, __half *outl, int64_t ldh,
                       int64_t strideH) {
  extern __shared__ __align__(16) float sh[];
  float *sA = sh;            // [d][64] row points
  float *sC = sh + d * 64;   // [d][64] column points
  const int q = blockIdx.z;
  const float *Xq = X + int64_t(q) * strideX;
  const float *sq = xsq + int64_t(q) * strideSq;
  float *oq = out + int64_t(q) * strideOut;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int e = tid; e < 64 * d; e += 256) {
    const int r = e / d, k = e - r * d;
    sA[k * 64 + r] = i0 + r < b ? Xq[int64_t(i0 + r) * ldx + k] : 0.0f;
    sC[k * 64 + r] = j0 + r < b ? Xq[int64_t(j0 + r) * ldx + k] : 0.0f;
  }
  __syncthreads();
  float dot[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) dot[a][c] = 0.0f;
  for (int k = 0; k < d; ++k) {
    const float4 ra = *reinterpret_cast<const float4 *>(sA + k * 64 + ty * 4);
    const float4 rc = *reinterpret_cast<const float4 *>(sC + k * 64 + tx * 4);
    const float av[4] = {ra.x, ra.y, ra.z, ra.w}, cv[4] = {rc.x, rc.y, rc.z, rc.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) dot[a][c] = fmaf(av[a], cv[c], dot[a][c]);
  }
  const int j = j0 + tx * 4;
  float csq[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) csq[c] = j + c < b ? sq[j + c] : 0.0f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + ty * 4 + a;
    if (i >= b) break;
    const float rs = sq[i];
    float v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      v[c] = (i == j + c) ? variance
                          : variance * kernel_value<FAM>(fmaf(-2.0f, dot[a][c], rs + csq[c]));
    float *o = oq + int64_t(i) * ldo + j;
    if (j + 3 < b) {
      *reinterpret_cast<float4 *>(o) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (j + c < b) o[c] = v[c];
    }
    if (outh) {
      const float iv = 1.0f / variance;
      __half hh[4], ll[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float k = v[c] * iv;
        hh[c] = __float2half_rn(k);
        ll[c] = __float2half_rn(k - __half2float(hh[c]));
      }
      const int64_t ho = int64_t(q) * strideH + int64_t(i) * ldh + j;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (j + c < b) {
          outh[ho + c] = hh[c];
          outl[ho + c] = ll[c];
        }
    }
  }
}

// fp64 tile for the dense-access API (KernelOracle.tile/block/dense,
// kernels.py:118-143): the reference's own arithmetic -- z = x / l in fp64,
// sq = |z_r|^2 + |z_c|^2 - 2 z_r.z_c, sq = 0 where the ids match, clamp at 0,
// family values in fp64 -- so dense blocks are PSD to fp64 rounding (the
// hot path's K_BB uses the fp32 tile above).
template <int FAM>
__device__ __forceinline__ double kernel_value64(double sq) {
  sq = fmax(sq, 0.0);
  if constexpr (FAM == SAP_RBF) {
    return exp(-0.5 * sq);
  } else if constexpr (FAM == SAP_MATERN32) {
    const double a = 1.7320508075688772 * sqrt(sq);
    return (1.0 + a) * exp(-a);
  } else {
    const double a = 2.23606797749979 * sqrt(sq);
    return (1.0 + a + (5.0 / 3.0) * sq) * exp(-a);
  }
}

template <int FAM>
__global__ void ktile64_kernel(const double *X, const double *inv_ls, int d,
                               const int64_t *row_ids, int64_t na, const int64_t *col_ids,
                               int64_t nc, double variance, double *out, int64_t ldo) {
  const int64_t i = int64_t(blockIdx.y) * blockDim.y + threadIdx.y;
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= na || j >= nc) return;
  const int64_t ri = row_ids[i], cj = col_ids[j];
  double v = variance;
  if (ri != cj) {
    double nr = 0.0, ncs = 0.0, dot = 0.0;
    for (int k = 0; k < d; ++k) {
      const double zr = X[ri * d + k] * inv_ls[k], zc = X[cj * d + k] * inv_ls[k];
      nr = fma(zr, zr, nr);
      ncs = fma(zc, zc, ncs);
      dot = fma(zr, zc, dot);
    }
    v = variance * kernel_value64<FAM>(nr + ncs - 2.0 * dot);
  }
  out[i * ldo + j] = v;
}

// ---------------------------------------------------------------------------
// gradient gather (solvers.py:376-377), lazy Nesterov rows, materialisation

__global__ void grad_gather_kernel(const float *G, int64_t ldg, const float *P, const float *Q,
                                   const float *Y, int64_t ldp, double zp, double zq,
                                   const int64_t *loc, int64_t b, int m, double lam, double *g,
                                   int64_t ldgo) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int64_t i = e / m;
  const int c = int(e % m);
  double v = double(G[i * ldg + c]);
  const int64_t j = loc[i];
  if (j >= 0) {
    const int64_t o = int64_t(c) * ldp + j;
    double z = zp * double(P[o]);
    if (Q) z += zq * double(Q[o]);
    v += lam * z - double(Y[o]);
  }
  g[i * ldgo + c] = v;
}

// Block-row update of the lazy Nesterov state, threads laid out column-major
// over (row i, column c): a warp covers 32 block rows of ONE column, so the per-column magnitude bounds
// take one warp-reduced atomic per warp instead of one per element.
__global__ void pq_update_cm_kernel(float *P, float *Q, int64_t ldp, const int64_t *loc, int64_t b,
                                    int m, const double *D, int64_t ldd, const double *eta_dev,
                                    double zp, double zq, double e0, double e1, float *WB,
                                    int64_t ldwb, float *Pb, float *Qb) {
  const int64_t bw = (b + 31) / 32 * 32;  // rows padded to whole warps
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= bw * m) return;  // warp-uniform: bw * m is a multiple of 32
  const int c = int(e / bw);
  const int64_t i = e % bw;
  const int64_t j = i < b ? loc[i] : -1;
  float pa = 0.0f, qa = 0.0f;
  if (j >= 0) {
    const double eta = eta_dev[0];
    const double dd = D[i * ldd + c];
    const int64_t o = int64_t(c) * ldp + j;
    const double p = P[o];
    const double q = Q ? double(Q[o]) : 0.0;
    if (WB) WB[i * ldwb + c] = float(zp * p + zq * q - eta * dd);
    const float pn = float(p + e0 * eta * dd);
    P[o] = pn;
    pa = fabsf(pn);
    if (Q) {
      const float qn = float(q + e1 * eta * dd);
      Q[o] = qn;
      qa = fabsf(qn);
    }
  }
  if (Pb) {
    const unsigned mx = __reduce_max_sync(0xffffffffu, __float_as_uint(pa));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(reinterpret_cast<int *>(Pb + c), int(mx));
  }
  if (Qb && Q) {
    const unsigned mx = __reduce_max_sync(0xffffffffu, __float_as_uint(qa));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(reinterpret_cast<int *>(Qb + c), int(mx));
  }
}

// ---------------------------------------------------------------------------
// SDD (solvers.py:463-516): velocity *= 0.9; velocity[B] -= eta*grad;
// w += velocity; estimate += avg * (w - estimate), as a block scatter of the
// block rows' new velocity plus ONE dense pass over (V, W, E).

__global__ void sdd_block_kernel(const float *V, int64_t ldv, const int64_t *loc, int64_t b, int m,
                                 const double *g, int64_t ldg, double eta, double momentum,
                                 float *VB, int *pos) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int64_t i = e / m;
  const int c = int(e % m);
  const int64_t j = loc[i];
  if (j < 0) return;
  // fp32 like the dense pass, in the reference's order: (0.9 v) - eta g
  const float vm = float(momentum) * V[int64_t(c) * ldv + j];
  VB[i * m + c] = vm - float(eta * g[i * ldg + c]);
  if (c == 0) pos[j] = int(i);
}

// four consecutive rows per thread (16-byte accesses; ldv is a multiple of 4)
__global__ void sdd_dense_kernel(float *__restrict__ V, float *__restrict__ W,
                                 float *__restrict__ E, int64_t ldv, int64_t rows4, int m,
                                 const float *__restrict__ VB, int *__restrict__ pos,
                                 float momentum, float avg) {
  const int64_t j4 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j4 >= rows4) return;
  const int4 p = reinterpret_cast<const int4 *>(pos)[j4];
  const bool any = p.x >= 0 || p.y >= 0 || p.z >= 0 || p.w >= 0;
#pragma unroll 4
  for (int c = 0; c < m; ++c) {
    const int64_t o = int64_t(c) * ldv / 4 + j4;
    float4 v = reinterpret_cast<const float4 *>(V)[o];
    float4 w = reinterpret_cast<const float4 *>(W)[o];
    float4 e = reinterpret_cast<const float4 *>(E)[o];
    v.x = p.x >= 0 ? VB[int64_t(p.x) * m + c] : momentum * v.x;
    v.y = p.y >= 0 ? VB[int64_t(p.y) * m + c] : momentum * v.y;
    v.z = p.z >= 0 ? VB[int64_t(p.z) * m + c] : momentum * v.z;
    v.w = p.w >= 0 ? VB[int64_t(p.w) * m + c] : momentum * v.w;
    w.x += v.x; w.y += v.y; w.z += v.z; w.w += v.w;
    e.x += avg * (w.x - e.x); e.y += avg * (w.y - e.y);
    e.z += avg * (w.z - e.z); e.w += avg * (w.w - e.w);
    reinterpret_cast<float4 *>(V)[o] = v;
    reinterpret_cast<float4 *>(W)[o] = w;
    reinterpret_cast<float4 *>(E)[o] = e;
  }
  if (any) reinterpret_cast<int4 *>(pos)[j4] = make_int4(-1, -1, -1, -1);  // clean for the next step
}

__global__ void combine_kernel(float *out, int64_t ldo, const float *P, const float *Q,
                               int64_t ldp, int64_t n, int m, float a, float bq) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * m) return;
  const int c = int(e / n);
  const int64_t j = e % n;
  float v = a * P[int64_t(c) * ldp + j];
  if (Q) v = fmaf(bq, Q[int64_t(c) * ldp + j], v);
  out[int64_t(c) * ldo + j] = v;
}

// Fixed-order reduction of the split partials: out = variance * sum_s part[s].
__global__ void krows_reduce_kernel(const float *__restrict__ part, int splits, int64_t b, int m,
                                    float variance, float *out, int64_t ldo, int c0,
                                    int accumulate) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int64_t i = e / m;
  const int c = int(e % m);
  float s = 0.0f;
  for (int k = 0; k < splits; ++k) s += part[int64_t(k) * b * m + e];
  float *o = out + i * ldo + c0 + c;
  const float v = variance * s;
  *o = accumulate ? *o + v : v;
}


// ---------------------------------------------------------------------------
// FP32 FFMA throughput probe (the roofline denominator of the FFMA path):
// 8 independent dependency chains per thread, 2 flops per FFMA.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float *out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float x = 0.9999f, y = 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], x, y);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------------------
// krows dispatch

constexpr int kTargetCtas = 2 * 148;  // a pure function of the shape: deterministic

int pick_splits(int64_t b, int m, int64_t tiles) {
  // Choose the column split so the grid fills whole waves of 2 CTAs per SM
  // (148 SMs); a pure function of the shape, so results are deterministic.
  const int64_t row_tiles = (b + kFfmaBM - 1) / kFfmaBM;
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(tiles / 8, 4096));
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= std::min<int64_t>(max_s, 4 * kTargetCtas); ++s) {
    const int64_t total = row_tiles * s;
    const int64_t waves = (total + kTargetCtas - 1) / kTargetCtas;
    if (waves > 4) break;
    const double eff = double(total) / double(waves * kTargetCtas);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return int(best);
}

int launch_ffma_rbf(KrowsParams p, int dp, cudaStream_t st);
int launch_ffma_m32(KrowsParams p, int dp, cudaStream_t st);
int launch_ffma_m52(KrowsParams p, int dp, cudaStream_t st);

int padded_dim(int ldx) {
  for (int dp : {4, 8, 12, 16, 32, 64})
    if (ldx <= dp) return dp;
  return -1;
}

}  // namespace sap

using namespace sap;

template <typename T>
static int ktile_launch(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
                        const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc,
                        int ldx, int d, int family, double variance, T *out, int64_t ldo,
                        void *stream) {
  if (na <= 0 || nc <= 0 || ldo < nc || ldx < d || d < 1)
    return fail(SAP_ERR_CONTRACT, "ktile: bad shape");
  dim3 blk(32, 8), grid(unsigned((nc + 31) / 32), unsigned((na + 31) / 32));
  cudaStream_t st = S(stream);
  const float var = float(variance);
  const size_t smem = size_t(2 * 32 * (ldx + 1)) * sizeof(float);
  switch (family) {
    case SAP_RBF:
      ktile_kernel<SAP_RBF, T><<<grid, blk, smem, st>>>(Ra, rasqn, row_ids, na, Rc, rcsqn,
                                                        col_ids, nc, ldx, d, var, out, ldo);
      break;
    case SAP_MATERN32:
      ktile_kernel<SAP_MATERN32, T><<<grid, blk, smem, st>>>(Ra, rasqn, row_ids, na, Rc, rcsqn,
                                                             col_ids, nc, ldx, d, var, out, ldo);
      break;
    case SAP_MATERN52:
      ktile_kernel<SAP_MATERN52, T><<<grid, blk, smem, st>>>(Ra, rasqn, row_ids, na, Rc, rcsqn,
                                                             col_ids, nc, ldx, d, var, out, ldo);
      break;
    default: return fail(SAP_ERR_CONTRACT, "ktile: unknown family %d", family);
  }
  return check_launch("ktile_kernel");
}

extern "C" {

int sap_abi_version(void) { return SAP_ABI_VERSION; }

const char *sap_last_error(void) { return g_last_error.c_str(); }

long long sap_launch_count(void) { return g_launches.load(); }

int sap_ffma_peak(float *out, int iters, void *stream) {
  ffma_peak_kernel<<<148 * 4, 256, 0, S(stream)>>>(out, iters);
  return check_launch("ffma_peak_kernel");
}

int sap_prepare_points(const double *X, int64_t n, int d, const double *inv_ls, float *Xs, int ldx,
                       float *sqn, void *stream) {
  if (n < 0 || d < 1 || ldx < d || ldx % 4 != 0)
    return fail(SAP_ERR_CONTRACT, "prepare_points: bad shape n=%lld d=%d ldx=%d",
                (long long)n, d, ldx);
  if (n == 0) return SAP_OK;
  prepare_points_kernel<<<unsigned((n + 255) / 256), 256, 0, S(stream)>>>(X, n, d, inv_ls, Xs, ldx,
                                                                         sqn);
  return check_launch("prepare_points_kernel");
}

int sap_gather_points(const float *Xs, const float *sqn, int ldx, const int64_t *idx, int64_t b,
                      int64_t base, float *Rs, float *rsqn, void *stream) {
  if (b <= 0) return fail(SAP_ERR_CONTRACT, "gather_points: empty index block");
  const int64_t tot = b * ldx;
  gather_points_kernel<<<unsigned((tot + 255) / 256), 256, 0, S(stream)>>>(Xs, sqn, ldx, idx, b,
                                                                          base, Rs, rsqn);
  return check_launch("gather_points_kernel");
}

size_t sap_krows_workspace(int64_t b, int m, int64_t ncols) {
  const int64_t tiles = (ncols + kFfmaBN - 1) / kFfmaBN;
  const int mc = m < 128 ? m : 128;
  const int s = pick_splits(b, mc, tiles);
  return s > 1 ? size_t(s) * size_t(b) * size_t(mc) * sizeof(float) : 0;
}

int sap_krows_times(const float *Xs, const float *sqn, int ldx, int64_t ncols,
                    const int64_t *col_ids, int64_t col_base, const float *Rs, const float *rsqn,
                    const int64_t *row_ids, int64_t b, int d, const float *A, const float *Bm,
                    int64_t lda, int m, double ca, double cb, int family, double variance,
                    float *out, int64_t ldo, int accumulate, void *ws, size_t ws_bytes,
                    void *stream) {
  if (b <= 0 || m <= 0 || ncols < 0 || d < 1)
    return fail(SAP_ERR_CONTRACT, "krows_times: bad shape b=%lld m=%d ncols=%lld d=%d",
                (long long)b, m, (long long)ncols, d);
  if (ldx < d || ldx % 4 != 0) return fail(SAP_ERR_CONTRACT, "krows_times: ldx=%d", ldx);
  if (lda < ncols) return fail(SAP_ERR_CONTRACT, "krows_times: lda < ncols");
  if (ldo < m) return fail(SAP_ERR_CONTRACT, "krows_times: ldo < m");
  if (family < SAP_RBF || family > SAP_MATERN52)
    return fail(SAP_ERR_CONTRACT, "krows_times: unknown family %d", family);
  const int dp = padded_dim(ldx);
  if (dp < 0) return fail(SAP_ERR_CONTRACT, "krows_times: d=%d exceeds 64", d);
  if (ldx != dp)
    return fail(SAP_ERR_CONTRACT, "krows_times: ldx=%d must equal the padded width %d", ldx, dp);
  cudaStream_t st = S(stream);
  if (ncols == 0) {
    if (!accumulate) {
      for (int64_t i = 0; i < b; ++i)
        if (cudaMemsetAsync(out + i * ldo, 0, sizeof(float) * m, st) != cudaSuccess)
          return fail(SAP_ERR_DEVICE, "memset failed");
    }
    return SAP_OK;
  }
  KrowsParams p{};
  p.Xs = Xs; p.sqn = sqn; p.ldx = ldx; p.ncols = ncols; p.col_ids = col_ids;
  p.col_base = col_base; p.Rs = Rs; p.rsqn = rsqn; p.row_ids = row_ids; p.b = b;
  p.A = A; p.Bm = Bm; p.lda = lda; p.ca = float(ca); p.cb = float(cb);
  p.variance = float(variance); p.ldo = ldo; p.accumulate = accumulate;
  p.tiles = (ncols + kFfmaBN - 1) / kFfmaBN;
  for (int c0 = 0; c0 < m; c0 += 128) {
    const int mc = std::min(128, m - c0);
    p.m = mc;
    p.c0 = c0;
    p.splits = pick_splits(b, mc, p.tiles);
    if (p.splits > 1) {
      const size_t need = size_t(p.splits) * size_t(b) * size_t(mc) * sizeof(float);
      if (!ws || ws_bytes < need)
        return fail(SAP_ERR_CONTRACT, "krows_times: workspace %zu < %zu bytes", ws_bytes, need);
      p.out = static_cast<float *>(ws);
    } else {
      p.out = out;
    }
    int rc;
    switch (family) {
      case SAP_RBF: rc = launch_ffma_rbf(p, dp, st); break;
      case SAP_MATERN32: rc = launch_ffma_m32(p, dp, st); break;
      default: rc = launch_ffma_m52(p, dp, st); break;
    }
    if (rc != SAP_OK) return rc;
    if (p.splits > 1) {
      const int64_t tot = b * mc;
      krows_reduce_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(
          static_cast<const float *>(ws), p.splits, b, mc, float(variance), out, ldo, c0,
          accumulate);
      if ((rc = check_launch("krows_reduce_kernel")) != SAP_OK) return rc;
    }
  }
  return SAP_OK;
}

int sap_ktile(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
              const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc, int ldx,
              int d, int family, double variance, double *out, int64_t ldo, void *stream) {
  return ktile_launch(Ra, rasqn, row_ids, na, Rc, rcsqn, col_ids, nc, ldx, d, family, variance,
                      out, ldo, stream);
}

int sap_ktile_f32(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
                  const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc,
                  int ldx, int d, int family, double variance, float *out, int64_t ldo,
                  void *stream) {
  return ktile_launch(Ra, rasqn, row_ids, na, Rc, rcsqn, col_ids, nc, ldx, d, family, variance,
                      out, ldo, stream);
}

int sap_ktile_f32_batch_split(const float *X, int64_t strideX, const float *xsq,
                              int64_t strideSq, int b, int count, int ldx, int d, int family,
                              double variance, float *out, int64_t ldo, int64_t strideOut,
                              void *outh, void *outl, int64_t ldh, int64_t strideH,
                              void *stream) {
  if (b <= 0 || count <= 0 || ldx < d || d < 1 || d > 64 || ldo < b || ldo % 4 ||
      strideOut % 4 || (reinterpret_cast<uintptr_t>(out) & 15) || (outh && (!outl || ldh < b)) ||
      !(variance > 0.0))
    return fail(SAP_ERR_CONTRACT, "ktile_f32_batch: bad shape b=%d d=%d ldo=%lld", b, d,
                (long long)ldo);
  __half *oh = static_cast<__half *>(outh), *ol = static_cast<__half *>(outl);
  dim3 grid(unsigned((b + 63) / 64), unsigned((b + 63) / 64), unsigned(count));
  const size_t smem = size_t(2 * 64 * d) * sizeof(float);
  cudaStream_t st = S(stream);
  const float var = float(variance);
  switch (family) {
    case SAP_RBF:
      ktile_batch_kernel<SAP_RBF><<<grid, 256, smem, st>>>(X, strideX, xsq, strideSq, b, ldx, d,
                                                           var, out, ldo, strideOut, oh, ol, ldh,
                                                           strideH);
      break;
    case SAP_MATERN32:
      ktile_batch_kernel<SAP_MATERN32><<<grid, 256, smem, st>>>(X, strideX, xsq, strideSq, b,
                                                                ldx, d, var, out, ldo, strideOut,
                                                                oh, ol, ldh, strideH);
      break;
    case SAP_MATERN52:
      ktile_batch_kernel<SAP_MATERN52><<<grid, 256, smem, st>>>(X, strideX, xsq, strideSq, b,
                                                                ldx, d, var, out, ldo, strideOut,
                                                                oh, ol, ldh, strideH);
      break;
    default: return fail(SAP_ERR_CONTRACT, "ktile_f32_batch: unknown family %d", family);
  }
  return check_launch("ktile_batch_kernel");
}

int sap_ktile_f32_batch(const float *X, int64_t strideX, const float *xsq, int64_t strideSq,
                        int b, int count, int ldx, int d, int family, double variance, float *out,
                        int64_t ldo, int64_t strideOut, void *stream) {
  return sap_ktile_f32_batch_split(X, strideX, xsq, strideSq, b, count, ldx, d, family, variance,
                                   out, ldo, strideOut, nullptr, nullptr, 0, 0, stream);
}

int sap_grad_gather(const float *G, int64_t ldg, const float *P, const float *Q, const float *Y,
                    int64_t ldp, double zp, double zq, const int64_t *loc, int64_t b, int m,
                    double lam, double *g, int64_t ldgo, void *stream) {
  if (b <= 0 || m <= 0) return fail(SAP_ERR_CONTRACT, "grad_gather: bad shape");
  const int64_t tot = b * m;
  grad_gather_kernel<<<unsigned((tot + 255) / 256), 256, 0, S(stream)>>>(
      G, ldg, P, Q, Y, ldp, zp, zq, loc, b, m, lam, g, ldgo);
  return check_launch("grad_gather_kernel");
}

int sap_pq_update(float *P, float *Q, int64_t ldp, const int64_t *loc, int64_t b, int m,
                  const double *D, int64_t ldd, const double *eta_dev, double zp, double zq,
                  double e0, double e1, float *WB, int64_t ldwb, float *Pb, float *Qb,
                  void *stream) {
  if (b <= 0 || m <= 0) return fail(SAP_ERR_CONTRACT, "pq_update: bad shape");
  const int64_t tot = (b + 31) / 32 * 32 * m;
  pq_update_cm_kernel<<<unsigned((tot + 255) / 256), 256, 0, S(stream)>>>(
      P, Q, ldp, loc, b, m, D, ldd, eta_dev, zp, zq, e0, e1, WB, ldwb, Pb, Qb);
  return check_launch("pq_update_kernel");
}

int sap_combine(float *out, int64_t ldo, const float *P, const float *Q, int64_t ldp, int64_t n,
                int m, double a, double b, void *stream) {
  if (n < 0 || m <= 0) return fail(SAP_ERR_CONTRACT, "combine: bad shape");
  if (n == 0) return SAP_OK;
  const int64_t tot = n * m;
  combine_kernel<<<unsigned((tot + 255) / 256), 256, 0, S(stream)>>>(out, ldo, P, Q, ldp, n, m,
                                                                    float(a), float(b));
  return check_launch("combine_kernel");
}

int sap_sdd_update(float *V, float *W, float *E, int64_t ldv, int64_t rows, int m,
                   const int64_t *loc, int64_t b, const double *g, int64_t ldg, double eta,
                   double momentum, double avg, float *VB, int *pos, void *stream) {
  if (rows < 0 || m <= 0 || b < 0 || ldv < rows)
    return fail(SAP_ERR_CONTRACT, "sdd_update: bad shape");
  int rc;
  if (b > 0) {
    const int64_t tot = b * m;
    sdd_block_kernel<<<unsigned((tot + 255) / 256), 256, 0, S(stream)>>>(
        V, ldv, loc, b, m, g, ldg, eta, momentum, VB, pos);
    if ((rc = check_launch("sdd_block_kernel")) != SAP_OK) return rc;
  }
  if (rows == 0) return SAP_OK;
  if (rows % 4 || ldv % 4)
    return fail(SAP_ERR_CONTRACT, "sdd_update: rows and ldv must be multiples of 4");
  const int64_t rows4 = rows / 4;
  sdd_dense_kernel<<<unsigned((rows4 + 255) / 256), 256, 0, S(stream)>>>(
      V, W, E, ldv, rows4, m, VB, pos, float(momentum), float(avg));
  return check_launch("sdd_dense_kernel");
}

int sap_ktile64(const double *X, const double *inv_ls, int d, const int64_t *row_ids, int64_t na,
                const int64_t *col_ids, int64_t nc, int family, double variance, double *out,
                int64_t ldo, void *stream) {
  if (na <= 0 || nc <= 0 || d < 1 || ldo < nc)
    return fail(SAP_ERR_CONTRACT, "ktile64: bad shape");
  dim3 blk(32, 8), grid(unsigned((nc + 31) / 32), unsigned((na + 7) / 8));
  cudaStream_t st = S(stream);
  switch (family) {
    case SAP_RBF:
      ktile64_kernel<SAP_RBF><<<grid, blk, 0, st>>>(X, inv_ls, d, row_ids, na, col_ids, nc,
                                                    variance, out, ldo);
      break;
    case SAP_MATERN32:
      ktile64_kernel<SAP_MATERN32><<<grid, blk, 0, st>>>(X, inv_ls, d, row_ids, na, col_ids, nc,
                                                         variance, out, ldo);
      break;
    case SAP_MATERN52:
      ktile64_kernel<SAP_MATERN52><<<grid, blk, 0, st>>>(X, inv_ls, d, row_ids, na, col_ids, nc,
                                                         variance, out, ldo);
      break;
    default: return fail(SAP_ERR_CONTRACT, "ktile64: unknown family %d", family);
  }
  return check_launch("ktile64_kernel");
}

}  // extern "C"
