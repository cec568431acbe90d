// Tensor-core (tcgen05 / TMEM / TMA) block-row kernel product for sm_100a:
//
//   G[i, c] = variance * sum_j k(x_{B_i}, x_j) * Z[j, c]        (dist.py:108-127)
//
// structured like a flash-attention forward pass with the softmax replaced by
// the covariance function and no running max:
//
//   GEMM1  S = A . C^T    kind::tf32, 3-term split (hi*hi + hi*lo + lo*hi) of
//                         augmented features, so S = c_fam * |x_i - x_j|^2 to
//                         ~1e-6 (the squared norms ride along as extra K
//                         columns; see build_aug below)           -> TMEM
//   epilogue P = 2^14 k(S) in registers (ex2/sqrt on MUFU), split into fp16
//                         hi + lo and written back over S            -> TMEM
//   GEMM2  G += P_hi Z_hi + P_hi Z_lo + P_lo Z_hi  kind::f16, A from TMEM,
//                         B = per-column-scaled fp16 split of Z (smem, TMA)
//
// The 3-term splits keep the product at fp32 accuracy (a single fp16/tf32
// pass would leave ~3e-4 relative error). Warp roles (one CTA
// per SM, persistent over (row tile, column split) work units):
//   warp 0      TMA producer (X/Z column tiles, 3-4 stage ring; row tile A)
//   warp 1      MMA issuer (single thread): GEMM1(j+1) overlaps epilogue(j)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: one TMEM lane (= one block row) per thread
// Per-unit partial sums go to a workspace and are reduced in a fixed order
// (deterministic, no atomics), with the variance and the per-column Z scale
// undone in the reduction.
#include <cstdio>
#include <cstdarg>
#include <mutex>

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace tck {

constexpr int BM = 128;          // block rows per unit (TMEM lanes)
constexpr int NT = 128;          // points per column tile (GEMM1 N)
constexpr int kThreads = 256;
constexpr float kPScale = 16384.0f;  // 2^14: keeps P's fp16 split out of subnormals
constexpr float kLn2 = 0.69314718055994531f;

struct Params {
  int64_t b;          // block rows
  int64_t ncols;      // points in this shard
  int64_t col_base;   // global id of point 0 (diagonal rule)
  const int64_t *row_ids;  // global ids of the block rows, NULL = no diagonal rule
  int ka;             // augmented feature width (32 or 64)
  int nz;             // GEMM2 N (RHS columns padded to 16)
  int m;              // real RHS columns
  int row_tiles;
  int splits;
  int64_t tiles;      // column tiles of NT points
  int stages;
  float *part;        // [splits][b][m] partial sums (scaled)
};

__device__ __forceinline__ void split_range(int64_t tiles, int splits, int s, int64_t &t0,
                                            int64_t &t1) {
  const int64_t q = tiles / splits, r = tiles % splits;
  t0 = s * q + (s < r ? s : r);
  t1 = t0 + q + (s < r ? 1 : 0);
}

template <int FAM>
__device__ __forceinline__ float pvalue(float s) {
  s = fmaxf(s, 0.0f);
  if constexpr (FAM == SAP_RBF) {
    return ex2_approx(14.0f - s);
  } else {
    const float t = sqrt_approx(s);
    const float e = ex2_approx(14.0f - t);
    if constexpr (FAM == SAP_MATERN32) {
      return fmaf(t, kLn2, 1.0f) * e;
    } else {
      return fmaf(t, fmaf(t, kLn2 * kLn2 / 3.0f, kLn2), 1.0f) * e;
    }
  }
}

__device__ __forceinline__ void split2(float p0, float p1, uint32_t &hi, uint32_t &lo) {
  const __half2 h = __floats2half2_rn(p0, p1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(p0 - hf.x, p1 - hf.y);
  hi = *reinterpret_cast<const uint32_t *>(&h);
  lo = *reinterpret_cast<const uint32_t *>(&l);
}

template <int FAM>
__global__ void __launch_bounds__(kThreads, 1)
    krows_tc_kernel(const __grid_constant__ CUtensorMap tm_rows,
                    const __grid_constant__ CUtensorMap tm_cols,
                    const __grid_constant__ CUtensorMap tm_zhi,
                    const __grid_constant__ CUtensorMap tm_zlo, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  const uint32_t a_bytes = BM * p.ka * 4;              // row tile (A of GEMM1)
  const uint32_t x_bytes = NT * p.ka * 4;              // column tile (B of GEMM1)
  const uint32_t zatom = p.nz * 128;                   // one 64-point K atom of Z
  const uint32_t z_bytes = 2 * zatom;                  // NT = 128 points = 2 atoms
  const uint32_t stage_bytes = x_bytes + 2 * z_bytes;  // X + Z_hi + Z_lo
  uint8_t *sA = smem;                                  // [2][a_bytes]
  uint8_t *sStage = smem + 2 * a_bytes;                // [stages][stage_bytes]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sStage + p.stages * stage_bytes);
  // barrier slots
  uint64_t *full = bars;                 // [stages]
  uint64_t *empty = bars + p.stages;     // [stages]
  uint64_t *a_full = empty + p.stages;   // [2]
  uint64_t *a_empty = a_full + 2;        // [2]
  uint64_t *s_full = a_empty + 2;        // [2]
  uint64_t *p_full = s_full + 2;         // [2]
  uint64_t *g_full = p_full + 2;         // [2]
  uint64_t *g_empty = g_full + 2;        // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(g_empty + 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(tc::smem_u32(&a_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&a_empty[k]), 1);
      tc::mbar_init(tc::smem_u32(&s_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&p_full[k]), 4);
      tc::mbar_init(tc::smem_u32(&g_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&g_empty[k]), 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_rows);
    tc::prefetch_tmap(&tm_cols);
    tc::prefetch_tmap(&tm_zhi);
    tc::prefetch_tmap(&tm_zlo);
  }
  if (warp == 2) {
    tc::tmem_alloc(tc::smem_u32(tmem_slot), 512);
    tc::tmem_relinquish();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int units = p.row_tiles * p.splits;
  const int katoms = p.ka / 32;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (tc::elect_one()) {
      uint32_t it = 0;  // global stage counter
      int uc = 0;       // unit counter of this CTA
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const int rt = u % p.row_tiles, split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int ab = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_empty[ab]), ((uc >> 1) & 1) ^ 1);
        const uint32_t abar = tc::smem_u32(&a_full[ab]);
        tc::mbar_expect_tx(abar, a_bytes);
        for (int ka = 0; ka < katoms; ++ka)
          tc::tma_load_2d(tc::smem_u32(sA + ab * a_bytes + ka * BM * 128), &tm_rows, abar, ka * 32,
                          rt * BM);
        for (int64_t t = t0; t < t1; ++t, ++it) {
          const uint32_t s = it % p.stages;
          tc::mbar_wait(tc::smem_u32(&empty[s]), ((it / p.stages) & 1) ^ 1);
          const uint32_t fbar = tc::smem_u32(&full[s]);
          tc::mbar_expect_tx(fbar, stage_bytes);
          uint8_t *st = sStage + s * stage_bytes;
          const int32_t col0 = int32_t(t * NT);
          for (int ka = 0; ka < katoms; ++ka)
            tc::tma_load_2d(tc::smem_u32(st + ka * NT * 128), &tm_cols, fbar, ka * 32, col0);
          for (int za = 0; za < 2; ++za) {
            tc::tma_load_2d(tc::smem_u32(st + x_bytes + za * zatom), &tm_zhi, fbar,
                            col0 + za * 64, 0);
            tc::tma_load_2d(tc::smem_u32(st + x_bytes + z_bytes + za * zatom), &tm_zlo, fbar,
                            col0 + za * 64, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (tc::elect_one()) {
      const uint32_t id1 = tc::idesc(2, BM, NT);      // tf32, M=128, N=128
      const uint32_t id2 = tc::idesc(0, BM, p.nz);    // f16,  M=128, N=nz
      uint32_t it = 0;   // stage counter (matches producer)
      uint32_t tcn = 0;  // tile counter (S/P double buffer)
      int uc = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const int split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int nt = int(t1 - t0);
        const int ab = uc & 1, gb = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_full[ab]), (uc >> 1) & 1);
        tc::mbar_wait(tc::smem_u32(&g_empty[gb]), ((uc >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t a_base = tc::smem_u32(sA + ab * a_bytes);
        const uint32_t g_tmem = tmem + 256 + gb * p.nz;
        auto gemm1 = [&](uint32_t itj, uint32_t tcj) {
          const uint32_t s = itj % p.stages;
          tc::mbar_wait(tc::smem_u32(&full[s]), (itj / p.stages) & 1);
          tc::fence_after();
          const uint32_t x_base = tc::smem_u32(sStage + s * stage_bytes);
          const uint32_t d = tmem + (tcj & 1) * NT;
#pragma unroll 1
          for (int k = 0; k < p.ka / 8; ++k) {
            const uint32_t koff = (k >> 2) * (BM * 128) + (k & 3) * 32;
            const uint32_t koffx = (k >> 2) * (NT * 128) + (k & 3) * 32;
            tc::mma_tf32_ss(d, tc::sdesc_k_sw128(a_base + koff, 1024),
                            tc::sdesc_k_sw128(x_base + koffx, 1024), id1, k > 0);
          }
          tc::commit(tc::smem_u32(&s_full[tcj & 1]));
        };
        if (nt > 0) gemm1(it, tcn);
        for (int j = 0; j < nt; ++j) {
          const uint32_t itj = it + j, tcj = tcn + j;
          if (j + 1 < nt) gemm1(itj + 1, tcj + 1);
          if (j + 1 == nt) tc::commit(tc::smem_u32(&a_empty[ab]));  // all GEMM1 of the unit issued
          tc::mbar_wait(tc::smem_u32(&p_full[tcj & 1]), (tcj >> 1) & 1);
          tc::fence_after();
          const uint32_t s = itj % p.stages;
          const uint32_t zhi = tc::smem_u32(sStage + s * stage_bytes + x_bytes);
          const uint32_t zlo = zhi + z_bytes;
          const uint32_t pbase = tmem + (tcj & 1) * NT;
#pragma unroll 1
          for (int c = 0; c < NT / 32; ++c) {
#pragma unroll
            for (int k16 = 0; k16 < 2; ++k16) {
              const uint32_t boff = (c >> 1) * zatom + (c & 1) * 64 + k16 * 32;
              const uint64_t bh = tc::sdesc_k_sw128(zhi + boff, 1024);
              const uint64_t bl = tc::sdesc_k_sw128(zlo + boff, 1024);
              const uint32_t ahi = pbase + c * 32 + k16 * 8;
              const uint32_t alo = ahi + 16;
              const uint32_t acc0 = (j > 0 || c > 0 || k16 > 0) ? 1u : 0u;
              tc::mma_f16_ts(g_tmem, ahi, bh, id2, acc0);
              tc::mma_f16_ts(g_tmem, ahi, bl, id2, 1u);
              tc::mma_f16_ts(g_tmem, alo, bh, id2, 1u);
            }
          }
          tc::commit(tc::smem_u32(&empty[s]));
        }
        if (nt == 0) tc::commit(tc::smem_u32(&a_empty[ab]));
        tc::commit(tc::smem_u32(&g_full[gb]));
        it += nt;
        tcn += nt;
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int row_in_tile = q * 32 + lane;  // TMEM lane = block row within the tile
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    uint32_t tcn = 0;
    int uc = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
      const int rt = u % p.row_tiles, split = u / p.row_tiles;
      int64_t t0, t1;
      split_range(p.tiles, p.splits, split, t0, t1);
      const int64_t grow = int64_t(rt) * BM + row_in_tile;
      const int64_t rid = (p.row_ids && grow < p.b) ? p.row_ids[grow] : INT64_MIN;
      for (int64_t t = t0; t < t1; ++t, ++tcn) {
        const int buf = tcn & 1;
        tc::mbar_wait(tc::smem_u32(&s_full[buf]), (tcn >> 1) & 1);
        tc::fence_after();
        const uint32_t sbase = tmem + lane_off + buf * NT;
        const int64_t dcol = rid - (p.col_base + t * NT);  // diagonal column in this tile?
#pragma unroll 1
        for (int c = 0; c < NT / 32; ++c) {
          uint32_t v[32];
          tc::ld32(sbase + c * 32, v);
          tc::wait_ld();
          const int dc = int(dcol - c * 32);
          const bool diag = dcol >= c * 32 && dcol < c * 32 + 32;
          uint32_t hi[16], lo[16];
          if (__any_sync(0xffffffffu, diag)) {
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              float p0 = pvalue<FAM>(__uint_as_float(v[e]));
              float p1 = pvalue<FAM>(__uint_as_float(v[e + 1]));
              if (diag && dc == e) p0 = kPScale;
              if (diag && dc == e + 1) p1 = kPScale;
              split2(p0, p1, hi[e / 2], lo[e / 2]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; e += 2)
              split2(pvalue<FAM>(__uint_as_float(v[e])), pvalue<FAM>(__uint_as_float(v[e + 1])),
                     hi[e / 2], lo[e / 2]);
          }
          tc::st16(sbase + c * 32, hi);
          tc::st16(sbase + c * 32 + 16, lo);
        }
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[buf]));
      }
      // unit done: drain G (nz fp32 columns) into the partial-sum workspace
      const int gb = uc & 1;
      tc::mbar_wait(tc::smem_u32(&g_full[gb]), (uc >> 1) & 1);
      tc::fence_after();
      const uint32_t gbase = tmem + lane_off + 256 + gb * p.nz;
      float *dst = p.part + (int64_t(split) * p.b + grow) * p.m;
      const bool live = grow < p.b;
      for (int c0 = 0; c0 < p.nz; c0 += 16) {
        uint32_t v[16];
        tc::ld16(gbase + c0, v);
        tc::wait_ld();
        if (live) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c0 + e < p.m) dst[c0 + e] = (t1 > t0) ? __uint_as_float(v[e]) : 0.0f;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&g_empty[gb]));
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// augmented features for the 3-term tf32 distance GEMM
//
// With z = x * sqrt(c_fam) / lengthscale and n = |z|^2 (fp64), hi() the tf32
// truncation and lo() the tf32-rounded remainder:
//   row form    [ zh, zh, zl, nh, nl, 1, 1, 0... ]
//   column form [-2zh, -2zl, -2zh, 1, 1, nh, nl, 0... ]
// so <row_i, col_j> = |z_i|^2 + |z_j|^2 - 2 z_i.z_j (to ~2^-20 |z|^2) =
// c_fam * squared scaled distance (kernels.py:123-125).

__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void build_aug_kernel(const double *X, int64_t n, int d, const double *inv_ls,
                                 double cfam, int ka, float *RA, float *CA) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double sc = sqrt(cfam);
  double nrm = 0.0;
  float *ra = RA ? RA + j * ka : nullptr;
  float *ca = CA ? CA + j * ka : nullptr;
  for (int k = 0; k < d; ++k) {
    const double z = X[j * d + k] * inv_ls[k] * sc;
    nrm = fma(z, z, nrm);
    const float zh = tf32_trunc(float(z));
    const float zl = tf32_round(float(z - double(zh)));
    if (ra) { ra[k] = zh; ra[d + k] = zh; ra[2 * d + k] = zl; }
    if (ca) { ca[k] = -2.0f * zh; ca[d + k] = -2.0f * zl; ca[2 * d + k] = -2.0f * zh; }
  }
  const float nh = tf32_trunc(float(nrm));
  const float nl = tf32_round(float(nrm - double(nh)));
  const int o = 3 * d;
  if (ra) { ra[o] = nh; ra[o + 1] = nl; ra[o + 2] = 1.0f; ra[o + 3] = 1.0f; }
  if (ca) { ca[o] = 1.0f; ca[o + 1] = 1.0f; ca[o + 2] = nh; ca[o + 3] = nl; }
  for (int k = o + 4; k < ka; ++k) {
    if (ra) ra[k] = 0.0f;
    if (ca) ca[k] = 0.0f;
  }
}

__global__ void gather_rows_kernel(const float *RA, int ka, const int64_t *idx, int64_t b,
                                   int64_t bpad, float *out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= bpad * ka) return;
  const int64_t i = e / ka;
  out[e] = i < b ? RA[idx[i] * ka + (e % ka)] : 0.0f;
}

// Z operand: ZT_hi/ZT_lo[c][j] = fp16 split of scale_c * (zp P[c][j] + zq Q[c][j]),
// scale_c = 2^floor(log2(16384 / bound_c)) from per-column magnitude bounds.
__global__ void z_operand_kernel(const float *P, const float *Q, int64_t ldp, int64_t n, int m,
                                 float zp, float zq, const float *Pb, const float *Qb, int nz,
                                 int64_t ldz, __half *Zhi, __half *Zlo, float *zscale) {
  const int c = blockIdx.y;
  float bound = fabsf(zp) * Pb[c] + (Q ? fabsf(zq) * Qb[c] : 0.0f);
  float sc = 1.0f;
  if (c < m && bound > 0.0f && isfinite(bound)) sc = exp2f(floorf(log2f(16384.0f / bound)));
  sc = fminf(fmaxf(sc, 0x1p-100f), 0x1p100f);
  if (blockIdx.x == 0 && threadIdx.x == 0) zscale[c] = sc;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ldz;
       j += int64_t(gridDim.x) * blockDim.x) {
    float z = 0.0f;
    if (c < m && j < n) {
      z = zp * P[int64_t(c) * ldp + j];
      if (Q) z = fmaf(zq, Q[int64_t(c) * ldp + j], z);
      z *= sc;
    }
    const __half h = __float2half_rn(z);
    Zhi[int64_t(c) * ldz + j] = h;
    Zlo[int64_t(c) * ldz + j] = __float2half_rn(z - __half2float(h));
  }
}

// per-column max |A| (magnitude bounds for RHS that are not solver state)
__global__ void colabsmax_kernel(const float *A, int64_t lda, int64_t n, float *out) {
  const int c = blockIdx.y;
  float mx = 0.0f;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x)
    mx = fmaxf(mx, fabsf(A[int64_t(c) * lda + j]));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(out + c), __float_as_int(mx));
}

__global__ void tc_reduce_kernel(const float *part, int splits, int64_t b, int m, float variance,
                                 const float *zscale, float *out, int64_t ldo, int accumulate) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int64_t i = e / m;
  const int c = int(e % m);
  float s = 0.0f;
  for (int k = 0; k < splits; ++k) s += part[int64_t(k) * b * m + e];
  const float v = s * (variance / (kPScale * zscale[c]));
  float *o = out + i * ldo + c;
  *o = accumulate ? *o + v : v;
}

// ---------------------------------------------------------------------------
// host side

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}

bool make_map(CUtensorMap *m, CUtensorMapDataType dt, const void *base, uint64_t inner,
              uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kSms = 148;

int tc_splits(int64_t b, int64_t tiles) {
  const int64_t rt = (b + BM - 1) / BM;
  int64_t best = 1;
  double best_eff = -1.0;
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(tiles / 4, 4096));
  for (int64_t s = 1; s <= std::min<int64_t>(max_s, 8 * kSms); ++s) {
    const int64_t total = rt * s;
    const int64_t waves = (total + kSms - 1) / kSms;
    if (waves > 8) break;
    const double eff = double(total) / double(waves * kSms);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return int(best);
}

}  // namespace tck
}  // namespace sap

using namespace sap;
using namespace sap::tck;

extern "C" {

int sap_tc_points(const double *X, int64_t n, int d, const double *inv_ls, int family, int ka,
                  float *RA, float *CA, void *stream) {
  if (n < 0 || d < 1 || (ka != 32 && ka != 64) || 3 * d + 4 > ka)
    return fail(SAP_ERR_CONTRACT, "tc_points: d=%d does not fit ka=%d", d, ka);
  const double l2e = 1.4426950408889634;
  double cfam = family == SAP_RBF ? 0.5 * l2e : (family == SAP_MATERN32 ? 3.0 : 5.0) * l2e * l2e;
  if (n == 0) return SAP_OK;
  build_aug_kernel<<<unsigned((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(X, n, d, inv_ls,
                                                                               cfam, ka, RA, CA);
  return check_launch("build_aug_kernel");
}

int sap_tc_gather_rows(const float *RA, int ka, const int64_t *idx, int64_t b, int64_t bpad,
                       float *out, void *stream) {
  if (b <= 0 || bpad < b) return fail(SAP_ERR_CONTRACT, "tc_gather_rows: bad shape");
  const int64_t tot = bpad * ka;
  gather_rows_kernel<<<unsigned((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(RA, ka, idx, b,
                                                                                   bpad, out);
  return check_launch("gather_rows_kernel");
}

int sap_z_operand(const float *P, const float *Q, int64_t ldp, int64_t n, int m, double zp,
                  double zq, const float *Pb, const float *Qb, int nz, int64_t ldz, void *Zhi,
                  void *Zlo, float *zscale, void *stream) {
  if (m <= 0 || nz < m || nz % 16 || ldz < n || ldz % 8)
    return fail(SAP_ERR_CONTRACT, "z_operand: bad shape m=%d nz=%d ldz=%lld", m, nz,
                (long long)ldz);
  dim3 grid(unsigned(std::min<int64_t>((ldz + 255) / 256, 256)), unsigned(nz));
  z_operand_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      P, Q, ldp, n, m, float(zp), float(zq), Pb, Qb, nz, ldz, static_cast<__half *>(Zhi),
      static_cast<__half *>(Zlo), zscale);
  return check_launch("z_operand_kernel");
}

int sap_colabsmax(const float *A, int64_t lda, int64_t n, int m, float *out, void *stream) {
  if (m <= 0 || n < 0) return fail(SAP_ERR_CONTRACT, "colabsmax: bad shape");
  if (cudaMemsetAsync(out, 0, sizeof(float) * m, (cudaStream_t)stream) != cudaSuccess)
    return fail(SAP_ERR_DEVICE, "colabsmax: memset failed");
  if (n == 0) return SAP_OK;
  dim3 grid(unsigned(std::min<int64_t>((n + 255) / 256, 128)), unsigned(m));
  colabsmax_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, n, out);
  return check_launch("colabsmax_kernel");
}

size_t sap_krows_tc_workspace(int64_t b, int m, int64_t ncols) {
  const int64_t tiles = (ncols + NT - 1) / NT;
  return size_t(tc_splits(b, tiles)) * size_t(b) * size_t(m) * sizeof(float);
}

int sap_krows_tc(const float *CA, int64_t ncols, int ka, const float *RAg, int64_t bpad,
                 const int64_t *row_ids, int64_t b, int64_t col_base, const void *Zhi,
                 const void *Zlo, int nz, int64_t ldz, const float *zscale, int m, int family,
                 double variance, float *out, int64_t ldo, int accumulate, void *ws,
                 size_t ws_bytes, void *stream) {
  if (b <= 0 || m <= 0 || ncols <= 0 || (ka != 32 && ka != 64) || nz % 16 || nz < m ||
      nz > 128 || bpad % BM || bpad < b || ldz % 8 || ldz < ncols)
    return fail(SAP_ERR_CONTRACT, "krows_tc: bad shape b=%lld m=%d nz=%d ncols=%lld ka=%d",
                (long long)b, m, nz, (long long)ncols, ka);
  if (ldo < m) return fail(SAP_ERR_CONTRACT, "krows_tc: ldo < m");
  const int64_t tiles = (ncols + NT - 1) / NT;
  Params p{};
  p.b = b;
  p.ncols = ncols;
  p.col_base = col_base;
  p.row_ids = row_ids;
  p.ka = ka;
  p.nz = nz;
  p.m = m;
  p.row_tiles = int(bpad / BM);
  p.tiles = tiles;
  p.splits = tc_splits(b, tiles);
  const size_t need = size_t(p.splits) * size_t(b) * size_t(m) * sizeof(float);
  if (!ws || ws_bytes < need)
    return fail(SAP_ERR_CONTRACT, "krows_tc: workspace %zu < %zu bytes", ws_bytes, need);
  p.part = static_cast<float *>(ws);
  const size_t a_bytes = size_t(BM) * ka * 4, x_bytes = size_t(NT) * ka * 4;
  const size_t stage_bytes = x_bytes + 4 * size_t(nz) * 128;
  const size_t fixed = 1024 + 2 * a_bytes + 256;
  const size_t cap = 227 * 1024;
  int stages = int(std::min<size_t>(4, (cap - fixed) / stage_bytes));
  if (stages < 2) return fail(SAP_ERR_CONTRACT, "krows_tc: tile does not fit shared memory");
  p.stages = stages;
  const size_t smem = fixed + size_t(stages) * stage_bytes;

  CUtensorMap tm_rows, tm_cols, tm_zhi, tm_zlo;
  if (!make_map(&tm_rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, RAg, ka, bpad, size_t(ka) * 4, 32, BM) ||
      !make_map(&tm_cols, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CA, ka, ncols, size_t(ka) * 4, 32, NT) ||
      !make_map(&tm_zhi, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Zhi, ncols, nz, size_t(ldz) * 2, 64, nz) ||
      !make_map(&tm_zlo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Zlo, ncols, nz, size_t(ldz) * 2, 64, nz))
    return fail(SAP_ERR_DEVICE, "krows_tc: cuTensorMapEncodeTiled failed");

  cudaStream_t st = (cudaStream_t)stream;
  const int units = p.row_tiles * p.splits;
  const int grid = std::min(units, kSms);
  int rc;
  switch (family) {
#define SAP_TC_LAUNCH(F)                                                                      \
  cudaFuncSetAttribute(krows_tc_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                       int(smem));                                                           \
  krows_tc_kernel<F><<<grid, kThreads, smem, st>>>(tm_rows, tm_cols, tm_zhi, tm_zlo, p);     \
  break;
    case SAP_RBF: SAP_TC_LAUNCH(SAP_RBF)
    case SAP_MATERN32: SAP_TC_LAUNCH(SAP_MATERN32)
    case SAP_MATERN52: SAP_TC_LAUNCH(SAP_MATERN52)
#undef SAP_TC_LAUNCH
    default: return fail(SAP_ERR_CONTRACT, "krows_tc: unknown family %d", family);
  }
  if ((rc = check_launch("krows_tc_kernel")) != SAP_OK) return rc;
  const int64_t tot = b * m;
  tc_reduce_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(p.part, p.splits, b, m,
                                                                float(variance), zscale, out, ldo,
                                                                accumulate);
  return check_launch("tc_reduce_kernel");
}

}  // extern "C"
