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
//                         columns; see build_aug in krows_tc.cu)     -> TMEM
//   epilogue P = 2^14 k(S) in registers (ex2/sqrt on MUFU), split into fp16
//                         hi + lo and written back over S            -> TMEM
//   GEMM2  G += P_hi Z_hi + P_hi Z_lo + P_lo Z_hi  kind::f16, A from TMEM,
//                         B = per-column-scaled fp16 split of Z (smem, TMA)
//
// The 3-term splits keep the product at fp32 accuracy (a single fp16/tf32
// pass would leave ~3e-4 relative error). One CTA per SM,
// persistent over (row tile, column split) work units; warp roles:
//   warp 0      TMA producer (STAGES-deep ring of 64-point X/Z tiles)
//   warp 1      MMA issuer (single thread): GEMM1 runs NB-1 tiles ahead
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: two warpgroups, one TMEM lane (= block row) per
//               thread, each warpgroup converts one 32-column half of a tile
// The TMEM accumulator is drained every kSeg tiles into fp32 registers (long
// tensor-core accumulation chains drift: 8.5e-5 relative at 2.7e4 points per
// chain, measured) and each unit's sum goes to a workspace that is reduced
// in fixed order (deterministic, no atomics).
//
// All loop bookkeeping of the two single-thread roles is incremental (no
// divisions) and smem descriptors are precomputed: those threads' serial
// instruction latency, not the tensor pipe, bounded the first version.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "zop.cuh"

namespace sap {
namespace tck {

constexpr int BM = 128;           // block rows per unit (TMEM lanes)
constexpr int NT = 64;            // points per column tile (GEMM1 N, one Z swizzle atom)
constexpr int NB = 4;             // S/P tiles in flight in TMEM
constexpr int kThreads = 384;     // 4 control warps + 2 epilogue warpgroups
constexpr int kSeg = 16;          // tiles per TMEM accumulator segment
constexpr float kPScale = 16384.0f;  // 2^14: keeps P's fp16 split out of subnormals
constexpr float kLn2 = 0.69314718055994531f;
constexpr float kPExp = 14.0f;         // log2 kPScale, folded into GEMM1 for RBF

// 2^x on the FMA pipe (MUFU is the epilogue's binding unit at 16 lanes/clk/SM
// against 128 for FFMA): round-to-nearest split x = j + f, f in [-1/2, 1/2],
// degree-5 fit of 2^f (max rel. error 2.4e-7 in fp32 Horner, the same as
// ex2.approx), exponent added as an integer. x is floored at -125 so j stays
// a normal exponent; 2^-125 is far below P's fp16 resolution.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.0f);
  const float t = __fadd_rn(x, 12582912.0f);            // 1.5 * 2^23: j in the low bits
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  float p = fmaf(f, 0.0013276224490255117f, 0.00967553909868002f);
  p = fmaf(p, f, 0.05550714209675789f);
  p = fmaf(p, f, 0.24022120237350464f);
  p = fmaf(p, f, 0.6931469440460205f);
  p = fmaf(p, f, 1.0000001192092896f);
  return __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23));
}

// which of the 32 entries of a TMEM chunk take the polynomial exp2 (measured
// sweeps, config 3, after the epilogue's clock instrumentation was compiled
// out: none for either family -- RBF 1/8 +2.4%, 1/4 +3.3%; Matern 1/8 +3.7%)
#ifndef SAP_POLY_RBF_MASK
#define SAP_POLY_RBF_MASK 0x0u
#endif
#ifndef SAP_POLY_MAT_MASK
#define SAP_POLY_MAT_MASK 0x0u
#endif
template <int FAM>
__host__ __device__ constexpr bool poly_entry(int e) {
  return (((FAM == SAP_RBF ? SAP_POLY_RBF_MASK : SAP_POLY_MAT_MASK) >> e) & 1u) != 0;
}
constexpr uint32_t kSmemCap = 227 * 1024;

struct Params {
  int64_t b;               // block rows
  int64_t ncols;           // points in this shard
  int64_t col_base;        // global id of point 0 (diagonal rule)
  const int64_t *row_ids;  // global ids of the block rows, NULL = no diagonal rule
  int m;                   // real RHS columns
  int row_tiles;
  int splits;
  int64_t tiles;           // column tiles of NT points
  float *part;             // [splits][m][b] partial sums (scaled; rows contiguous)
  int debug;               // profiling switches, 0 in production
  unsigned long long *prof;  // per-CTA role timers (SAP_TC_DEBUG=9), else NULL
  zop::Next zn;            // next iterate's operand (CTA-pair kernel side job; Zhi NULL: none)
  unsigned long long *sched;  // dynamic unit counter (CTA-pair kernel): high word = the launch's
                              // epoch, low word = units taken; NULL: static round-robin units
  unsigned epoch;             // this launch's tag (a counter left by another launch, or any
                              // stale value, is re-armed by the first fetch)
};

template <int NZ, int KA>
struct Geometry {
  static constexpr uint32_t a_bytes = BM * KA * 4;        // row tile (A of GEMM1)
  static constexpr uint32_t x_bytes = NT * KA * 4;        // column tile (B of GEMM1)
  static constexpr uint32_t z_bytes = NZ * 128;           // 64-point K atom of Z (hi or lo)
  static constexpr uint32_t stage_bytes = x_bytes + 2 * z_bytes;
  static constexpr uint32_t fixed = 1024 + 2 * a_bytes + 512;
  static constexpr uint32_t stages_raw = (kSmemCap - fixed) / stage_bytes;
  static constexpr uint32_t STAGES = stages_raw > 8 ? 8 : stages_raw;
  static constexpr uint32_t smem = fixed + STAGES * stage_bytes;
  static constexpr bool fits = STAGES >= NB;  // GEMM1 runs NB-1 tiles ahead of GEMM2
};

__device__ __forceinline__ void split_range(int64_t tiles, int splits, int s, int64_t &t0,
                                            int64_t &t1) {
  const int64_t q = tiles / splits, r = tiles % splits;
  t0 = s * q + (s < r ? s : r);
  t1 = t0 + q + (s < r ? 1 : 0);
}

// P = 2^14 k from the GEMM1 output S: for RBF S = 14 - s already (the offset
// and sign ride in the augmented features, build_aug_kernel); a tiny positive
// excess from rounding near s = 0 is harmless. Matern: S = s.
// Matern distance t = sqrt(|s|) (one MUFU.SQRT, the |.| folded into its
// operand) by default; SAP_MATERN_RSQ=1: t = s * rsqrt(max(s, 1e-30)) (two
// more instructions). Round 1 measured the sqrt form 0.9% slower; with the
// out-of-phase epilogue and the one-atomicAdd unit fetch it is 5.5% faster
// (config 3 krows 1.345-1.350 -> 1.270-1.275 ms, 3 A/B pairs)
#ifndef SAP_MATERN_RSQ
#define SAP_MATERN_RSQ 0
#endif
template <int FAM, bool POLY = false>
__device__ __forceinline__ float pvalue(float s) {
  if constexpr (FAM == SAP_RBF) {
    return POLY ? ex2_poly(s) : ex2_approx(s);
  } else if constexpr (FAM == SAP_COSINE) {
    // random-feature prior: P = 2^14 cos(s), s = x.F + p; reduced to
    // [-pi, pi] first (cos.approx is accurate to ~2^-21 there)
    const float r = s * 0.15915494309189535f;
    const float f = r - rintf(r);
    float c;
    asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(f * 6.283185307179586f));
    return kPScale * c;
  } else {
    // the 2^14 scale rides on the polynomial, so ex2 takes -t directly;
    // t = sqrt(|s|): |.| absorbs negative rounding near s = 0 (t ~ 0, k ~ 1)
    // and s = 0 gives t = 0 exactly (the rsqrt form needs a floor there)
#if SAP_MATERN_RSQ
    s = fmaxf(s, 1e-30f);
    const float t = s * rsqrt_approx(s);
#else
    const float t = sqrt_approx(fabsf(s));
#endif
    const float e = POLY ? ex2_poly(-t) : ex2_approx(-t);
    if constexpr (FAM == SAP_MATERN32) {
      return fmaf(t, kPScale * kLn2, kPScale) * e;
    } else {
      return fmaf(t, fmaf(t, kPScale * kLn2 * kLn2 / 3.0f, kPScale * kLn2), kPScale) * e;
    }
  }
}

#ifndef SAP_SPLIT_TRUNC
#define SAP_SPLIT_TRUNC 1
#endif
// fp16 hi/lo split of two P values. Truncating the fp32 mantissa to fp16's 11
// significant bits (LOP3, full-rate ALU) gives a hi that converts exactly and
// a lo = p - hi that is exact in fp32 before its own rounding, so P_hi + P_lo
// carries ~2^-23 relative error -- the same as a round-to-nearest hi, without
// the half-rate f16->f32 back-conversion. (Values under fp16's normal range,
// P < 2^-14 = 2^-28 of the largest kernel value, lose the exactness; their
// absolute error is negligible.)
__device__ __forceinline__ void split2(float p0, float p1, uint32_t &hi, uint32_t &lo) {
#if SAP_SPLIT_TRUNC
  const float h0 = __uint_as_float(__float_as_uint(p0) & 0xFFFFE000u);
  const float h1 = __uint_as_float(__float_as_uint(p1) & 0xFFFFE000u);
  const __half2 h = __floats2half2_rn(h0, h1);
  const __half2 l = __floats2half2_rn(__fsub_rn(p0, h0), __fsub_rn(p1, h1));
#else
  const __half2 h = __floats2half2_rn(p0, p1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(p0 - hf.x, p1 - hf.y);
#endif
  hi = *reinterpret_cast<const uint32_t *>(&h);
  lo = *reinterpret_cast<const uint32_t *>(&l);
}

// K-major SWIZZLE_128B descriptor with the start-address field left 0; the
// address (>> 4, < 2^14 for any smem address) is added to the low bits.
constexpr uint64_t kDescBase = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
                               (uint64_t(1) << 46) | (uint64_t(2) << 61);

template <int FAM, int NZ, int KA>
__global__ void __launch_bounds__(kThreads, 1)
    krows_tc_kernel(const __grid_constant__ CUtensorMap tm_rows,
                    const __grid_constant__ CUtensorMap tm_cols,
                    const __grid_constant__ CUtensorMap tm_zhi,
                    const __grid_constant__ CUtensorMap tm_zlo, const Params p) {
  using Geo = Geometry<NZ, KA>;
  constexpr uint32_t STAGES = Geo::STAGES;
  constexpr int KATOMS = KA / 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  uint8_t *sA = smem;                        // [2][a_bytes]
  uint8_t *sStage = smem + 2 * Geo::a_bytes;  // [STAGES][stage_bytes]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sStage + STAGES * Geo::stage_bytes);
  uint64_t *full = bars;                // [STAGES]  TMA -> MMA
  uint64_t *empty = full + STAGES;      // [STAGES]  MMA -> TMA
  uint64_t *a_full = empty + STAGES;    // [2]       row tile loaded
  uint64_t *a_empty = a_full + 2;       // [2]       row tile consumed
  uint64_t *s_full = a_empty + 2;       // [NB]      S tile ready (MMA -> epilogue)
  uint64_t *p_full = s_full + NB;       // [NB]      P tile ready (epilogue -> MMA)
  uint64_t *g_full = p_full + NB;       // [2]       accumulator segment done
  uint64_t *g_empty = g_full + 2;       // [2]       accumulator segment drained
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(g_empty + 2);

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < STAGES; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    for (int k = 0; k < NB; ++k) {
      tc::mbar_init(tc::smem_u32(&s_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&p_full[k]), 8);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(tc::smem_u32(&a_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&a_empty[k]), 1);
      tc::mbar_init(tc::smem_u32(&g_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&g_empty[k]), 8);
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

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (tc::elect_one()) {
      uint32_t s = 0, ph = 0;  // stage ring cursor
      int uc = 0;
      const uint32_t full0 = tc::smem_u32(full), empty0 = tc::smem_u32(empty);
      const uint32_t stage0 = tc::smem_u32(sStage);
      const uint32_t tx = p.debug == 3 ? Geo::x_bytes : Geo::stage_bytes;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const int rt = u % p.row_tiles, split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int ab = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_empty[ab]), ((uc >> 1) & 1) ^ 1);
        const uint32_t abar = tc::smem_u32(&a_full[ab]);
        tc::mbar_expect_tx(abar, Geo::a_bytes);
#pragma unroll
        for (int ka = 0; ka < KATOMS; ++ka)
          tc::tma_load_2d(tc::smem_u32(sA + ab * Geo::a_bytes + ka * BM * 128), &tm_rows, abar,
                          ka * 32, rt * BM);
        for (int64_t t = t0; t < t1; ++t) {
          tc::mbar_wait(empty0 + 8 * s, ph ^ 1);
          const uint32_t fbar = full0 + 8 * s;
          if (p.debug == 7) {
            tc::mbar_arrive(fbar);
            if (++s == STAGES) { s = 0; ph ^= 1; }
            continue;
          }
          tc::mbar_expect_tx(fbar, tx);
          const uint32_t st = stage0 + s * Geo::stage_bytes;
          const int32_t col0 = int32_t(t * NT);
#pragma unroll
          for (int ka = 0; ka < KATOMS; ++ka)
            tc::tma_load_2d(st + ka * NT * 128, &tm_cols, fbar, ka * 32, col0);
          if (p.debug != 3) {
            tc::tma_load_2d(st + Geo::x_bytes, &tm_zhi, fbar, col0, 0);
            tc::tma_load_2d(st + Geo::x_bytes + Geo::z_bytes, &tm_zlo, fbar, col0, 0);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (tc::elect_one()) {
      constexpr uint32_t id1 = tc::idesc(2, BM, NT);  // tf32, M=128, N=64
      constexpr uint32_t id2 = tc::idesc(0, BM, NZ);  // f16,  M=128, N=nz
      const uint32_t full0 = tc::smem_u32(full), empty0 = tc::smem_u32(empty);
      const uint32_t sfull0 = tc::smem_u32(s_full), pfull0 = tc::smem_u32(p_full);
      const uint64_t stage_desc0 = kDescBase | (tc::smem_u32(sStage) >> 4);
      const uint64_t a_desc0 = kDescBase | (tc::smem_u32(sA) >> 4);
      // GEMM1 cursor (runs NB-1 tiles ahead) and GEMM2 cursor
      uint32_t s1 = 0, ph1 = 0, r1 = 0;
      uint32_t s2 = 0, r2 = 0, ph2 = 0;
      uint32_t sc = 0;  // accumulator segment counter (G double buffer)
      int uc = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
        const int split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int nt = int(t1 - t0);
        const int ab = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_full[ab]), (uc >> 1) & 1);
        tc::fence_after();
        const uint64_t a_desc = a_desc0 + ((ab * Geo::a_bytes) >> 4);
        auto gemm1 = [&]() {
          tc::mbar_wait(full0 + 8 * s1, ph1);
          tc::fence_after();
          const uint64_t x_desc = stage_desc0 + ((s1 * Geo::stage_bytes) >> 4);
          const uint32_t d = tmem + r1 * NT;
#pragma unroll
          for (int k = 0; k < KA / 8; ++k) {
            if (p.debug >= 6) break;
            const uint32_t ko = ((k >> 2) * (BM * 128) + (k & 3) * 32) >> 4;
            const uint32_t kx = ((k >> 2) * (NT * 128) + (k & 3) * 32) >> 4;
            tc::mma_tf32_ss(d, a_desc + ko, x_desc + kx, id1, k > 0);
          }
          tc::commit(sfull0 + 8 * r1);
          if (++s1 == STAGES) { s1 = 0; ph1 ^= 1; }
          r1 = (r1 + 1) & (NB - 1);
        };
        const int pre = nt < NB - 1 ? nt : NB - 1;
        for (int j = 0; j < pre; ++j) gemm1();
        if (nt <= NB - 1) tc::commit(tc::smem_u32(&a_empty[ab]));
        uint32_t g_tmem = 0;
        int seg_j = 0;
        for (int j = 0; j < nt; ++j) {
          const bool seg_first = seg_j == 0;
          const bool seg_last = seg_j == kSeg - 1 || j + 1 == nt;
          if (seg_first) {
            const int gb = sc & 1;
            tc::mbar_wait(tc::smem_u32(&g_empty[gb]), ((sc >> 1) & 1) ^ 1);
            g_tmem = tmem + 256 + gb * NZ;
          }
          tc::mbar_wait(pfull0 + 8 * r2, ph2);
          tc::fence_after();
          const uint64_t zhi = stage_desc0 + ((s2 * Geo::stage_bytes + Geo::x_bytes) >> 4);
          const uint64_t zlo = zhi + (Geo::z_bytes >> 4);
          const uint32_t pbase = tmem + r2 * NT;
          if (p.debug < 4) {
#pragma unroll
            for (int c = 0; c < NT / 32; ++c) {
#pragma unroll
              for (int k16 = 0; k16 < 2; ++k16) {
                const uint32_t bo = (c * 64 + k16 * 32) >> 4;
                const uint32_t ahi = pbase + c * 32 + k16 * 8;
                const uint32_t acc0 = (!seg_first || c > 0 || k16 > 0) ? 1u : 0u;
                tc::mma_f16_ts(g_tmem, ahi, zhi + bo, id2, acc0);
                if (p.debug != 2) {
                  tc::mma_f16_ts(g_tmem, ahi, zlo + bo, id2, 1u);
                  tc::mma_f16_ts(g_tmem, ahi + 16, zhi + bo, id2, 1u);
                }
              }
            }
          }
          tc::commit(empty0 + 8 * s2);
          if (seg_last) {
            tc::commit(tc::smem_u32(&g_full[sc & 1]));
            ++sc;
            seg_j = 0;
          } else {
            ++seg_j;
          }
          if (++s2 == STAGES) s2 = 0;
          r2 = (r2 + 1) & (NB - 1);
          if (r2 == 0) ph2 ^= 1;
          // refill the ring: tile j+NB-1 reuses the S buffer of tile j-1,
          // whose P the GEMM2 above (in-order pipe) has already consumed
          if (j + NB - 1 < nt) {
            gemm1();
            if (j + NB == nt) tc::commit(tc::smem_u32(&a_empty[ab]));
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int h = (warp - 4) >> 2;          // epilogue warpgroup 0 or 1
    const int row_in_tile = q * 32 + lane;  // TMEM lane = block row within the tile
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    constexpr int NACC = ((NZ / 2 + 15) / 16) * 16;  // accumulator columns of warpgroup 0
    const int g0 = h ? NACC : 0, g1 = h ? NZ : NACC;
    const uint32_t sfull0 = tc::smem_u32(s_full), pfull0 = tc::smem_u32(p_full);
    uint32_t r = 0, ph = 0, sc = 0;
    float acc[NACC];  // fp32 accumulator of this row across the segments of a unit
#pragma unroll
    for (int c = 0; c < NACC; ++c) acc[c] = 0.0f;
    bool pend = false, pend_last = false, pend_live = false;
    float *pend_dst = nullptr;
    auto drain = [&]() {  // add a finished TMEM segment (one tile late)
      const int gb = sc & 1;
      tc::mbar_wait(tc::smem_u32(&g_full[gb]), (sc >> 1) & 1);
      tc::fence_after();
      const uint32_t gbase = tmem + lane_off + 256 + gb * NZ;
#pragma unroll
      for (int c0 = 0; c0 < NACC; c0 += 16) {
        if (g0 + c0 < g1) {
          uint32_t v[16];
          tc::ld16(gbase + g0 + c0, v);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&g_empty[gb]));
      ++sc;
      pend = false;
      if (pend_last) {
        if (pend_live) {
#pragma unroll
          for (int c = 0; c < NACC; ++c)
            if (g0 + c < g1 && g0 + c < p.m) pend_dst[int64_t(g0 + c) * p.b] = acc[c];
        }
#pragma unroll
        for (int c = 0; c < NACC; ++c) acc[c] = 0.0f;
      }
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int rt = u % p.row_tiles, split = u / p.row_tiles;
      int64_t t0, t1;
      split_range(p.tiles, p.splits, split, t0, t1);
      const int64_t grow = int64_t(rt) * BM + row_in_tile;
      const bool live = grow < p.b;
      float *dst = p.part + int64_t(split) * p.m * p.b + (live ? grow : 0);
      const int64_t rid = (p.row_ids && live) ? p.row_ids[grow] : INT64_MIN;
      if (t1 == t0 && live)
        for (int c = g0; c < g1 && c < p.m; ++c) dst[int64_t(c) * p.b] = 0.0f;
      int seg_j = 0;
      for (int64_t t = t0; t < t1; ++t) {
        tc::mbar_wait(sfull0 + 8 * r, ph);
        tc::fence_after();
        const uint32_t taddr = tmem + lane_off + r * NT + h * 32;
        if (p.debug >= 5) {
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(pfull0 + 8 * r);
          r = (r + 1) & (NB - 1);
          if (r == 0) ph ^= 1;
          if (pend) drain();
          if (seg_j == kSeg - 1 || t + 1 == t1) {
            pend = true; pend_last = t + 1 == t1; pend_live = live; pend_dst = dst; seg_j = 0;
          } else {
            ++seg_j;
          }
          continue;
        }
        uint32_t v[32];
        tc::ld32(taddr, v);
        tc::wait_ld();
        const int64_t dc64 = rid - (p.col_base + t * NT) - h * 32;  // diagonal column?
        const bool diag = dc64 >= 0 && dc64 < 32;
        const int dc = int(dc64);
        uint32_t hi[16], lo[16];
        if (p.debug == 1 || p.debug == 4) {
#pragma unroll
          for (int e = 0; e < 16; ++e) { hi[e] = v[2 * e]; lo[e] = v[2 * e + 1]; }
        } else if (__any_sync(0xffffffffu, diag)) {
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
          for (int e = 0; e < 32; e += 2) {
            const float x0 = __uint_as_float(v[e]), x1 = __uint_as_float(v[e + 1]);
            split2(poly_entry<FAM>(e) ? pvalue<FAM, true>(x0) : pvalue<FAM>(x0),
                   poly_entry<FAM>(e + 1) ? pvalue<FAM, true>(x1) : pvalue<FAM>(x1), hi[e / 2],
                   lo[e / 2]);
          }
        }
        tc::st16(taddr, hi);
        tc::st16(taddr + 16, lo);
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(pfull0 + 8 * r);
        r = (r + 1) & (NB - 1);
        if (r == 0) ph ^= 1;
        if (pend) drain();
        if (seg_j == kSeg - 1 || t + 1 == t1) {
          pend = true;
          pend_last = t + 1 == t1;
          pend_live = live;
          pend_dst = dst;
          seg_j = 0;
        } else {
          ++seg_j;
        }
      }
    }
    if (pend) drain();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem, 512);
}

template <int FAM, int NZ, int KA>
bool launch_tc_shape(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                     const CUtensorMap &zl, const Params &p, int grid, cudaStream_t st) {
  if constexpr (!Geometry<NZ, KA>::fits) {
    return false;
  } else {
    constexpr uint32_t smem = Geometry<NZ, KA>::smem;
    cudaFuncSetAttribute(krows_tc_kernel<FAM, NZ, KA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    krows_tc_kernel<FAM, NZ, KA><<<grid, kThreads, smem, st>>>(a, c, zh, zl, p);
    return true;
  }
}

template <int FAM>
bool launch_tc_family(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                      const CUtensorMap &zl, const Params &p, int nz, int ka, int grid,
                      cudaStream_t st) {
#define SAP_TC_KA(NZV)                                                             \
  return ka == 32 ? launch_tc_shape<FAM, NZV, 32>(a, c, zh, zl, p, grid, st)      \
                  : launch_tc_shape<FAM, NZV, 64>(a, c, zh, zl, p, grid, st);
  switch (nz) {
    case 16: SAP_TC_KA(16)
    case 32: SAP_TC_KA(32)
    case 48: SAP_TC_KA(48)
    case 64: SAP_TC_KA(64)
    case 80: SAP_TC_KA(80)
    case 96: SAP_TC_KA(96)
    case 112: SAP_TC_KA(112)
    case 128: SAP_TC_KA(128)
    default: return false;
  }
#undef SAP_TC_KA
}

// tc_fits(nz, ka): whether the tile ring of that shape fits shared memory
inline bool tc_fits(int nz, int ka) {
  const uint32_t stage = NT * ka * 4 + 2 * nz * 128;
  const uint32_t fixed = 1024 + 2 * BM * ka * 4 + 512;
  return nz % 16 == 0 && nz >= 16 && nz <= 128 && (ka == 32 || ka == 64) &&
         (kSmemCap - fixed) / stage >= uint32_t(NB);
}

}  // namespace tck
}  // namespace sap
