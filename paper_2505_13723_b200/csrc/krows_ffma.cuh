// FFMA implementation of the block-row kernel product
//   out[i, c] = variance * sum_j k(r_i, x_j) * R[j, c],   R = ca*A + cb*Bm
// (reference: dist.py:108-147 over kernels.py:118-127).
//
// This is the general-shape path: any d <= 64, any m, any row/column point
// sets (K1 block rows, K2 sketch K[B,B]Omega, K4 prediction, K5 full
// residual). The north-star shape (m = 65) runs on the tcgen05 kernel in
// krows_tc.cuh; this kernel also serves as its on-device cross-check.
//
// CTA = 256 threads, a 128-row tile of r_i against 32-point column tiles:
//   phase A: each thread evaluates 16 kernel entries (row coords in
//            registers, column coords broadcast from smem) -> Ks[32][128];
//   phase B: register-blocked rank-32 update acc[8 rows][MT cols] from
//            Ks (LDS.128) and the RHS tile Rt[32][16*MT+1].
// The next column tile is prefetched into registers during phase B.
// Columns are split over gridDim.y; partials go to a workspace and are
// reduced in fixed split order (deterministic, no atomics).
#pragma once

#include "common.cuh"

namespace sap {

constexpr int kFfmaThreads = 256;
constexpr int kFfmaBM = 128;  // rows per CTA
constexpr int kFfmaBN = 32;   // points per column tile

struct KrowsParams {
  const float *Xs, *sqn;
  int ldx;
  int64_t ncols;
  const int64_t *col_ids;
  int64_t col_base;
  const float *Rs, *rsqn;
  const int64_t *row_ids;
  int64_t b;
  const float *A, *Bm;
  int64_t lda;
  int m;            // columns handled by this launch (<= 16*MT)
  int c0;           // first RHS column of this launch
  float ca, cb;
  float variance;
  float *out;       // final output (splits == 1) or workspace partials
  int64_t ldo;
  int accumulate;
  int splits;
  int64_t tiles;    // number of 32-point column tiles
};

template <int FAM, int DP, int MT>
__global__ void __launch_bounds__(kFfmaThreads, (MT <= 5 && DP <= 16) ? 2 : 1)
    krows_ffma_kernel(const KrowsParams p) {
  constexpr int MC = 16 * MT;
  constexpr int MCP = MC + 1;
  constexpr int XV = kFfmaBN * DP / 4;                 // float4 per column-coord tile
  constexpr int XPER = (XV + kFfmaThreads - 1) / kFfmaThreads;
  constexpr int RPER = MC * kFfmaBN / kFfmaThreads;    // RHS elements per thread (MT*2)

  __shared__ __align__(16) float Ks[kFfmaBN][kFfmaBM];
  __shared__ __align__(16) float Xc[kFfmaBN * DP];
  __shared__ float Cn[kFfmaBN];
  __shared__ int64_t Cid[kFfmaBN];
  __shared__ float Rt[kFfmaBN * MCP];

  const int tid = threadIdx.x;
  const int64_t row0 = int64_t(blockIdx.x) * kFfmaBM;
  const int split = blockIdx.y;

  // column tile range of this split (balanced contiguous partition)
  const int64_t q = p.tiles / p.splits, rem = p.tiles % p.splits;
  const int64_t t_begin = split * q + (split < rem ? split : rem);
  const int64_t t_end = t_begin + q + (split < rem ? 1 : 0);

  // phase-A identity: one row, 16 of the 32 columns
  const int arow = tid % kFfmaBM;
  const int ahalf = tid / kFfmaBM;
  const int64_t grow = row0 + arow;
  float rc[DP];
  float rn = 0.0f;
  int64_t rid = -1;
  if (grow < p.b) {
    const float4 *src = reinterpret_cast<const float4 *>(p.Rs + grow * p.ldx);
#pragma unroll
    for (int k = 0; k < DP / 4; ++k) {
      float4 v = src[k];
      rc[4 * k] = v.x; rc[4 * k + 1] = v.y; rc[4 * k + 2] = v.z; rc[4 * k + 3] = v.w;
    }
    rn = p.rsqn[grow];
    if (p.row_ids) rid = p.row_ids[grow];
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) rc[k] = 0.0f;
  }

  // phase-B identity: rows tr*8..+7, columns tc + 16*k
  const int tr = tid / 16, tc = tid % 16;
  float acc[8][MT];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int k = 0; k < MT; ++k) acc[r][k] = 0.0f;

  // register staging for the prefetch
  float4 xs[XPER];
  float cn_st = 0.0f;
  int64_t cid_st = -1;
  float rs[RPER];

  auto load_tile = [&](int64_t t) {
    const int64_t j0 = t * kFfmaBN;
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int v = tid + u * kFfmaThreads;
      xs[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (v < XV) {
        const int jj = v / (DP / 4), kk = v % (DP / 4);
        if (j0 + jj < p.ncols)
          xs[u] = reinterpret_cast<const float4 *>(p.Xs + (j0 + jj) * p.ldx)[kk];
      }
    }
    if (tid < kFfmaBN) {
      const int64_t j = j0 + tid;
      cn_st = j < p.ncols ? p.sqn[j] : 0.0f;
      cid_st = j < p.ncols ? (p.col_ids ? p.col_ids[j] : p.col_base + j) : -2;
    }
    const int jl = tid % kFfmaBN;
    const int64_t j = j0 + jl;
#pragma unroll
    for (int u = 0; u < RPER; ++u) {
      const int c = tid / kFfmaBN + u * (kFfmaThreads / kFfmaBN);
      float v = 0.0f;
      if (j < p.ncols && c < p.m) {
        const int64_t off = int64_t(p.c0 + c) * p.lda + j;
        v = p.ca * p.A[off];
        if (p.Bm) v = fmaf(p.cb, p.Bm[off], v);
      }
      rs[u] = v;
    }
  };
  auto store_tile = [&]() {
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int v = tid + u * kFfmaThreads;
      if (v < XV) reinterpret_cast<float4 *>(Xc)[v] = xs[u];
    }
    if (tid < kFfmaBN) { Cn[tid] = cn_st; Cid[tid] = cid_st; }
    const int jl = tid % kFfmaBN;
#pragma unroll
    for (int u = 0; u < RPER; ++u) {
      const int c = tid / kFfmaBN + u * (kFfmaThreads / kFfmaBN);
      Rt[jl * MCP + c] = rs[u];
    }
  };

  if (t_begin < t_end) load_tile(t_begin);
  for (int64_t t = t_begin; t < t_end; ++t) {
    __syncthreads();  // previous phase B finished reading Ks / Rt
    store_tile();
    __syncthreads();
    if (t + 1 < t_end) load_tile(t + 1);  // in flight during the math below

    // phase A: 16 kernel entries per thread
#pragma unroll 4
    for (int jj = 0; jj < 16; ++jj) {
      const int j = ahalf * 16 + jj;
      const float *xc = Xc + j * DP;
      float dot = 0.0f;
#pragma unroll
      for (int k = 0; k < DP; ++k) dot = fmaf(rc[k], xc[k], dot);
      float sq = fmaf(-2.0f, dot, rn + Cn[j]);
      if (rid == Cid[j]) sq = 0.0f;
      Ks[j][arow] = kernel_value<FAM>(sq);
    }
    __syncthreads();

    // phase B: acc += Ks^T (rows) x Rt (columns)
#pragma unroll 8
    for (int j = 0; j < kFfmaBN; ++j) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&Ks[j][tr * 8]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&Ks[j][tr * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[MT];
#pragma unroll
      for (int k = 0; k < MT; ++k) bv[k] = Rt[j * MCP + tc + 16 * k];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k < MT; ++k) acc[r][k] = fmaf(av[r], bv[k], acc[r][k]);
    }
  }

  // epilogue: direct (splits == 1) or partial into the workspace
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t i = row0 + tr * 8 + r;
    if (i >= p.b) continue;
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      const int c = tc + 16 * k;
      if (c >= p.m) continue;
      if (p.splits == 1) {
        float *o = p.out + i * p.ldo + p.c0 + c;
        const float v = p.variance * acc[r][k];
        *o = p.accumulate ? *o + v : v;
      } else {
        p.out[(int64_t(split) * p.b + i) * p.m + c] = acc[r][k];
      }
    }
  }
}

}  // namespace sap
