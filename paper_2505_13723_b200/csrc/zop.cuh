// The tensor-core product's right-hand-side operand: Z = zp*P + zq*Q (the
// lazy Nesterov pair) scaled per column by a power of two and
// split into fp16 hi/lo, stored [nz][ldz] (RHS column c's points contiguous).
// Shared by the stand-alone pass (sap_z_operand), the block-row kernel's
// overlapped next-iterate pass (krows_tc2.cuh) and the fused Phase IV kernel's
// block-row patch and fallback pass (phase4.cu), so all three write
// bit-identical operands.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace sap {
namespace zop {

// scale_c = 2^floor(log2(1024 / bound_c)) from per-column magnitude bounds:
// the column's largest value maps into [512, 1024], 64x below fp16's maximum,
// so an operand whose scale was fixed before an update stays finite unless a
// column grows 64x in one iteration. The headroom costs no precision that
// matters: hi/lo keep 22 significant bits down to lo's subnormal floor of
// 2^-24, i.e. 2^-34 of the column's largest value.
// Rows c >= m (MMA padding) are not touched: the caller zeroes them once.
__device__ __forceinline__ float scale(float zp, float zq, const float *Pb, const float *Qb,
                                       bool hasq, int c) {
  const float bound = fabsf(zp) * Pb[c] + (hasq ? fabsf(zq) * Qb[c] : 0.0f);
  float sc = 1.0f;
  if (bound > 0.0f && isfinite(bound)) sc = exp2f(floorf(log2f(1024.0f / bound)));
  return fminf(fmaxf(sc, 0x1p-100f), 0x1p100f);
}

__device__ __forceinline__ void split(float z, __half &h, __half &l) {
  h = __float2half_rn(z);
  l = __float2half_rn(z - __half2float(h));
}

// a scaled value whose hi part would not be finite (the bounds the scale was
// chosen from were exceeded): the operand must be rebuilt with a new scale
__device__ __forceinline__ bool overflows(float zs) { return !(fabsf(zs) < 65000.0f); }

// Eight consecutive points j..j+7 of column c: z = a*P + bq*Q (a = zp*scale,
// bq = zq*scale), rows from n up to ldz zero; 16-byte loads.
template <bool kStream>
__device__ __forceinline__ void load8(const float *pr, const float *qr, int64_t j, int64_t n,
                                      float a, float bq, float (&z)[8]) {
  if (j + 8 <= n) {
    float4 p0, p1;
    if constexpr (kStream) {
      p0 = __ldcs(reinterpret_cast<const float4 *>(pr + j));
      p1 = __ldcs(reinterpret_cast<const float4 *>(pr + j + 4));
    } else {
      p0 = *reinterpret_cast<const float4 *>(pr + j);
      p1 = *reinterpret_cast<const float4 *>(pr + j + 4);
    }
    z[0] = a * p0.x; z[1] = a * p0.y; z[2] = a * p0.z; z[3] = a * p0.w;
    z[4] = a * p1.x; z[5] = a * p1.y; z[6] = a * p1.z; z[7] = a * p1.w;
    if (qr) {
      float4 q0, q1;
      if constexpr (kStream) {
        q0 = __ldcs(reinterpret_cast<const float4 *>(qr + j));
        q1 = __ldcs(reinterpret_cast<const float4 *>(qr + j + 4));
      } else {
        q0 = *reinterpret_cast<const float4 *>(qr + j);
        q1 = *reinterpret_cast<const float4 *>(qr + j + 4);
      }
      z[0] = fmaf(bq, q0.x, z[0]); z[1] = fmaf(bq, q0.y, z[1]);
      z[2] = fmaf(bq, q0.z, z[2]); z[3] = fmaf(bq, q0.w, z[3]);
      z[4] = fmaf(bq, q1.x, z[4]); z[5] = fmaf(bq, q1.y, z[5]);
      z[6] = fmaf(bq, q1.z, z[6]); z[7] = fmaf(bq, q1.w, z[7]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t jj = j + e;
      z[e] = jj < n ? (qr ? fmaf(bq, qr[jj], a * pr[jj]) : a * pr[jj]) : 0.0f;
    }
  }
}

// fp16 hi/lo split of eight values, one 16-byte store to each half
template <bool kStream>
__device__ __forceinline__ void store8(const float (&z)[8], __half *hr, __half *lr, int64_t j) {
  __align__(16) __half h[8], l[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) split(z[e], h[e], l[e]);
  if constexpr (kStream) {
    __stcs(reinterpret_cast<uint4 *>(hr + j), *reinterpret_cast<const uint4 *>(h));
    __stcs(reinterpret_cast<uint4 *>(lr + j), *reinterpret_cast<const uint4 *>(l));
  } else {
    *reinterpret_cast<uint4 *>(hr + j) = *reinterpret_cast<const uint4 *>(h);
    *reinterpret_cast<uint4 *>(lr + j) = *reinterpret_cast<const uint4 *>(l);
  }
}

// The operand of the next iterate, Z_{t+1} = zp*P + zq*Q, written into a
// second buffer while the current one is being consumed (block-row kernel
// side job; the Phase IV kernel patches the block rows afterwards).
struct Next {
  const float *P, *Q;   // lazy state, column-major m x ldp (Q may be NULL)
  int64_t ldp, n;       // n = points of this shard
  int m;
  float zp, zq;         // coefficients of Z_{t+1}
  const float *Pb, *Qb; // per-column magnitude bounds of P and Q
  __half *Zhi, *Zlo;    // [nz][ldz] next-iterate buffer (NULL: no side job)
  int64_t ldz;
  float *zscale;        // [nz] scales of the next-iterate buffer
};

// Part `part` of `parts` of the whole pass, with `nthr` cooperating threads
// (thread `tid`): contiguous point ranges per part so the loads stream. Short
// columns per part (config 2: ~84 8-point groups) make the part's (column,
// group) items one flat index space, groups fastest, two items in flight per
// thread (the control warps hold 64 registers): a column-at-a-time loop left
// the pass latency-bound there and longer than the block-row product it hides
// under (config 2: 3860 -> 4470 iterations/s).
__device__ __forceinline__ void next_pass(const Next &zn, int part, int parts, int tid, int nthr) {
  const int64_t groups = zn.ldz / 8;
  const int64_t g0 = groups * part / parts, g1 = groups * (part + 1) / parts;
  const unsigned ng = unsigned(g1 - g0);
  const bool hasq = zn.Q != nullptr;
  if (part == 0)
    for (int c = tid; c < zn.m; c += nthr) zn.zscale[c] = scale(zn.zp, zn.zq, zn.Pb, zn.Qb, hasq, c);
  if (ng == 0) return;
  if (ng >= 4u * unsigned(nthr)) {
    // long columns (config 3: ~845 groups per part): column at a time, which
    // measured faster there than the flat loop below (its index arithmetic
    // and deeper memory pressure cost the RBF block product 11%)
    for (int c = 0; c < zn.m; ++c) {
      const float sc = scale(zn.zp, zn.zq, zn.Pb, zn.Qb, hasq, c);
      const float ca = zn.zp * sc, cb = zn.zq * sc;
      const float *pr = zn.P + int64_t(c) * zn.ldp;
      const float *qr = hasq ? zn.Q + int64_t(c) * zn.ldp : nullptr;
      __half *hr = zn.Zhi + int64_t(c) * zn.ldz, *lr = zn.Zlo + int64_t(c) * zn.ldz;
      int64_t g = g0 + tid;
      for (; g + nthr < g1; g += 2 * nthr) {  // two groups per step: 64 B of loads in flight
        float z0[8], z1[8];
        load8<true>(pr, qr, g * 8, zn.n, ca, cb, z0);
        load8<true>(pr, qr, (g + nthr) * 8, zn.n, ca, cb, z1);
        store8<true>(z0, hr, lr, g * 8);
        store8<true>(z1, hr, lr, (g + nthr) * 8);
      }
      if (g < g1) {
        float z0[8];
        load8<true>(pr, qr, g * 8, zn.n, ca, cb, z0);
        store8<true>(z0, hr, lr, g * 8);
      }
    }
    return;
  }
  const unsigned total = ng * unsigned(zn.m);
  constexpr int kD = 2;
  int cur = -1;
  float a = 0.0f, bq = 0.0f;
  for (unsigned base = unsigned(tid); base < total; base += kD * unsigned(nthr)) {
    float z[kD][8];
    int cc[kD];
    int64_t jj[kD];
#pragma unroll
    for (int u = 0; u < kD; ++u) {
      const unsigned it = base + unsigned(u * nthr);
      cc[u] = -1;
      if (it < total) {
        const int c = int(it / ng);
        if (c != cur) {
          const float sc = scale(zn.zp, zn.zq, zn.Pb, zn.Qb, hasq, c);
          a = zn.zp * sc;
          bq = zn.zq * sc;
          cur = c;
        }
        cc[u] = c;
        jj[u] = (g0 + int64_t(it - unsigned(c) * ng)) * 8;
        load8<true>(zn.P + int64_t(c) * zn.ldp, hasq ? zn.Q + int64_t(c) * zn.ldp : nullptr,
                    jj[u], zn.n, a, bq, z[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kD; ++u)
      if (cc[u] >= 0)
        store8<true>(z[u], zn.Zhi + int64_t(cc[u]) * zn.ldz, zn.Zlo + int64_t(cc[u]) * zn.ldz,
                     jj[u]);
  }
}

}  // namespace zop
}  // namespace sap
