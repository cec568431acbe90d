// Fused, batched power-iteration stepsize (reference randnla.py:165-196,
// rand_power_stepsize, as called from solvers.py:389-396):
//
//   H = P^{-1/2} (K_BB + lam I) P^{-1/2},  P^{-1/2} x = x/sqrt(rho) + U diag(E) U^T x,
//   E = (S + rho)^{-1/2} - rho^{-1/2},
//   v <- v0;  10 x { y = H v;  est = v.y;  v = y/||y|| };  eta = 1/est.
//
// One thread-block cluster of C CTAs per batch element (one ADASAP
// iteration of a lookahead batch). CTA c of the cluster owns rows [lo, hi) of
// K_BB (fp32, the values the tile kernel computes) and of U (fp64); the
// length-b vector w = P^{-1/2} v is replicated in every CTA's shared memory
// by DSMEM broadcast, and the two reductions of a step (U^T z and the two
// scalars v.y = w.z, |y|^2 = z.P^{-1} z) combine per-CTA partials read over
// DSMEM in a fixed rank order, so every CTA holds bitwise-identical results
// (the loop runs on w, see the kernel; the iterates are the reference's). K_BB is
// streamed once per step (b^2 * 4 bytes): the kernel is bound by L2/HBM
// bandwidth, replacing ~12 batched cuBLAS/elementwise launches per step.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/sapgp_b200.h"

namespace cg = cooperative_groups;

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace pw {

// Cluster size per launch (4, 8 or 16 CTAs per batch element): the batch's
// clusters fill the GPU in ONE wave where they can -- 32 iterations as
// clusters of 4 (128 CTAs) ran in 1.22 ms against 1.56 ms as 3.5 waves of
// clusters of 16 -- and a small batch (the ramp's first, whose stepsize the
// first step waits for) keeps 16 CTAs per iteration for latency.
// SAP_POWER_CLUSTER forces one size (16 is a non-portable cluster size,
// which B200 supports).
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerPass = 4;  // rows a warp dots at once (amortises w reads)

struct Args {
  const float *K;      // [count][b][ldk]
  int64_t ldk, strideK;
  const double *U;     // [count][b][r] (row-major) or null when r == 0
  int64_t strideU;
  const double *E;     // [count][r]
  const double *rho;   // [count]
  const double *v0;    // [count][b], unit norm
  int b, r, iters;
  double lam;
  double *eta;         // [count]
  int *bad;            // [count], OR-ed
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of two values; result valid in every thread
__device__ __forceinline__ void block_sum2(double &a, double &c, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  c = warp_sum(c);
  __syncthreads();
  if (lane == 0) {
    red[2 * warp] = a;
    red[2 * warp + 1] = c;
  }
  __syncthreads();
  a = 0.0;
  c = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    a += red[2 * w];
    c += red[2 * w + 1];
  }
}

// rows per CTA (a multiple of 4 with the symmetric sweep: its column blocks
// start on 16-byte boundaries)
__host__ __device__ inline int row_block(int b, int C, int sym) {
  const int per = (b + C - 1) / C;
  return sym ? (per + 3) & ~3 : per;
}
constexpr int kSymCols = 512;  // columns of one sub-range of the symmetric sweep

template <int kCluster>
__global__ void __launch_bounds__(kThreads, 1) power_kernel(const Args a, const int u_smem,
                                                           const int sym) {
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  const int q = blockIdx.x / kCluster;  // batch element
  const int b = a.b, r = a.r;
  const int per = row_block(b, kCluster, sym);
  const int lo = min(b, int(crank) * per), hi = min(b, lo + per);
  const int nloc = hi - lo;
  const int b4 = (b + 3) & ~3;

  extern __shared__ __align__(16) double sm[];
  double *vloc = sm;                  // [per]   v on own rows
  double *zloc = vloc + per;          // [per]   w, then z, then y on own rows
  double *part = zloc + per;          // [r]     own partial of U^T x
  double *coef = part + r;            // [r]     E * (U^T x), full
  double *spart = coef + r;           // [2]     own partial of v.y, |y|^2
  double *red = spart + 2;            // [2*kWarps] block reduction scratch
  double *scratch = red + 2 * kWarps; // [2*kThreads]
  float *wf = reinterpret_cast<float *>(scratch + 2 * kThreads);  // [b4] replicated w (fp32)
  // symmetric sweep only: own rows' direct sums, transposed contributions to
  // every column (read by the owners over DSMEM), per-warp column partials
  double *zdir = reinterpret_cast<double *>(wf + b4);         // [per]
  double *tpart = zdir + (sym ? per : 0);                     // [b4]
  float *tw = reinterpret_cast<float *>(tpart + (sym ? b4 : 0));  // [kWarps][kSymCols]
  double *us = reinterpret_cast<double *>(tw + (sym ? kWarps * kSymCols : 0));  // [nloc][r] own U rows (opt.)

  const float *K = a.K + int64_t(q) * a.strideK;
  const double *Ug = r ? a.U + int64_t(q) * a.strideU + int64_t(lo) * r : nullptr;
  const double *E = r ? a.E + int64_t(q) * r : nullptr;
  const double rho = a.rho[q];
  const double isr = 1.0 / sqrt(rho);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool vec4 = (a.ldk & 3) == 0 && (a.strideK & 3) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.K) & 15) == 0;
  // own rows of U, from shared memory when they fit (loaded once)
  const double *U = Ug;
  if (u_smem && r) {
    for (int e = tid; e < nloc * r; e += kThreads) us[e] = Ug[e];
    U = us;
  }
  for (int i = tid; i < nloc; i += kThreads) vloc[i] = a.v0[int64_t(q) * b + lo + i];
  for (int j = b + tid; j < b4; j += kThreads) wf[j] = 0.0f;
  __syncthreads();

  // coef = E * (U^T x) over the cluster, x given on own rows
  // (or F * (U^T x), F = 1/(S+rho) - 1/rho = E (E + 2/sqrt(rho)), with pinv)
  const bool u_vec2 = (r & 1) == 0 && r / 2 <= kThreads &&
                      (reinterpret_cast<uintptr_t>(U) & 15) == 0;
  auto ut_times = [&](const double *x, bool pinv) {
    if (u_vec2) {
      // column pairs (16-byte loads), kThreads / (r/2) row groups, two rows per
      // trip with their own running sums: four independent fp64 chains and
      // eight loads in flight per thread (the one-column form was latency-bound
      // on L2 at ~23 B/clk per SM); groups combined in a fixed order
      const int r2 = r >> 1, G = kThreads / r2, g = tid / r2, k2 = tid % r2;
      double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
      if (g < G) {
        const double2 *U2 = reinterpret_cast<const double2 *>(U);
        int i = g;
#pragma unroll 4
        for (; i + G < nloc; i += 2 * G) {
          const double2 ua = U2[i * r2 + k2], uc = U2[(i + G) * r2 + k2];
          const double xa = x[i], xc = x[i + G];
          s0 = fma(ua.x, xa, s0);
          s1 = fma(ua.y, xa, s1);
          t0 = fma(uc.x, xc, t0);
          t1 = fma(uc.y, xc, t1);
        }
        if (i < nloc) {
          const double2 ua = U2[i * r2 + k2];
          s0 = fma(ua.x, x[i], s0);
          s1 = fma(ua.y, x[i], s1);
        }
      }
      scratch[2 * tid] = s0 + t0;
      scratch[2 * tid + 1] = s1 + t1;
      __syncthreads();
      if (tid < r) {
        double t = 0.0;
        for (int gg = 0; gg < G; ++gg) t += scratch[2 * (gg * r2 + (tid >> 1)) + (tid & 1)];
        part[tid] = t;
      }
    } else if (r <= kThreads) {
      // kThreads / r row groups per column, combined in a fixed order
      const int G = kThreads / r, g = tid / r, k = tid % r;
      double s = 0.0;
      if (g < G) {
#pragma unroll 4
        for (int i = g; i < nloc; i += G) s = fma(U[i * r + k], x[i], s);
      }
      scratch[tid] = s;
      __syncthreads();
      if (tid < r) {
        double t = 0.0;
        for (int gg = 0; gg < G; ++gg) t += scratch[gg * r + tid];
        part[tid] = t;
      }
    } else {
      for (int k = tid; k < r; k += kThreads) {
        double t = 0.0;
        for (int i = 0; i < nloc; ++i) t = fma(U[i * r + k], x[i], t);
        part[k] = t;
      }
    }
    cluster.sync();
    for (int k = tid; k < r; k += kThreads) {
      double v[kCluster];
#pragma unroll
      for (int c = 0; c < kCluster; ++c) v[c] = cluster.map_shared_rank(part, c)[k];
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < kCluster; ++c) s += v[c];
      coef[k] = (pinv ? E[k] * fma(2.0, isr, E[k]) : E[k]) * s;
    }
    __syncthreads();
  };
  // out_i = x_i / sqrt(rho) + U[i,:] . coef on own rows: each thread owns rows
  // tid, tid + kThreads, ... (U rows from shared memory; a thread's dot is
  // sequential in k, the same order for every row)
  // U[i,:] . coef with kSplit threads per row (adjacent lanes, each a
  // contiguous quarter of k, combined by a fixed shuffle tree): four times
  // shorter fp64 dependency chains than one thread per row
  constexpr int kSplit = 4;
  const int kq = (r + kSplit - 1) / kSplit, part_id = tid % kSplit;
  auto row_dot = [&](int i) {
    double s = 0.0;
    if (i < nloc && u_vec2) {
      // the kSplit lanes of a row take interleaved column pairs: 64
      // contiguous bytes per row and load, two running sums per lane
      const double2 *u2 = reinterpret_cast<const double2 *>(U + i * r);
      const double2 *c2 = reinterpret_cast<const double2 *>(coef);
      double sa = 0.0, sb = 0.0;
#pragma unroll 4
      for (int k2 = part_id; k2 < (r >> 1); k2 += kSplit) {
        const double2 u = u2[k2], c = c2[k2];
        sa = fma(u.x, c.x, sa);
        sb = fma(u.y, c.y, sb);
      }
      s = sa + sb;
    } else if (i < nloc) {
      const double *ur = U + i * r;
      const int k1 = min(r, (part_id + 1) * kq);
      for (int k = part_id * kq; k < k1; ++k) s = fma(ur[k], coef[k], s);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    return s;
  };
  auto apply_u = [&](const double *x, double *out) {
    for (int i0 = 0; i0 < nloc; i0 += kThreads / kSplit) {
      const int i = i0 + tid / kSplit;
      const double s = r ? row_dot(i) : 0.0;
      if (part_id == 0 && i < nloc) out[i] = fma(x[i], isr, s);
    }
    __syncthreads();
  };

  double est = 0.0;
  bool bad = false;
#ifdef SAP_POWER_PROF
  unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tc0 = clock64(), tc1;
#define PP(k) do { tc1 = clock64(); tp[k] += tc1 - tc0; tc0 = tc1; } while (0)
#else
#define PP(k) do {} while (0)
#endif
  // Symmetric sweep (K_BB is exactly symmetric): the b x b matrix as C x C
  // blocks of the CTAs' row ranges. CTA c reads, in its own rows, the
  // diagonal block (c, c), the blocks (c, c+k) for k = 1 .. C/2-1, and half of
  // (c, c+C/2) (c < C/2: its columns' first half; c >= C/2: its own rows'
  // second half against all of block c-C/2's columns), and adds each
  // off-diagonal block's transpose times its own w to the other rows: every
  // entry of K_BB is read once per step instead of the full matrix, 2.5 of 4
  // blocks at C = 4 (the sweep is HBM-bound). Direct sums per row in zdir,
  // transposed ones per column in tpart, combined in a fixed rank order.
  auto rect = [&](int r0, int r1, int j0, int j1, bool tr) {
    // empty: no rows, or a column block past b (clamped starts are not
    // 16-byte aligned); uniform over the CTA
    if (r1 <= r0 || j1 <= j0) return;
    const int J1 = min(b4, (j1 + 3) & ~3);
    for (int s0 = j0; s0 < J1; s0 += kSymCols) {
      const int s1 = min(J1, s0 + kSymCols);
      float tacc[kSymCols / 128][4];
#pragma unroll
      for (int c = 0; c < kSymCols / 128; ++c)
#pragma unroll
        for (int u = 0; u < 4; ++u) tacc[c][u] = 0.0f;
      for (int i0 = r0 + warp * kRowsPerPass; i0 < r1; i0 += kWarps * kRowsPerPass) {
        const float *krow[kRowsPerPass];
        float wr[kRowsPerPass], acc[kRowsPerPass];
#pragma unroll
        for (int rr = 0; rr < kRowsPerPass; ++rr) {
          const int i = min(i0 + rr, r1 - 1);  // clamped rows: weight 0, sums discarded
          krow[rr] = K + int64_t(lo + i) * a.ldk;
          wr[rr] = i0 + rr < r1 ? wf[lo + i0 + rr] : 0.0f;
          acc[rr] = 0.0f;
        }
        float4 kv[kSymCols / 128][kRowsPerPass];
#pragma unroll
        for (int c = 0; c < kSymCols / 128; ++c) {
          const int j = s0 + lane * 4 + 128 * c;
#pragma unroll
          for (int rr = 0; rr < kRowsPerPass; ++rr)
            kv[c][rr] = j < s1 ? __ldg(reinterpret_cast<const float4 *>(krow[rr] + j))
                               : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
#pragma unroll
        for (int c = 0; c < kSymCols / 128; ++c) {
          const int j = s0 + lane * 4 + 128 * c;
          if (j >= s1) break;
          const float4 w4 = *reinterpret_cast<const float4 *>(wf + j);
#pragma unroll
          for (int rr = 0; rr < kRowsPerPass; ++rr) {
            acc[rr] = fmaf(kv[c][rr].x, w4.x, acc[rr]);
            acc[rr] = fmaf(kv[c][rr].y, w4.y, acc[rr]);
            acc[rr] = fmaf(kv[c][rr].z, w4.z, acc[rr]);
            acc[rr] = fmaf(kv[c][rr].w, w4.w, acc[rr]);
            if (tr) {
              tacc[c][0] = fmaf(kv[c][rr].x, wr[rr], tacc[c][0]);
              tacc[c][1] = fmaf(kv[c][rr].y, wr[rr], tacc[c][1]);
              tacc[c][2] = fmaf(kv[c][rr].z, wr[rr], tacc[c][2]);
              tacc[c][3] = fmaf(kv[c][rr].w, wr[rr], tacc[c][3]);
            }
          }
        }
#pragma unroll
        for (int rr = 0; rr < kRowsPerPass; ++rr) {
          const double sd = warp_sum(double(acc[rr]));
          if (lane == 0 && i0 + rr < r1) zdir[i0 + rr] += sd;
        }
      }
      if (tr) {
#pragma unroll
        for (int c = 0; c < kSymCols / 128; ++c)
#pragma unroll
          for (int u = 0; u < 4; ++u) tw[warp * kSymCols + lane * 4 + 128 * c + u] = tacc[c][u];
        __syncthreads();
        for (int jj = tid; jj < s1 - s0; jj += kThreads) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) t += double(tw[w * kSymCols + jj]);
          tpart[s0 + jj] += t;
        }
      }
      __syncthreads();  // zdir rows / tw reused by the next sub-range or rectangle
    }
  };
  auto blk_lo = [&](int cc) { return min(b, cc * per); };
  auto blk_hi = [&](int cc) { return min(b, cc * per + per); };
  auto blk_half = [&](int cc) {
    const int nn = blk_hi(cc) - blk_lo(cc);
    return min(nn, ((nn >> 1) + 3) & ~3);
  };
  auto sym_sweep = [&]() {
    for (int i = tid; i < nloc; i += kThreads) zdir[i] = 0.0;
    for (int j = tid; j < b4; j += kThreads) tpart[j] = 0.0;
    __syncthreads();
    const int c = int(crank);
    rect(0, nloc, lo, hi, false);
    for (int k = 1; k < kCluster / 2; ++k) {
      const int cp = (c + k) % kCluster;
      rect(0, nloc, blk_lo(cp), blk_hi(cp), true);
    }
    const int cp = (c + kCluster / 2) % kCluster;
    if (c < kCluster / 2) rect(0, nloc, blk_lo(cp), blk_lo(cp) + blk_half(cp), true);
    else rect(blk_half(c), nloc, blk_lo(cp), blk_hi(cp), true);
    cluster.sync();  // every CTA's tpart complete
    for (int i = tid; i < nloc; i += kThreads) {
      double t = 0.0;
      for (int cc = 0; cc < kCluster; ++cc) t += cluster.map_shared_rank(tpart, cc)[lo + i];
      zloc[i] = fma(a.lam, zloc[i], zdir[i] + t);
    }
    __syncthreads();
    // peers read this tpart before they reach the step's next cluster barrier
    // (U^T z's, or the scalars' when r = 0), which every CTA passes before it
    // zeroes its tpart for the next step
  };

  // The iteration runs on w = P^{-1/2} v rather than on v (the same iterates,
  // Rayleigh quotients and norms, reassociated):
  //   z = (K + lam I) w,  est = v.y = w.z,  |y|^2 = z.P^{-1} z = z.u,
  //   u = P^{-1} z = z/rho + U diag(F) U^T z,  w <- u/|y|,
  // two passes over the CTA's U rows per step instead of four (U^T v, U coef,
  // U^T z, U coef) and one cluster barrier fewer; w_0 = P^{-1/2} v_0 once.
  const double irho = 1.0 / rho;
  auto broadcast_w = [&]() {  // own rows of w (vloc) -> every CTA's wf, fp32
    for (int c = 0; c < kCluster; ++c) {
      float *dst = cluster.map_shared_rank(wf, c);
      for (int i = tid; i < nloc; i += kThreads) dst[lo + i] = float(vloc[i]);
    }
    cluster.sync();
  };
  if (r) ut_times(vloc, false);
  apply_u(vloc, zloc);
  for (int i = tid; i < nloc; i += kThreads) vloc[i] = zloc[i];
  __syncthreads();
  broadcast_w();
  PP(0);
  // vloc and zloc hold w on own rows at the top of a step
  for (int it = 0; it < a.iters; ++it) {
    if (sym) {
      sym_sweep();
    } else {
    // z = K w + lam w on own rows: a warp dots kRowsPerPass rows at once, fp32
    // products summed per lane (64 terms for b = 2000), lanes combined in fp64
    for (int i0 = warp * kRowsPerPass; i0 < nloc; i0 += kWarps * kRowsPerPass) {
      float acc[kRowsPerPass];
#pragma unroll
      for (int rr = 0; rr < kRowsPerPass; ++rr) acc[rr] = 0.0f;
      if (vec4) {
        // kChunks 128-column chunks of the kRowsPerPass rows are loaded
        // before any is used: 16 x 16-byte loads in flight per lane (the
        // compiler otherwise interleaved load and use, leaving the loop
        // latency-bound on HBM at ~9 B/clk per SM)
        constexpr int kChunks = 4;
        const float *krow[kRowsPerPass];
#pragma unroll
        for (int rr = 0; rr < kRowsPerPass; ++rr)
          krow[rr] = K + int64_t(lo + min(i0 + rr, nloc - 1)) * a.ldk;  // clamped rows discarded below
        for (int j0 = lane * 4; j0 < b4; j0 += 128 * kChunks) {
          float4 kv[kChunks][kRowsPerPass];
#pragma unroll
          for (int c = 0; c < kChunks; ++c) {
            const int j = j0 + 128 * c;
#pragma unroll
            for (int rr = 0; rr < kRowsPerPass; ++rr)
              kv[c][rr] = j < b4 ? __ldg(reinterpret_cast<const float4 *>(krow[rr] + j))
                                 : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          }
#pragma unroll
          for (int c = 0; c < kChunks; ++c) {
            const int j = j0 + 128 * c;
            if (j >= b4) break;
            const float4 w4 = *reinterpret_cast<const float4 *>(wf + j);
#pragma unroll
            for (int rr = 0; rr < kRowsPerPass; ++rr) {
              acc[rr] = fmaf(kv[c][rr].x, w4.x, acc[rr]);
              acc[rr] = fmaf(kv[c][rr].y, w4.y, acc[rr]);
              acc[rr] = fmaf(kv[c][rr].z, w4.z, acc[rr]);
              acc[rr] = fmaf(kv[c][rr].w, w4.w, acc[rr]);
            }
          }
        }
      } else {
        for (int j = lane; j < b; j += 32) {
#pragma unroll
          for (int rr = 0; rr < kRowsPerPass; ++rr) {
            const int i = min(i0 + rr, nloc - 1);
            acc[rr] = fmaf(K[int64_t(lo + i) * a.ldk + j], wf[j], acc[rr]);
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < kRowsPerPass; ++rr) {
        const double s = warp_sum(double(acc[rr]));
        const int i = i0 + rr;
        if (lane == 0 && i < nloc) zloc[i] = fma(a.lam, zloc[i], s);
      }
    }
    __syncthreads();
    }
    PP(3);
    // u = P^{-1} z on own rows, the partials of w.z and z.u
    if (r) ut_times(zloc, true);
    PP(4);
    double dvy = 0.0, dyy = 0.0;
    for (int i0 = 0; i0 < nloc; i0 += kThreads / kSplit) {
      const int i = i0 + tid / kSplit;
      const double s = r ? row_dot(i) : 0.0;
      if (part_id == 0 && i < nloc) {
        const double z = zloc[i];
        const double u = fma(z, irho, s);
        dvy = fma(vloc[i], z, dvy);
        dyy = fma(z, u, dyy);
        zloc[i] = u;
      }
    }
    PP(5);
    block_sum2(dvy, dyy, red);
    if (tid == 0) {
      spart[0] = dvy;
      spart[1] = dyy;
    }
    cluster.sync();
    double sv[2 * kCluster];
#pragma unroll
    for (int c = 0; c < kCluster; ++c) {
      const double *sp = cluster.map_shared_rank(spart, c);
      sv[2 * c] = sp[0];
      sv[2 * c + 1] = sp[1];
    }
    double vy = 0.0, yy = 0.0;
#pragma unroll
    for (int c = 0; c < kCluster; ++c) {
      vy += sv[2 * c];
      yy += sv[2 * c + 1];
    }
    est = vy;
    bad = bad || !(yy > 0.0);  // |y| = 0 (z = 0); a rounding-negative z.P^{-1}z alike
    const double inv = yy > 0.0 ? 1.0 / sqrt(yy) : 0.0;
    for (int i = tid; i < nloc; i += kThreads) {
      const double w = zloc[i] * inv;
      vloc[i] = w;
      zloc[i] = w;
    }
    __syncthreads();
    PP(6);
    // every CTA has finished this step's sweep (reading its wf) and its reads
    // of the peers' part before the scalar barrier above, and reads the
    // peers' spart before the broadcast's barrier: no peer data is overwritten
    // while still needed
    if (it + 1 < a.iters) broadcast_w();
    PP(2);
  }
#ifdef SAP_POWER_PROF
  if (blockIdx.x == 0 && tid == 0)
    printf("power prof (cycles): w0 %llu bcast+sync %llu gemv %llu ut_z %llu u %llu "
           "red+sync %llu\n", tp[0], tp[2], tp[3], tp[4], tp[5], tp[6]);
#endif
  bad = bad || !(est > 0.0);
  if (crank == 0 && tid == 0) {
    a.eta[q] = 1.0 / est;
    if (bad) a.bad[q] |= 1;
  }
  cluster.sync();  // no CTA exits while a peer may still read its shared memory
}

}  // namespace pw
}  // namespace sap

extern "C" int sap_power_stepsize(const float *Kbb, int64_t ldk, int64_t strideK,
                                  const double *U, int64_t strideU, int r, const double *E,
                                  const double *rho, const double *v0, int b, int count,
                                  double lam, int iters, double *eta, int *bad, void *stream) {
  using namespace sap;
  if (b <= 0 || count <= 0 || iters <= 0 || r < 0 || ldk < b || (r && (!U || !E)))
    return fail(SAP_ERR_CONTRACT, "power_stepsize: bad shape b=%d r=%d count=%d", b, r, count);
  int C = 16;
  if (const char *e = getenv("SAP_POWER_CLUSTER")) {
    C = atoi(e);
  } else {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
        sms = 148;
    }
    while (C > 4 && count * C > sms) C /= 2;  // one wave if clusters of >= 4 allow it
  }
  if (C != 4 && C != 8 && C != 16)
    return fail(SAP_ERR_CONTRACT, "power_stepsize: cluster size %d (4, 8 or 16)", C);
  // the symmetric sweep (half of K_BB's bytes) needs 16-byte rows;
  // SAP_POWER_SYM=0/1 forces the full / the symmetric sweep
  const bool vec4 = (ldk & 3) == 0 && (strideK & 3) == 0 &&
                    (reinterpret_cast<uintptr_t>(Kbb) & 15) == 0;
  // (blocks of >= 384 rows: with C = 16 at b = 2000 the many small
  // rectangles made it 2x slower, 1.07 vs 0.49 ms for 8 iterations; at C = 4
  // 0.755 vs 0.895 ms for 32)
  const char *se = getenv("SAP_POWER_SYM");
  const size_t b4 = size_t((b + 3) & ~3);
  auto smem_base = [&](int sy) {
    const size_t pr = size_t(pw::row_block(b, C, sy));
    return sizeof(double) * (2 * pr + 2 * size_t(r) + 2 + 2 * pw::kWarps + 2 * pw::kThreads) +
           sizeof(float) * b4 +
           (sy ? sizeof(double) * (pr + b4) + sizeof(float) * size_t(pw::kWarps) * pw::kSymCols
               : 0);
  };
  constexpr size_t kCap = 200 * 1024;
  // the symmetric sweep's extra shared memory (~b x 8 bytes more) must fit
  // too: at b = 10 000 (config 5) it does not, and the full sweep runs
  const int sym = (vec4 && ((se && *se) ? atoi(se) != 0 : (b + C - 1) / C >= 384) &&
                   smem_base(1) <= kCap) ? 1 : 0;
  const int per = pw::row_block(b, C, sym);
  const size_t base = smem_base(sym);
  const size_t with_u = base + sizeof(double) * size_t(per) * size_t(r);
  if (base > kCap) return fail(SAP_ERR_CONTRACT, "power_stepsize: b=%d exceeds shared memory", b);
  const int u_smem = with_u <= kCap ? 1 : 0;
  const size_t smem = u_smem ? with_u : base;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pw::power_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCap));
    cudaFuncSetAttribute(pw::power_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCap));
    cudaFuncSetAttribute(pw::power_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCap));
    cudaFuncSetAttribute(pw::power_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  pw::Args a{Kbb, ldk, strideK, U, strideU, E, rho, v0, b, r, iters, lam, eta, bad};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(count * C));
  cfg.blockDim = dim3(pw::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(C);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = C == 4 ? cudaLaunchKernelEx(&cfg, pw::power_kernel<4>, a, u_smem, sym)
                        : C == 8 ? cudaLaunchKernelEx(&cfg, pw::power_kernel<8>, a, u_smem, sym)
                                 : cudaLaunchKernelEx(&cfg, pw::power_kernel<16>, a, u_smem, sym);
  if (e != cudaSuccess) return fail(SAP_ERR_DEVICE, "power_kernel: %s", cudaGetErrorString(e));
  return check_launch("power_kernel");
}
