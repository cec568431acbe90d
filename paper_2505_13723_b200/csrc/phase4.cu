// Phase IV of an ADASAP iteration (solvers.py:376-401) in three stream-ordered
// launches: the gradient gather, the Nystrom-Woodbury apply and
// the lazy Nesterov block update, plus the block rows of the next iterate's
// tensor-core operand.
//
//   A  g[i, c]  = sum_s part[s][c][i] * variance / (2^14 zscale_c)      (K[B,:] Z)
//               + lam * Z[B_i, c] - Y[B_i, c]                 solvers.py:376-377
//   -- launch --
//   B+C t       = U^T g, one 8 x 8 tile per CTA over all b rows (phase4_ut_kernel)
//               (SAP_P4_TPART=1: B as per-CTA partials T_k = U[rows_k]^T g[rows_k]
//               in stage A, C their fixed-order sum, phase4_reduce_kernel)
//   -- launch --
//   D  D[i, :]  = g[i, :] - (U Mc)[i, :] t          randnla.py:109-134 (1/rho rides
//                                                   on the stepsize eta/rho)
//      lazy update of the block rows (sap_pq_update's arithmetic),
//      Z_{t+1}[B] into the next operand buffer, overflow flag
//   E  if an updated block row left the next operand's scale: the last CTA of
//      D rebuilds it (rare: the scale leaves 64x headroom)
//
// The two small fp64 GEMMs (B: r x m x b, D: rows x m x r per CTA) run on
// the FP64 tensor cores (mma.sync m8n8k4 .f64) from shared-memory tiles laid
// out so every fragment load is bank-conflict free. Every reduction runs in a
// fixed order (no floating-point atomics): the result is bitwise
// reproducible, and the gradient equals the unfused chain (tc_reduce +
// sap_grad_gather) bit for bit.
//
// Stages are separate launches rather than one cooperative kernel with grid
// barriers: a cooperative grid must find every SM free at once, and behind
// the lookahead's high-priority side-stream kernels it waited tens of
// milliseconds (measured); separate launches interleave with them. The
// launches use programmatic dependent launch to hide most of the gaps.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "zop.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace p4 {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr float kPScale = 16384.0f;  // krows_tc.cuh: P = 2^14 k(S)
constexpr int kRB = 16;              // block rows per sub-chunk (two m8 tiles)
constexpr int kRSB = 20;             // row stride of the K = rows operands (= 4 mod 16)
constexpr int kKC = 128;             // r per K chunk of phase D
constexpr int kRSD = kKC + 4;        // row stride of the K = r operands (= 4 mod 16)

__device__ __forceinline__ int64_t dmin(int64_t x, int64_t y) { return x < y ? x : y; }

// D(8x8) += A(8x4, row) B(4x8, col) in fp64 on the tensor cores. Fragments
// (lane = 4 g + q): a = A[g][q], b = B[q][g], d0/d1 = D[g][2q], D[g][2q+1].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct Args {
  sap_step_args a;
  double *Tpart;   // [grid][r*m]
  double *t;       // [r*m]
  unsigned *done;  // [1] CTAs of stage 2 finished (zeroed; reset by the last one)
  int parts;      // partials T_k (stage 0's grid)
  int rows_per;    // block rows per CTA
  int do_grad, do_apply, has_next;
  int stage;       // 0: A (+B with tpart), 2: D (+E); C is phase4_ut_kernel or, with
                   // tpart, phase4_reduce_kernel
  int tpart;       // 1: B as per-CTA partials of stage 0 + C their sum (SAP_P4_TPART=1)
  int dbg;         // profiling: 5 skips B's product, 6 D's product, 7 the update,
                   // 8 the rebuild check (E), 9 the next operand's block rows
};

// Shared-memory carve-up (doubles unless noted); m8 = m rounded up to 8,
// r8 = r rounded up to 8.
//   gT [m8][kRSB]   gradient rows, transposed (B operand of phase B)
//   uT [r8][kRSB]   U rows, transposed (A operand of phase B)
//   v  [kRB][kRSD]  (U Mc) rows, one K chunk (A operand of phase D)
//   tT [m8][kRSD]   t, transposed, one K chunk (B operand of phase D)
//   bound (float) [2m], zs (float) [m]
inline size_t smem_bytes(int m, int r) {
  const size_t m8 = (m + 7) / 8 * 8, r8 = (std::max(r, 1) + 7) / 8 * 8;
  const size_t d = m8 * kRSB + r8 * kRSB + size_t(kRB) * kRSD + m8 * kRSD;
  return d * 8 + (3 * size_t(m) + 1) * 4;
}

// sum over the splits of one partial-sum element, eight running sums in a
// fixed order (bitwise the order of tc_reduce_kernel), loads issued 32 at a
// time so the L2 latency overlaps
__device__ __forceinline__ float reduce_splits(const float *pe, int splits, int64_t bm) {
  float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  int k = 0;
  for (; k + 32 <= splits; k += 32) {
    float x[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) x[u] = __ldcg(pe + int64_t(k + u) * bm);
#pragma unroll
    for (int u = 0; u < 32; ++u) acc[u & 7] += x[u];
  }
  for (; k + 8 <= splits; k += 8) {
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcg(pe + int64_t(k + u) * bm);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += x[u];
  }
  // the < 8 left over, into acc[0..]: static indices keep acc in registers
#pragma unroll
  for (int u = 0; u < 7; ++u)
    if (k + u < splits) acc[u] += __ldcg(pe + int64_t(k + u) * bm);
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) phase4_kernel(const Args A) {
  const sap_step_args &a = A.a;
  extern __shared__ __align__(16) double sm[];
  const int m = a.m, r = a.r;
  const int m8 = (m + 7) / 8 * 8, r8 = (r + 7) / 8 * 8;
  const int64_t b = a.b;
  const int rm = r * m;
  double *sgT = sm;
  double *suT = sgT + m8 * kRSB;
  double *sv = suT + (r > 0 ? r8 : 8) * kRSB;
  double *stT = sv + kRB * kRSD;
  float *sbound = reinterpret_cast<float *>(stT + m8 * kRSD);
  float *szs = sbound + 2 * m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fg = lane >> 2, fq = lane & 3;  // fragment row / column of this lane
  const int64_t i0 = dmin(b, int64_t(blockIdx.x) * A.rows_per);
  const int64_t i1 = dmin(b, i0 + A.rows_per);
  const int ntl = m8 / 8;
  const bool woodbury = A.do_apply && r > 0 && (A.stage != 0 || A.tpart);
  // stream order with the previous stage (programmatic dependent launch: this
  // grid was scheduled early, its inputs are complete after the wait); the
  // next stage may then be scheduled, to wait in turn
  pdl_wait();
  pdl_trigger();

  // gradient rows [c0, c0+nr) into sgT (zero padded to m8 x kRB)
  auto load_rows = [&](int64_t c0, int nr, bool grad) {
    for (int o = tid; o < m8 * kRB; o += kThreads) {
      const int c = o / kRB, ii = o % kRB;
      if (c >= m || ii >= nr) sgT[c * kRSB + ii] = 0.0;
    }
    if (grad) {
      // thread o -> (column c, row ii), rows fastest: coalesced partial loads
      for (int o = tid; o < nr * m; o += kThreads) {
        const int c = o / nr, ii = o % nr;
        const int64_t i = c0 + ii;
        // the row's local index and the partials are independent loads; the
        // lam Z - Y gathers follow the index
        const int64_t j = a.loc[i];
        float v;
        if (a.part) {
          const float s = reduce_splits(a.part + int64_t(c) * b + i, a.splits, b * m);
          v = s * (a.variance / (kPScale * a.zscale[c]));
        } else {
          v = a.G[i * a.ldg + c];
        }
        float pv = 0.0f, qv = 0.0f, yv = 0.0f;
        if (j >= 0) {
          const int64_t oo = int64_t(c) * a.ldp + j;
          pv = a.P[oo];
          if (a.Q) qv = a.Q[oo];
          yv = a.Y[oo];
        }
        double gv = double(v);
        if (j >= 0) {
          double z = a.zp * double(pv);
          if (a.Q) z += a.zq * double(qv);
          gv += a.lam * z - double(yv);
        }
        sgT[c * kRSB + ii] = gv;
        a.g[i * a.ldgo + c] = gv;
      }
    } else {
      for (int o = tid; o < nr * m; o += kThreads) {
        const int c = o / nr, ii = o % nr;
        sgT[c * kRSB + ii] = __ldcg(a.g + (c0 + ii) * a.ldgo + c);
      }
    }
  };

  if (A.stage == 0) {
    // ---------------- A + B: gradient rows, partial U^T g ----------------
    double *Tk = A.Tpart + int64_t(blockIdx.x) * rm;
    if (woodbury && i1 <= i0)
      for (int o = tid; o < rm; o += kThreads) Tk[o] = 0.0;
    for (int64_t c0 = i0; c0 < i1; c0 += kRB) {
      const int nr = int(dmin(kRB, i1 - c0));
      load_rows(c0, nr, A.do_grad);
      if (!woodbury) continue;
      for (int o0 = tid; o0 < r8 * kRB; o0 += 4 * kThreads) {  // U^T, zero padded
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = o0 + u * kThreads, jj = o % r8, ii = o / r8;
          x[u] = (o < r8 * kRB && jj < r && ii < nr) ? a.U[(c0 + ii) * a.ldu + jj] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = o0 + u * kThreads;
          if (o < r8 * kRB) suT[(o % r8) * kRSB + o / r8] = x[u];
        }
      }
      __syncthreads();
      if (A.dbg != 5) {
        // T_k (r x m) += U[rows]^T g[rows]: 8 x 8 tiles, K = kRB rows
        const bool first = c0 == i0;
        for (int tile = warp; tile < (r8 / 8) * ntl; tile += kWarps) {
          const int mt = tile / ntl, nt = tile % ntl;
          const int row = mt * 8 + fg, col = nt * 8 + 2 * fq;
          double d0 = 0.0, d1 = 0.0;
          if (!first) {
            if (row < r && col < m) d0 = Tk[row * m + col];
            if (row < r && col + 1 < m) d1 = Tk[row * m + col + 1];
          }
          const double *ua = suT + (mt * 8 + fg) * kRSB + fq;
          const double *gb = sgT + (nt * 8 + fg) * kRSB + fq;
#pragma unroll
          for (int ks = 0; ks < kRB / 4; ++ks) dmma(d0, d1, ua[4 * ks], gb[4 * ks]);
          if (row < r && col < m) Tk[row * m + col] = d0;
          if (row < r && col + 1 < m) Tk[row * m + col + 1] = d1;
        }
      }
      __syncthreads();
    }
    return;
  }

  // ---------------- D: D = g - UMc t, block update ----------------
  if (A.has_next && blockIdx.x == 0 && tid == 0) a.zflag[a.flag_idx ^ 1] = 0;
  const double eta = (a.Pw && a.eta_dev) ? a.eta_dev[0] : 0.0;
  const double dsc = a.dscale_dev ? 1.0 / a.dscale_dev[0] : 1.0;
  for (int c = tid; c < 2 * m; c += kThreads) sbound[c] = 0.0f;
  if (A.has_next && tid < m) szs[tid] = a.zscale_next[tid];
  const float zp1 = float(a.zp1), zq1 = float(a.zq1);
  bool over = false;
  const int ntiles = 2 * ntl;  // two 8-row tiles per kRB-row sub-chunk
  for (int64_t c0 = i0; c0 < i1; c0 += kRB) {
    const int nr = int(dmin(kRB, i1 - c0));
    __syncthreads();
    load_rows(c0, nr, false);
    // this warp's (up to two) 8 x 8 output tiles, accumulated over K chunks of r
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (woodbury && A.dbg != 6) {
      for (int k0 = 0; k0 < r; k0 += kKC) {
        const int kc = int(dmin(kKC, r - k0)), kc4 = (kc + 3) / 4 * 4;
        if (k0 > 0) __syncthreads();
        // (U Mc) rows and t^T of this K chunk, zero padded; loads issued eight
        // at a time per thread so their latencies overlap
        for (int o0 = tid; o0 < kRB * kc4; o0 += 8 * kThreads) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int o = o0 + u * kThreads, ii = o / kc4, jj = o % kc4;
            x[u] = (o < kRB * kc4 && ii < nr && jj < kc) ? a.UMc[(c0 + ii) * a.ldu + k0 + jj] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int o = o0 + u * kThreads;
            if (o < kRB * kc4) sv[(o / kc4) * kRSD + o % kc4] = x[u];
          }
        }
        for (int o0 = tid; o0 < m8 * kc4; o0 += 8 * kThreads) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int o = o0 + u * kThreads, c = o % m8, jj = o / m8;
            x[u] = (o < m8 * kc4 && c < m && jj < kc) ? __ldcg(A.t + int64_t(k0 + jj) * m + c)
                                                      : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int o = o0 + u * kThreads;
            if (o < m8 * kc4) stT[(o % m8) * kRSD + o / m8] = x[u];
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int tile = warp + u * kWarps;
          if (tile >= ntiles) break;
          const int mt = tile / ntl, nt = tile % ntl;
          const double *va = sv + (mt * 8 + fg) * kRSD + fq;
          const double *tb = stT + (nt * 8 + fg) * kRSD + fq;
          for (int ks = 0; ks < kc4 / 4; ++ks) dmma(acc[u][0], acc[u][1], va[4 * ks], tb[4 * ks]);
        }
      }
    } else {
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tile = warp + u * kWarps;
      if (tile >= ntiles) break;
      const int mt = tile / ntl, nt = tile % ntl;
      const int ii = mt * 8 + fg;
      if (ii >= nr) continue;
      const int64_t i = c0 + ii;
      const int64_t j = (!a.Pw || A.dbg == 7) ? -1 : a.loc[i];
      float pv[2] = {0.0f, 0.0f}, qv[2] = {0.0f, 0.0f};
      if (j >= 0) {  // both columns' state loads in flight together
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = nt * 8 + 2 * fq + e;
          if (c < m) {
            pv[e] = a.Pw[int64_t(c) * a.ldp + j];
            if (a.Qw) qv[e] = a.Qw[int64_t(c) * a.ldp + j];
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = nt * 8 + 2 * fq + e;
        if (c >= m) break;
        const double dd = sgT[c * kRSB + ii] - acc[u][e];
        if (a.D) a.D[i * a.ldd + c] = dd * dsc;
        if (j < 0) continue;
        const int64_t oo = int64_t(c) * a.ldp + j;
        const double p = pv[e], q = qv[e];
        if (a.WB) a.WB[i * a.ldwb + c] = float(a.zp * p + a.zq * q - eta * dd);
        const float pn = float(p + a.e0 * eta * dd);
        a.Pw[oo] = pn;
        float qn = 0.0f;
        if (a.Qw) {
          qn = float(q + a.e1 * eta * dd);
          a.Qw[oo] = qn;
        }
        if (a.Pb) atomicMax(reinterpret_cast<int *>(sbound + c), __float_as_int(fabsf(pn)));
        if (a.Qb && a.Qw)
          atomicMax(reinterpret_cast<int *>(sbound + m + c), __float_as_int(fabsf(qn)));
        if (A.has_next && A.dbg != 9) {
          const float sc = szs[c];
          float z = (zp1 * sc) * pn;
          if (a.Qw) z = fmaf(zq1 * sc, qn, z);
          over |= zop::overflows(z);
          __half h, l;
          zop::split(z, h, l);
          static_cast<__half *>(a.Zhi_next)[int64_t(c) * a.ldz + j] = h;
          static_cast<__half *>(a.Zlo_next)[int64_t(c) * a.ldz + j] = l;
        }
      }
    }
  }
  __syncthreads();
  for (int c = tid; c < m; c += kThreads) {
    if (a.Pb && sbound[c] > 0.0f)
      atomicMax(reinterpret_cast<int *>(a.Pb + c), __float_as_int(sbound[c]));
    if (a.Qb && a.Qw && sbound[m + c] > 0.0f)
      atomicMax(reinterpret_cast<int *>(a.Qb + c), __float_as_int(sbound[m + c]));
  }
  if (!A.has_next || A.dbg == 8) return;
  if (__syncthreads_or(over) && tid == 0) atomicOr(a.zflag + a.flag_idx, 1);
  // ---------------- E: rebuild the next operand if its scale was left ----------------
  // The last CTA to finish reads the flag (threadfence reduction pattern). The
  // scale leaves 64x headroom (zop::scale), so this is a rare slow path: one
  // CTA streams the whole operand.
  __shared__ int last;
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(A.done, 1u) == gridDim.x - 1;
    if (last) {
      atomicExch(A.done, 0u);
      __threadfence();
    }
  }
  __syncthreads();
  if (!last || *reinterpret_cast<volatile int *>(a.zflag + a.flag_idx) == 0) return;
  zop::Next zn{a.Pw, a.Qw, a.ldp, a.n_local, m, zp1, zq1, a.Pb, a.Qb,
               static_cast<__half *>(a.Zhi_next), static_cast<__half *>(a.Zlo_next), a.ldz,
               a.zscale_next};
  zop::next_pass(zn, 0, 1, tid, kThreads);
}

// ---------------- C: t = sum_k T_k (fixed order) ----------------
// sixteen lanes per output, each summing every sixteenth partial (loads issued
// ten at a time), combined in a fixed shuffle tree; a light kernel (few
// registers) so its CTAs are resident and waiting while stage 0 finishes
__global__ void __launch_bounds__(kThreads, 2) phase4_reduce_kernel(const Args A) {
  pdl_wait();
  pdl_trigger();
  constexpr int kL = 16, kU = 10;
  const int rm = A.a.r * A.a.m;
  const int64_t x = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t o = x / kL;
  const int q = int(x % kL);
  const int parts = A.parts;
  double s = 0.0;
  if (o < rm)
    for (int k0 = q; k0 < parts; k0 += kL * kU) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = k0 + kL * u;
        v[u] = k < parts ? __ldcg(A.Tpart + int64_t(k) * rm + o) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) s += v[u];
    }
#pragma unroll
  for (int w = 1; w < kL; w <<= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
  if (q == 0 && o < rm) A.t[o] = s;
}

// ---------------- B + C in one: t = U^T g, one 8 x 8 tile of t per CTA ----------------
// Every CTA reads all b rows of its 8 columns of U and of g (fp64, from L2)
// and runs the K = b contraction on the FP64 tensor cores, the 16 warps each
// taking every 16th group of four rows and their 8 x 8 partials summed in a
// fixed order: no per-CTA r x m partials in HBM (with 148 CTAs of ~7-14 rows,
// 7.7 MB written and read back per iteration at m = 65, r = 100) and no
// separate summing launch.
__global__ void __launch_bounds__(kThreads, 1) phase4_ut_kernel(const Args A) {
  pdl_wait();
  pdl_trigger();
  const sap_step_args &a = A.a;
  const int m = a.m, r = a.r;
  const int ntl = (m + 7) / 8;
  const int mt = blockIdx.x / ntl, nt = blockIdx.x % ntl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fg = lane >> 2, fq = lane & 3;
  const int64_t b = a.b, steps = (b + 3) / 4;
  const int ucol = mt * 8 + fg, gcol = nt * 8 + fg;
  const bool uok = ucol < r, gok = gcol < m;
  double d0 = 0.0, d1 = 0.0;
  constexpr int kU = 4;  // k-steps whose loads are in flight together
  for (int64_t k0 = warp; k0 < steps; k0 += int64_t(kWarps) * kU) {
    double av[kU], bv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = (k0 + int64_t(u) * kWarps) * 4 + fq;
      const bool ok = i < b;
      av[u] = (ok && uok) ? __ldg(a.U + i * a.ldu + ucol) : 0.0;
      bv[u] = (ok && gok) ? __ldcg(a.g + i * a.ldgo + gcol) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) dmma(d0, d1, av[u], bv[u]);
  }
  __shared__ double red[kWarps][64];
  red[warp][fg * 8 + 2 * fq] = d0;
  red[warp][fg * 8 + 2 * fq + 1] = d1;
  __syncthreads();
  if (tid < 64) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w][tid];
    const int row = mt * 8 + tid / 8, col = nt * 8 + tid % 8;
    if (row < r && col < m) A.t[int64_t(row) * m + col] = s;
  }
}

}  // namespace p4
}  // namespace sap

using namespace sap;

namespace {

int grid_for(int64_t b) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // at least four block rows per CTA; never more CTAs than SMs (co-residency)
  return int(std::max<int64_t>(1, std::min<int64_t>(sms, (b + 3) / 4)));
}

constexpr size_t kSmemMax = 220 * 1024;

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

extern "C" {

int sap_block_step_supported(int64_t b, int r, int m) {
  return (b > 0 && r >= 0 && m > 0 && m <= 128 && p4::smem_bytes(m, r) <= kSmemMax) ? 1 : 0;
}

size_t sap_block_step_workspace(int64_t b, int r, int m) {
  if (b <= 0 || r < 0 || m <= 0) return 0;
  const size_t rm = size_t(r) * size_t(m);
  return 256 + align256(size_t(grid_for(b)) * rm * 8) + align256(rm * 8);
}

int sap_block_step(const sap_step_args *args, int mode, void *ws, size_t ws_bytes,
                   void *stream) {
  if (!args) return fail(SAP_ERR_CONTRACT, "block_step: NULL arguments");
  const sap_step_args &a = *args;
  if (a.b <= 0 || a.m <= 0 || a.m > 128 || a.r < 0 || (mode & 3) == 0)
    return fail(SAP_ERR_CONTRACT, "block_step: bad shape b=%lld m=%d r=%d mode=%d",
                (long long)a.b, a.m, a.r, mode);
  const bool do_grad = mode & SAP_STEP_GRAD, do_apply = mode & SAP_STEP_APPLY;
  if (!a.g || a.ldgo < a.m) return fail(SAP_ERR_CONTRACT, "block_step: gradient buffer");
  if (do_grad && ((!a.part && !a.G) || (a.part && !a.zscale) || !a.loc || !a.P || !a.Y))
    return fail(SAP_ERR_CONTRACT, "block_step: gradient inputs missing");
  if (do_apply && a.r > 0 && (!a.U || !a.UMc || a.ldu < a.r))
    return fail(SAP_ERR_CONTRACT, "block_step: Woodbury factor missing");
  if (do_apply && a.Pw && (!a.loc || !a.eta_dev))
    return fail(SAP_ERR_CONTRACT, "block_step: update inputs missing");
  const bool has_next = do_apply && a.Pw && a.Zhi_next && a.Zlo_next && a.zscale_next && a.zflag;
  if (has_next && (a.ldp % 4 || a.ldz % 8 || a.ldz < a.n_local))
    return fail(SAP_ERR_CONTRACT, "block_step: next operand layout");
  const size_t need = sap_block_step_workspace(a.b, a.r, a.m);
  if (!ws || ws_bytes < need)
    return fail(SAP_ERR_CONTRACT, "block_step: workspace %zu < %zu bytes", ws_bytes, need);
  const size_t smem = p4::smem_bytes(a.m, a.r);
  if (smem > kSmemMax)
    return fail(SAP_ERR_CONTRACT, "block_step: shared memory %zu bytes (m=%d r=%d)", smem, a.m,
                a.r);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(p4::phase4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSmemMax));
    attr = true;
  }
  const int G = grid_for(a.b);
  p4::Args A{};
  A.a = a;
  const size_t rm = size_t(a.r) * size_t(a.m);
  A.Tpart = reinterpret_cast<double *>(static_cast<char *>(ws) + 256);
  A.t = reinterpret_cast<double *>(static_cast<char *>(ws) + 256 + align256(size_t(G) * rm * 8));
  A.parts = G;
  A.rows_per = int((a.b + G - 1) / G);
  A.do_grad = do_grad;
  A.do_apply = do_apply;
  A.has_next = has_next;
  {
    const char *e = getenv("SAP_P4_DEBUG");
    A.dbg = e ? atoi(e) : 0;
  }
  const bool woodbury = do_apply && a.r > 0;
  {
    const char *e = getenv("SAP_P4_TPART");
    A.tpart = e && atoi(e) != 0;
  }
  // stages, each one launch in stream order; programmatic dependent launch
  // lets the next stage's grid be scheduled while the previous one runs (it
  // waits in griddepcontrol.wait), so the launch gaps between them shrink
  A.done = static_cast<unsigned *>(ws);
  auto launch = [&](int stage, int grid, size_t sm) -> int {
    A.stage = stage;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(p4::kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = reinterpret_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = getenv("SAP_P4_NO_PDL") ? 0 : 1;
    const cudaError_t e = stage == 1   ? cudaLaunchKernelEx(&cfg, p4::phase4_reduce_kernel, A)
                          : stage == 3 ? cudaLaunchKernelEx(&cfg, p4::phase4_ut_kernel, A)
                                       : cudaLaunchKernelEx(&cfg, p4::phase4_kernel, A);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(SAP_ERR_DEVICE, "block_step: stage %d launch failed: %s", stage,
                  cudaGetErrorString(e));
    }
    return check_launch("phase4_kernel");
  };
  int rc;
  if (A.tpart) {  // stage 0 with per-CTA U^T g partials, summed by stage 1
    if ((do_grad || woodbury) && (rc = launch(0, G, smem)) != SAP_OK) return rc;
    if (!do_apply) return SAP_OK;
    if (woodbury &&
        (rc = launch(1, int((rm * 16 + p4::kThreads - 1) / p4::kThreads), 0)) != SAP_OK)
      return rc;
  } else {        // stage 0 (gradient rows only), then t = U^T g by 8 x 8 tiles
    if (do_grad && (rc = launch(0, G, smem)) != SAP_OK) return rc;
    if (!do_apply) return SAP_OK;
    if (woodbury &&
        (rc = launch(3, ((a.r + 7) / 8) * ((a.m + 7) / 8), 0)) != SAP_OK)
      return rc;
  }
  if ((rc = launch(2, G, smem)) != SAP_OK) return rc;
  return SAP_OK;
}

int sap_woodbury_apply(const double *U, const double *UMc, int64_t ldu, int64_t b, int r,
                       const double *g, int64_t ldg, int m, const double *rho_dev, double *D,
                       int64_t ldd, void *ws, size_t ws_bytes, void *stream) {
  if (!g || !D || ldd < m || ldg < m)
    return fail(SAP_ERR_CONTRACT, "woodbury_apply: bad arguments");
  sap_step_args a{};
  a.b = b;
  a.m = m;
  a.r = r;
  a.U = U;
  a.UMc = UMc;
  a.ldu = ldu;
  a.g = const_cast<double *>(g);
  a.ldgo = ldg;
  a.D = D;
  a.ldd = ldd;
  a.dscale_dev = rho_dev;
  return sap_block_step(&a, SAP_STEP_APPLY, ws, ws_bytes, stream);
}

}  // extern "C"
