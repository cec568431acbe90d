// Host API and helper kernels of the tensor-core block-row product (the
// kernel itself is in krows_tc.cuh, instantiated per family in krows_tc_*.cu).
#include <cstdio>
#include <cstdarg>
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <cstdlib>

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "krows_tc.cuh"
#include "krows_tc2.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace tck {

bool launch_tc_rbf(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                   const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc_m32(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                   const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc_m52(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                   const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc2_rbf(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                    const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc2_m32(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                    const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc2_m52(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                    const CUtensorMap &, const Params &, int, int, int, cudaStream_t);
bool launch_tc2_cos(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                    const CUtensorMap &, const Params &, int, int, int, cudaStream_t);

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

// augmented feature columns a family needs (RBF carries the exp2 offset)
inline int tc_features(int d, int family) { return 3 * d + 4 + (family == SAP_RBF ? 1 : 0); }

// Row form [zh, zh, zl, nh, nl, 1, 1] and column form [-2zh, -2zl, -2zh, 1, 1,
// nh, nl] give S = |z_i|^2 + |z_j|^2 - 2 z_i.z_j from a 3-term tf32 split. For
// RBF (rbf=1) the column form is negated and one more pair (1, 14) is
// appended, so the tensor core delivers S = 14 - s and the epilogue is a bare
// exp2 (P = 2^14 k).
__global__ void build_aug_kernel(const double *X, int64_t n, int d, const double *inv_ls,
                                 double cfam, int ka, int rbf, float *RA, float *CA) {
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
    const float cs = rbf ? 2.0f : -2.0f;
    if (ca) { ca[k] = cs * zh; ca[d + k] = cs * zl; ca[2 * d + k] = cs * zh; }
  }
  const float nh = tf32_trunc(float(nrm));
  const float nl = tf32_round(float(nrm - double(nh)));
  const int o = 3 * d;
  if (ra) { ra[o] = nh; ra[o + 1] = nl; ra[o + 2] = 1.0f; ra[o + 3] = 1.0f; }
  const float sg = rbf ? -1.0f : 1.0f;
  if (ca) { ca[o] = sg; ca[o + 1] = sg; ca[o + 2] = sg * nh; ca[o + 3] = sg * nl; }
  const int used = rbf ? o + 5 : o + 4;
  if (rbf) {
    if (ra) ra[o + 4] = 1.0f;
    if (ca) ca[o + 4] = tck::kPExp;
  }
  for (int k = used; k < ka; ++k) {
    if (ra) ra[k] = 0.0f;
    if (ca) ca[k] = 0.0f;
  }
}

// random-feature rows / columns (sap_cos_features): x.F + p from a 3-term split
__global__ void cos_features_kernel(const double *X, int64_t n, int d, const double *F,
                                    const double *phase, int64_t q, float *RA, float *CA) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr int ka = 32;
  if (RA && j < n) {
    float *ra = RA + j * ka;
    for (int k = 0; k < d; ++k) {
      const double x = X[j * d + k];
      const float h = tf32_trunc(float(x));
      ra[k] = h; ra[d + k] = h; ra[2 * d + k] = tf32_round(float(x - double(h)));
    }
    ra[3 * d] = 1.0f; ra[3 * d + 1] = 1.0f;
    for (int k = 3 * d + 2; k < ka; ++k) ra[k] = 0.0f;
  }
  if (CA && j < q) {
    float *ca = CA + j * ka;
    for (int k = 0; k < d; ++k) {
      const double f = F[j * d + k];
      const float h = tf32_trunc(float(f));
      ca[k] = h; ca[d + k] = tf32_round(float(f - double(h))); ca[2 * d + k] = h;
    }
    const double p = phase[j];
    const float ph = tf32_trunc(float(p));
    ca[3 * d] = ph; ca[3 * d + 1] = tf32_round(float(p - double(ph)));
    for (int k = 3 * d + 2; k < ka; ++k) ca[k] = 0.0f;
  }
}

__global__ void gather_rows_kernel(const float *RA, int ka, const int64_t *idx, int64_t b,
                                   int64_t bpad, float *out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= bpad * ka) return;
  const int64_t i = e / ka;
  out[e] = i < b ? RA[idx[i] * ka + (e % ka)] : 0.0f;
}

// column form of gathered points rebuilt from their row form (build_aug_kernel
// layouts; every step is a sign flip or a factor of 2, so it is exact): lets a
// block of points serve as the column set of a product (the Nystrom sketch
// K[B,B] Omega) without a column-form copy of every point
__global__ void gather_cols_kernel(const float *RA, int ka, int d, int rbf, const int64_t *idx,
                                   int64_t b, int64_t bpad, float *out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= bpad * ka) return;
  const int64_t i = e / ka;
  const int k = int(e % ka);
  float v = 0.0f;
  if (i < b) {
    const float *ra = RA + idx[i] * ka;
    const float cs = rbf ? 2.0f : -2.0f, sg = rbf ? -1.0f : 1.0f;
    const int o = 3 * d;
    if (k < d) v = cs * ra[k];                      // -2 zh   (x row zh)
    else if (k < 2 * d) v = cs * ra[d + k];         // -2 zl   (x row zh): ra[2d + (k-d)]
    else if (k < o) v = cs * ra[k - d];             // -2 zh   (x row zl): ra[d + (k-2d)]
    else if (k == o || k == o + 1) v = sg;          // 1       (x row nh, nl)
    else if (k == o + 2) v = sg * ra[o];            // nh      (x row 1)
    else if (k == o + 3) v = sg * ra[o + 1];        // nl      (x row 1)
    else if (k == o + 4 && rbf) v = tck::kPExp;     // 14      (x row 1)
  }
  out[e] = v;
}

// The operand passes use the shared helpers of zop.cuh, so the stand-alone
// pass, the block-row kernel's overlapped pass and the Phase IV patch write
// bit-identical operands.
// vectorised form: 8 consecutive points per thread (2 x float4 from P and Q,
// one 16-byte store each to Zhi and Zlo); needs 16-byte aligned rows
__global__ void z_operand_vec_kernel(const float *P, const float *Q, int64_t ldp, int64_t n,
                                     float zp, float zq, const float *Pb, const float *Qb,
                                     int64_t ldz, __half *Zhi, __half *Zlo, float *zscale) {
  const int c = blockIdx.y;
  const float sc = zop::scale(zp, zq, Pb, Qb, Q != nullptr, c);
  if (blockIdx.x == 0 && threadIdx.x == 0) zscale[c] = sc;
  const float a = zp * sc, bq = zq * sc;
  const float *pr = P + int64_t(c) * ldp;
  const float *qr = Q ? Q + int64_t(c) * ldp : nullptr;
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; j < ldz;
       j += int64_t(gridDim.x) * blockDim.x * 8) {
    float z[8];
    zop::load8<false>(pr, qr, j, n, a, bq, z);
    zop::store8<false>(z, Zhi + int64_t(c) * ldz, Zlo + int64_t(c) * ldz, j);
  }
}

__global__ void z_operand_kernel(const float *P, const float *Q, int64_t ldp, int64_t n,
                                 float zp, float zq, const float *Pb, const float *Qb,
                                 int64_t ldz, __half *Zhi, __half *Zlo, float *zscale) {
  const int c = blockIdx.y;
  const float sc = zop::scale(zp, zq, Pb, Qb, Q != nullptr, c);
  if (blockIdx.x == 0 && threadIdx.x == 0) zscale[c] = sc;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ldz;
       j += int64_t(gridDim.x) * blockDim.x) {
    float z = 0.0f;
    if (j < n) {
      z = zp * P[int64_t(c) * ldp + j];
      if (Q) z = fmaf(zq, Q[int64_t(c) * ldp + j], z);
      z *= sc;
    }
    zop::split(z, Zhi[int64_t(c) * ldz + j], Zlo[int64_t(c) * ldz + j]);
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
  // partials are [splits][m][b] (block rows contiguous): consecutive threads
  // take consecutive rows of one column, so every partial load is coalesced
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int c = int(e / b);
  const int64_t i = e % b;
  // eight independent partial sums: eight loads in flight per thread (the
  // partials of one element are b*m floats apart; a single running sum left
  // the kernel latency-bound)
  const int64_t bm = b * m;
  const float *pe = part + e;
  float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  int k = 0;
  for (; k + 8 <= splits; k += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += pe[int64_t(k + u) * bm];
  }
  for (int u = 0; k < splits; ++k, ++u) acc[u] += pe[int64_t(k) * bm];
  const float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
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
              uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
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
  if (n < 0 || d < 1 || (ka != 32 && ka != 64) || tc_features(d, family) > ka)
    return fail(SAP_ERR_CONTRACT, "tc_points: d=%d does not fit ka=%d", d, ka);
  const double l2e = 1.4426950408889634;
  double cfam = family == SAP_RBF ? 0.5 * l2e : (family == SAP_MATERN32 ? 3.0 : 5.0) * l2e * l2e;
  if (n == 0) return SAP_OK;
  build_aug_kernel<<<unsigned((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(X, n, d, inv_ls,
                                                                               cfam, ka, family == SAP_RBF, RA, CA);
  return check_launch("build_aug_kernel");
}

int sap_cos_features(const double *X, int64_t n, int d, const double *F, const double *phase,
                     int64_t q, float *RA, float *CA, void *stream) {
  if (n < 0 || q < 0 || d < 1 || 3 * d + 2 > 32)
    return fail(SAP_ERR_CONTRACT, "cos_features: d=%d outside the tensor-core path (d <= 9)", d);
  const int64_t rows = std::max(RA ? n : 0, CA ? q : 0);
  if (rows == 0) return SAP_OK;
  cos_features_kernel<<<unsigned((rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      X, n, d, F, phase, q, RA, CA);
  return check_launch("cos_features_kernel");
}

int sap_tc_gather_rows(const float *RA, int ka, const int64_t *idx, int64_t b, int64_t bpad,
                       float *out, void *stream) {
  if (b <= 0 || bpad < b) return fail(SAP_ERR_CONTRACT, "tc_gather_rows: bad shape");
  const int64_t tot = bpad * ka;
  gather_rows_kernel<<<unsigned((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(RA, ka, idx, b,
                                                                                   bpad, out);
  return check_launch("gather_rows_kernel");
}

int sap_tc_gather_cols(const float *RA, int ka, int d, int family, const int64_t *idx,
                       int64_t b, int64_t bpad, float *out, void *stream) {
  if (b <= 0 || bpad < b || tc_features(d, family) > ka)
    return fail(SAP_ERR_CONTRACT, "tc_gather_cols: bad shape");
  const int64_t tot = bpad * ka;
  gather_cols_kernel<<<unsigned((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      RA, ka, d, family == SAP_RBF, idx, b, bpad, out);
  return check_launch("gather_cols_kernel");
}

int sap_z_operand(const float *P, const float *Q, int64_t ldp, int64_t n, int m, double zp,
                  double zq, const float *Pb, const float *Qb, int nz, int64_t ldz, void *Zhi,
                  void *Zlo, float *zscale, void *stream) {
  if (m <= 0 || nz < m || nz % 16 || ldz < n || ldz % 8)
    return fail(SAP_ERR_CONTRACT, "z_operand: bad shape m=%d nz=%d ldz=%lld", m, nz,
                (long long)ldz);
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = ldp % 4 == 0 && al16(P) && (!Q || al16(Q)) && al16(Zhi) && al16(Zlo);
  cudaStream_t st = (cudaStream_t)stream;
  if (vec) {
    const int64_t groups = ldz / 8;
    dim3 grid(unsigned(std::min<int64_t>((groups + 255) / 256, 1024)), unsigned(m));
    z_operand_vec_kernel<<<grid, 256, 0, st>>>(P, Q, ldp, n, float(zp), float(zq), Pb, Qb, ldz,
                                               static_cast<__half *>(Zhi),
                                               static_cast<__half *>(Zlo), zscale);
    return check_launch("z_operand_vec_kernel");
  }
  dim3 grid(unsigned(std::min<int64_t>((ldz + 255) / 256, 256)), unsigned(m));
  z_operand_kernel<<<grid, 256, 0, st>>>(P, Q, ldp, n, float(zp), float(zq), Pb, Qb, ldz,
                                         static_cast<__half *>(Zhi), static_cast<__half *>(Zlo),
                                         zscale);
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

int sap_tc_supported(int d, int m) {
  const int f = tc_features(d, SAP_RBF);  // the widest family
  const int ka = f <= 32 ? 32 : 64;
  const int nz = (m + 15) / 16 * 16;
  return (f <= 64 && tc_fits(nz, ka)) ? 1 : 0;
}

// splits for the CTA-pair kernel: whole waves of 74 pairs over 256-row tiles
int tc2_splits(int64_t b, int64_t tiles) {
  if (const char *e = getenv("SAP_TC_SPLITS")) {  // experiments: a fixed split count
    const int s = atoi(e);
    if (s > 0) return int(std::min<int64_t>(s, std::max<int64_t>(1, tiles)));
  }
  const int64_t rt = (b + 2 * BM - 1) / (2 * BM);
  const int64_t pairs = kSms / 2;
  int64_t best = 1;
  double best_eff = -1.0;
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(tiles / 4, 4096));
  for (int64_t s = 1; s <= std::min<int64_t>(max_s, 8 * pairs); ++s) {
    const int64_t total = rt * s;
    const int64_t waves = (total + pairs - 1) / pairs;
    if (waves > 8) break;
    const double eff = double(total) / double(waves * pairs);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return int(best);
}

bool use_pair(int nz, int ka) {
  const char *e = getenv("SAP_TC_PAIR");
  return (!e || atoi(e) != 0) && tck2::tc2_fits(nz, ka);
}

size_t sap_krows_tc_workspace(int64_t b, int m, int64_t ncols) {
  const int64_t t1 = (ncols + NT - 1) / NT, t2 = (ncols + tck2::NT - 1) / tck2::NT;
  const int64_t s = std::max<int64_t>(tc_splits(b, t1), tc2_splits(b, t2));
  // partial sums, then (256-byte aligned) the dynamic unit counter
  return (size_t(s) * size_t(b) * size_t(m) * sizeof(float) + 255) / 256 * 256 + 256;
}

// launch tags of the dynamic unit counter (any start value works)
std::atomic<unsigned> g_tc_epoch{0x5a17u};
// launch epochs per workspace, consecutive, so each launch finds the counter
// slot the previous launch on that workspace armed for it (krows_tc2.cuh)
std::mutex g_epoch_mu;
std::unordered_map<const void *, unsigned> g_ws_epoch;
unsigned next_epoch(const void *ws) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  auto it = g_ws_epoch.find(ws);
  if (it == g_ws_epoch.end()) {
    if (g_ws_epoch.size() > 4096) g_ws_epoch.clear();  // bounded; a miss only costs one re-arm
    it = g_ws_epoch.emplace(ws, g_tc_epoch.fetch_add(0x10000u, std::memory_order_relaxed)).first;
  }
  return ++it->second;
}

int sap_krows_tc_next(const void *CA, int64_t ncols, int ka, const void *RAg, int64_t bpad,
                      const int64_t *row_ids, int64_t b, int64_t col_base, const void *Zhi,
                      const void *Zlo, int nz, int64_t ldz, const float *zscale, int m,
                      int family, double variance, float *out, int64_t ldo, int accumulate,
                      void *ws, size_t ws_bytes, int reduce, int *splits_out, const float *P,
                      const float *Q, int64_t ldp, double zp, double zq, const float *Pb,
                      const float *Qb, void *Zhi_next, void *Zlo_next, float *zscale_next,
                      void *stream) {
  const bool half = ka == tck2::kKaF16 || ka == tck2::kKaF16x64;  // 32 / 64 fp16 features
  const int kah = ka == tck2::kKaF16x64 ? 64 : 32;                 // their count
  if (b <= 0 || m <= 0 || ncols <= 0 || (ka != 32 && ka != 64 && !half) || nz % 16 || nz < m ||
      nz > 128 || bpad % BM || bpad < b || ldz % 8 || ldz < ncols || ncols > INT32_MAX)
    return fail(SAP_ERR_CONTRACT, "krows_tc: bad shape b=%lld m=%d nz=%d ncols=%lld ka=%d",
                (long long)b, m, nz, (long long)ncols, ka);
  if (reduce && ldo < m) return fail(SAP_ERR_CONTRACT, "krows_tc: ldo < m");
  if (!reduce && !splits_out) return fail(SAP_ERR_CONTRACT, "krows_tc: splits_out is NULL");
  if (Zhi_next && (!Zlo_next || !zscale_next || !P || !Pb || (Q && !Qb)))
    return fail(SAP_ERR_CONTRACT, "krows_tc: next operand arguments incomplete");
  const bool pair = use_pair(nz, ka) && bpad % (2 * BM) == 0;
  if (half && !pair)
    return fail(SAP_ERR_CONTRACT, "krows_tc: fp16 features need the CTA-pair kernel "
                "(bpad %% 256 == 0, nz=%d)", nz);
  const int nt = pair ? tck2::NT : NT;
  const int64_t tiles = (ncols + nt - 1) / nt;
  Params p{};
  p.b = b;
  p.ncols = ncols;
  p.col_base = col_base;
  p.row_ids = row_ids;
  p.m = m;
  p.row_tiles = int(bpad / (pair ? 2 * BM : BM));
  p.tiles = tiles;
  p.splits = pair ? tc2_splits(b, tiles) : tc_splits(b, tiles);
  {
    const char *dbg = getenv("SAP_TC_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
  }
  static unsigned long long *prof_buf = nullptr;
  const char *prof_env = getenv("SAP_TC_PROF");
  if (p.debug == 9 || (prof_env && atoi(prof_env))) {
    if (!prof_buf) cudaMalloc(&prof_buf, 148 * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prof_buf, 0, 148 * 16 * sizeof(unsigned long long), (cudaStream_t)stream);
    p.prof = prof_buf;
  }
  const size_t need = size_t(p.splits) * size_t(b) * size_t(m) * sizeof(float);
  if (!ws || ws_bytes < need)
    return fail(SAP_ERR_CONTRACT, "krows_tc: workspace %zu < %zu bytes", ws_bytes, need);
  p.part = static_cast<float *>(ws);
  {
    const size_t part_bytes = (need + 255) / 256 * 256;
    const char *st_env = getenv("SAP_TC_STATIC");
    if (ws_bytes >= part_bytes + 8 && !(st_env && atoi(st_env))) {
      p.sched = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + part_bytes);
      p.epoch = next_epoch(p.sched);
    }
  }
  // the next operand inside the CTA-pair kernel (16-byte vector rows only)
  auto al16 = [](const void *q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  // ... and only when the two control warps finish it under the product: the
  // pass moves 12 n m bytes at ~0.9 TB/s over the GPU (long columns per CTA)
  // or ~0.5 TB/s (short ones, zop::next_pass), the product takes ~b n /
  // (1.4e12 Matern, 2.2e12 RBF/cosine entries/s). Otherwise the separate pass
  // (full HBM bandwidth, ~13 us at config 2) is cheaper than a side job the
  // launch waits for (config 2: side job 0.151 ms launch vs ~0.12 + 0.013).
  // SAP_ZNEXT_SEPARATE=1 / SAP_ZNEXT_SIDE=1 force either.
  bool side_fits = true;
  if (!getenv("SAP_ZNEXT_SIDE")) {
    const double rate = family == SAP_MATERN32 || family == SAP_MATERN52 ? 1.4e12 : 2.2e12;
    const bool short_cols = (ldz / 8) / kSms < 4 * 64;
    const double side_s = 12.0 * double(ncols) * double(m) / (short_cols ? 0.5e12 : 0.9e12);
    const double prod_s = double(bpad) * double(ncols) / rate;
    side_fits = side_s < 0.95 * prod_s;
  }
  const bool side = Zhi_next && pair && ldp % 4 == 0 && ldz % 8 == 0 && al16(P) &&
                    (!Q || al16(Q)) && al16(Zhi_next) && al16(Zlo_next) && side_fits &&
                    getenv("SAP_ZNEXT_SEPARATE") == nullptr;
  if (side)
    p.zn = zop::Next{P, Q, ldp, ncols, m, float(zp), float(zq), Pb, Qb,
                     static_cast<__half *>(Zhi_next), static_cast<__half *>(Zlo_next), ldz,
                     zscale_next};
  if (!pair && !tc_fits(nz, ka))
    return fail(SAP_ERR_CONTRACT, "krows_tc: nz=%d ka=%d tile ring does not fit shared memory", nz,
                ka);

  // B operands: the pair kernel stages half a column tile (64 points) and
  // half of the right-hand sides (nz/2) per CTA
  const uint32_t xbox = pair ? tck2::NT / 2 : NT;
  const uint32_t zbox = pair ? nz / 2 : nz;
  CUtensorMap tm_rows, tm_cols, tm_zhi, tm_zlo;
  const bool fmaps_ok =
      half ? make_map(&tm_rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, RAg, kah, bpad, size_t(kah) * 2,
                      kah, BM, kah == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B) &&
                 make_map(&tm_cols, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, CA, kah, ncols,
                          size_t(kah) * 2, kah, xbox,
                          kah == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B)
           : make_map(&tm_rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, RAg, ka, bpad, size_t(ka) * 4, 32,
                      BM) &&
                 make_map(&tm_cols, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CA, ka, ncols,
                          size_t(ka) * 4, 32, xbox);
  if (!fmaps_ok ||
      !make_map(&tm_zhi, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Zhi, ncols, nz, size_t(ldz) * 2, 64, zbox) ||
      !make_map(&tm_zlo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Zlo, ncols, nz, size_t(ldz) * 2, 64, zbox))
    return fail(SAP_ERR_DEVICE, "krows_tc: cuTensorMapEncodeTiled failed");

  cudaStream_t st = (cudaStream_t)stream;
  const int units = p.row_tiles * p.splits;
  const int grid = pair ? 2 * std::min(units, kSms / 2) : std::min(units, kSms);
  int rc;
  bool launched;
  if (family == SAP_RBF)
    launched = pair ? launch_tc2_rbf(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st)
                    : launch_tc_rbf(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st);
  else if (family == SAP_MATERN32)
    launched = pair ? launch_tc2_m32(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st)
                    : launch_tc_m32(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st);
  else if (family == SAP_MATERN52)
    launched = pair ? launch_tc2_m52(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st)
                    : launch_tc_m52(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st);
  else if (family == SAP_COSINE)
    launched = pair && ka == 32 && !row_ids &&
               launch_tc2_cos(tm_rows, tm_cols, tm_zhi, tm_zlo, p, nz, ka, grid, st);
  else
    return fail(SAP_ERR_CONTRACT, "krows_tc: unknown family %d", family);
  if (!launched) return fail(SAP_ERR_CONTRACT, "krows_tc: shape nz=%d ka=%d unsupported", nz, ka);
  if ((rc = check_launch(pair ? "krows_tc2_kernel" : "krows_tc_kernel")) != SAP_OK) return rc;
  if (p.prof) {  // profiling only: per-role cycle totals, averaged over CTAs
    unsigned long long h[148 * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, p.prof, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[16] = {"prod.wait_empty", "prod.issue", "mma.wait_full", "mma.wait_pfull",
                             "mma.wait_gempty", "mma.issue_g1", "mma.issue_g2", "epi.wait_sfull",
                             "epi.convert", "epi.arrive", "epi.drain", "kernel",
                             "epi.first_tile_at", "epi.done_at", "sidejob.done_at",
                             "epi.take_unit"};
    for (int k = 0; k < 16; ++k) {
      double s0 = 0, s1 = 0; int n0 = 0, n1 = 0;
      for (int g = 0; g < grid; ++g) {
        if (g % 2 == 0) { s0 += h[g * 16 + k]; ++n0; } else { s1 += h[g * 16 + k]; ++n1; }
      }
      fprintf(stderr, "[tc prof] %-18s leader %12.0f  peer %12.0f cycles/CTA\n", names[k],
              n0 ? s0 / n0 : 0.0, n1 ? s1 / n1 : 0.0);
    }
  }
  if (Zhi_next && !side &&
      (rc = sap_z_operand(P, Q, ldp, ncols, m, zp, zq, Pb, Qb, nz, ldz, Zhi_next, Zlo_next,
                          zscale_next, stream)) != SAP_OK)
    return rc;
  if (!reduce) {
    *splits_out = p.splits;
    return SAP_OK;
  }
  const int64_t tot = b * m;
  tc_reduce_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(p.part, p.splits, b, m,
                                                                float(variance), zscale, out, ldo,
                                                                accumulate);
  return check_launch("tc_reduce_kernel");
}

int sap_krows_tc(const void *CA, int64_t ncols, int ka, const void *RAg, int64_t bpad,
                 const int64_t *row_ids, int64_t b, int64_t col_base, const void *Zhi,
                 const void *Zlo, int nz, int64_t ldz, const float *zscale, int m, int family,
                 double variance, float *out, int64_t ldo, int accumulate, void *ws,
                 size_t ws_bytes, void *stream) {
  return sap_krows_tc_next(CA, ncols, ka, RAg, bpad, row_ids, b, col_base, Zhi, Zlo, nz, ldz,
                           zscale, m, family, variance, out, ldo, accumulate, ws, ws_bytes, 1,
                           nullptr, nullptr, nullptr, 0, 0.0, 0.0, nullptr, nullptr, nullptr,
                           nullptr, nullptr, stream);
}

}  // extern "C"
