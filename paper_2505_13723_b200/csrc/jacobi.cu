// Batched symmetric eigensolver for the Nystrom factorisation's r x r Gram
// matrices (randnla.py:52-94 takes the SVD of the b x r half-sketch; the Gram
// route needs the eigenpairs of H = C^-T (Y^T Y) C^-1, r = 100 by default).
//
// Cyclic two-sided Jacobi in fp64, one CTA per matrix, the matrix and the
// accumulated rotations resident in shared memory (global scratch when r is
// too large for it). Each sweep runs r-1 rounds of r/2 disjoint rotations
// (round-robin "circle" ordering), so a round's rotations are computed in
// parallel and applied as one row pass and one column pass. A rotation is
// skipped when |a_pq| <= eps sqrt(|a_pp a_qq|) (the high-relative-accuracy
// threshold); the solve ends after a sweep without rotations. Eigenvalues
// are returned in descending order with the eigenvectors as matching
// columns -- numpy's eigh reversed, which is how the factorisation consumes
// them. Replaces the host LAPACK (np.linalg.eigh) round trip of round 1.
#include <cfloat>
#include <cmath>
#include <cstdio>

#include <cuda_runtime.h>

#include "common.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace jac {

constexpr int kThreads = 512;
constexpr int kMaxPairs = 256;  // r <= 512

struct Args {
  double *A;        // [count][r][lda] in: symmetric matrices; destroyed
  int64_t strideA;  // elements between matrices
  int lda, r, count;
  double *evals;    // [count][r] descending
  double *V;        // [count][r][ldv] eigenvectors (columns), descending order
  int64_t strideV;
  int ldv;
  int max_sweeps;
  int *sweeps;      // [count] sweeps used (nullable); -1 if not converged
  double *scratch;  // global scratch when the matrices do not fit shared memory
  int smem;         // 1: work arrays in shared memory
};

__global__ void __launch_bounds__(kThreads, 1) jacobi_kernel(const Args a) {
  extern __shared__ __align__(16) double sm[];
  const int r = a.r, n = r + (r & 1);  // even player count (a dummy index when r is odd)
  const int ld = n + 1;                // odd row stride: column passes spread over banks
  const int q = blockIdx.x, tid = threadIdx.x;
  double *H, *Vw;
  if (a.smem) {
    H = sm;
    Vw = sm + size_t(n) * ld;
  } else {
    H = a.scratch + size_t(q) * 2 * n * ld;
    Vw = H + size_t(n) * ld;
  }
  __shared__ double cs[kMaxPairs], sn[kMaxPairs];
  __shared__ int pp[kMaxPairs], qq[kMaxPairs];
  __shared__ int rotated;
  const double *Aq = a.A + int64_t(q) * a.strideA;
  for (int o = tid; o < n * n; o += kThreads) {
    const int i = o / n, j = o % n;
    H[i * ld + j] = (i < r && j < r) ? 0.5 * (Aq[int64_t(i) * a.lda + j] + Aq[int64_t(j) * a.lda + i])
                                     : 0.0;
    Vw[i * ld + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = n / 2, m1 = n - 1;
  int sweep = 0;
  bool converged = false;
  for (; sweep < a.max_sweeps && !converged; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int k = 0; k < m1; ++k) {
      // the round's pairs (circle method: player n-1 fixed, 0..n-2 rotate)
      for (int i = tid; i < half; i += kThreads) {
        int p, s;
        if (i == 0) {
          p = m1;
          s = k;
        } else {
          p = (k + i) % m1;
          s = (k - i + m1) % m1;
        }
        if (p > s) { const int t = p; p = s; s = t; }
        double c = 1.0, sv = 0.0;
        if (s < r) {  // the dummy index never rotates
          const double app = H[p * ld + p], aqq = H[s * ld + s], apq = H[p * ld + s];
          if (fabs(apq) > DBL_EPSILON * sqrt(fabs(app * aqq)) && apq != 0.0) {
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            sv = t * c;
            rotated = 1;
          }
        }
        pp[i] = p;
        qq[i] = s;
        cs[i] = c;
        sn[i] = sv;
      }
      __syncthreads();
      // rows p, q of every pair: H <- J^T H
      for (int o = tid; o < half * n; o += kThreads) {
        const int i = o / n, j = o % n;
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        double *rp = H + pp[i] * ld, *rq = H + qq[i] * ld;
        const double x = rp[j], y = rq[j];
        rp[j] = c * x - s * y;
        rq[j] = s * x + c * y;
      }
      __syncthreads();
      // columns p, q of every pair: H <- H J, V <- V J
      for (int o = tid; o < half * n; o += kThreads) {
        const int i = o / n, j = o % n;
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        double *hr = H + j * ld, *vr = Vw + j * ld;
        const int p = pp[i], t = qq[i];
        const double x = hr[p], y = hr[t];
        hr[p] = c * x - s * y;
        hr[t] = s * x + c * y;
        const double u = vr[p], w = vr[t];
        vr[p] = c * u - s * w;
        vr[t] = s * u + c * w;
      }
      __syncthreads();
      // the rotated pair's off-diagonal entries are zero by construction
      for (int i = tid; i < half; i += kThreads)
        if (sn[i] != 0.0) {
          H[pp[i] * ld + qq[i]] = 0.0;
          H[qq[i] * ld + pp[i]] = 0.0;
        }
      __syncthreads();
    }
    converged = rotated == 0;
    __syncthreads();
  }
  if (tid == 0 && a.sweeps) a.sweeps[q] = converged ? sweep : -1;
  // descending order: rank of each eigenvalue (ties by index)
  double *ev = a.evals + int64_t(q) * r;
  double *Vq = a.V + int64_t(q) * a.strideV;
  for (int i = tid; i < r; i += kThreads) {
    const double li = H[i * ld + i];
    int rank = 0;
    for (int j = 0; j < r; ++j) {
      const double lj = H[j * ld + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    ev[rank] = li;
    for (int k = 0; k < r; ++k) Vq[int64_t(k) * a.ldv + rank] = Vw[k * ld + i];
  }
}

}  // namespace jac
}  // namespace sap

using namespace sap;

extern "C" {

size_t sap_sym_eig_workspace(int r, int count) {
  const int n = r + (r & 1);
  const size_t bytes = size_t(2) * n * (n + 1) * 8;
  return bytes <= 200 * 1024 ? 0 : bytes * size_t(count);
}

int sap_sym_eig_batch(double *A, int64_t strideA, int lda, int r, int count, double *evals,
                      double *V, int64_t strideV, int ldv, int max_sweeps, int *sweeps, void *ws,
                      size_t ws_bytes, void *stream) {
  if (r <= 0 || r > 2 * jac::kMaxPairs || count <= 0 || lda < r || ldv < r || !A || !evals || !V)
    return fail(SAP_ERR_CONTRACT, "sym_eig_batch: bad shape r=%d count=%d", r, count);
  const int n = r + (r & 1);
  const size_t bytes = size_t(2) * n * (n + 1) * 8;
  jac::Args a{A, strideA, lda, r, count, evals, V, strideV, ldv, max_sweeps > 0 ? max_sweeps : 40,
              sweeps, static_cast<double *>(ws), bytes <= 200 * 1024};
  if (!a.smem && (!ws || ws_bytes < bytes * size_t(count)))
    return fail(SAP_ERR_CONTRACT, "sym_eig_batch: workspace %zu < %zu bytes", ws_bytes,
                bytes * size_t(count));
  const size_t smem = a.smem ? bytes : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jac::jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  jac::jacobi_kernel<<<count, jac::kThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("jacobi_kernel");
}

}  // extern "C"
