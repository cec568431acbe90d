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
//
// Two backends: cuSOLVER's batched syev (cusolverDnXsyevBatched, loaded at
// run time; the north star allows cuSOLVER for the small factorisations) by
// default -- 0.85 ms for a lookahead batch of 32 at r = 100 on one B200 --
// and the Jacobi kernel below (SAP_EIG=jacobi; 4.3 ms for the same batch on
// 32 SMs, measured with scripts/micro/eig_bench.cu).
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

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
      // rows p, q of every pair: H <- J^T H (warp per pair, lanes over columns)
      const int warp = tid >> 5, lane = tid & 31;
      for (int i = warp; i < half; i += kThreads / 32) {
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        double *rp = H + pp[i] * ld, *rq = H + qq[i] * ld;
        for (int j = lane; j < n; j += 32) {
          const double x = rp[j], y = rq[j];
          rp[j] = c * x - s * y;
          rq[j] = s * x + c * y;
        }
      }
      __syncthreads();
      // columns p, q of every pair: H <- H J, V <- V J (lanes over rows)
      for (int i = warp; i < half; i += kThreads / 32) {
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        const int p = pp[i], t = qq[i];
        for (int j = lane; j < n; j += 32) {
          double *hr = H + j * ld, *vr = Vw + j * ld;
          const double x = hr[p], y = hr[t];
          hr[p] = c * x - s * y;
          hr[t] = s * x + c * y;
          const double u = vr[p], w = vr[t];
          vr[p] = c * u - s * w;
          vr[t] = s * u + c * w;
        }
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

// cuSOLVER's output (column-major eigenvectors, ascending eigenvalues) into
// this API's layout (eigenvector columns of a row-major V, descending)
__global__ void reorder_kernel(const double *Acm, int64_t strideA, int lda, const double *w,
                               int r, double *evals, double *V, int64_t strideV, int ldv,
                               int *info) {
  const int q = blockIdx.y;
  const int64_t o = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= int64_t(r) * r) return;
  const int i = int(o / r), k = int(o % r);  // V[i][k] = eigvec_{r-1-k}[i]
  V[int64_t(q) * strideV + int64_t(i) * ldv + k] =
      Acm[int64_t(q) * strideA + int64_t(r - 1 - k) * lda + i];
  if (i == 0) evals[int64_t(q) * r + k] = w[int64_t(q) * r + r - 1 - k];
  if (o == 0 && info) info[q] = info[q] == 0 ? 0 : -1;  // this API: -1 = not converged
}

// cuSOLVER's batched syev, loaded at run time (the process may already hold
// torch's copy of libcusolver; no link-time dependency)
struct Cusolver {
  using Create = cusolverStatus_t (*)(cusolverDnHandle_t *);
  using SetStream = cusolverStatus_t (*)(cusolverDnHandle_t, cudaStream_t);
  using CreateParams = cusolverStatus_t (*)(cusolverDnParams_t *);
  using BufSize = cusolverStatus_t (*)(cusolverDnHandle_t, cusolverDnParams_t, cusolverEigMode_t,
                                       cublasFillMode_t, int64_t, cudaDataType, const void *,
                                       int64_t, cudaDataType, const void *, cudaDataType, size_t *,
                                       size_t *, int64_t);
  using Syev = cusolverStatus_t (*)(cusolverDnHandle_t, cusolverDnParams_t, cusolverEigMode_t,
                                    cublasFillMode_t, int64_t, cudaDataType, void *, int64_t,
                                    cudaDataType, void *, cudaDataType, void *, size_t, void *,
                                    size_t, int *, int64_t);
  Create create = nullptr;
  SetStream set_stream = nullptr;
  CreateParams create_params = nullptr;
  BufSize bufsize = nullptr;
  Syev syev = nullptr;
  bool ok = false;
};

Cusolver &cusolver() {
  static Cusolver c;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    c.create = reinterpret_cast<Cusolver::Create>(dlsym(h, "cusolverDnCreate"));
    c.set_stream = reinterpret_cast<Cusolver::SetStream>(dlsym(h, "cusolverDnSetStream"));
    c.create_params = reinterpret_cast<Cusolver::CreateParams>(dlsym(h, "cusolverDnCreateParams"));
    c.bufsize = reinterpret_cast<Cusolver::BufSize>(dlsym(h, "cusolverDnXsyevBatched_bufferSize"));
    c.syev = reinterpret_cast<Cusolver::Syev>(dlsym(h, "cusolverDnXsyevBatched"));
    c.ok = c.create && c.set_stream && c.create_params && c.bufsize && c.syev;
  });
  return c;
}

// cuSOLVER handles are not thread-safe and costly to create (and the first
// batched syev on a new handle initialises for ~0.1 s): a process-wide pool,
// a handle taken for the duration of one call, so the lookahead's producer
// threads -- new ones for every engine -- reuse warm handles.
struct Handle {
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t p = nullptr;
  std::vector<char> host_ws;
};
std::mutex g_pool_mu;
std::vector<Handle *> g_pool;

Handle *new_handle() {
  Handle *th = new Handle;
  Cusolver &c = cusolver();
  if (c.ok && c.create(&th->h) == CUSOLVER_STATUS_SUCCESS) c.create_params(&th->p);
  return th;
}

// The pool is filled once with warm handles: the first batched syev on a
// fresh handle initialises for ~0.1 s, which inside the lookahead stalls the
// solver; paying it up front (the first factorisation) keeps it out of steps.
constexpr int kWarmHandles = 8;
void prewarm_pool() {
  static std::once_flag once;
  std::call_once(once, [] {
    Cusolver &c = cusolver();
    if (!c.ok) return;
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return;
    double *buf = nullptr;
    int *info = nullptr;
    void *dws = nullptr;
    cudaMalloc(&buf, 64 * sizeof(double));
    cudaMalloc(&info, sizeof(int));
    const double eye[16] = {2, 0, 0, 0, 0, 3, 0, 0, 0, 0, 4, 0, 0, 0, 0, 5};
    std::vector<Handle *> made;
    for (int k = 0; k < kWarmHandles; ++k) {
      Handle *th = new_handle();
      made.push_back(th);
      if (!th->h) continue;
      size_t dw = 0, hw = 0;
      if (c.bufsize(th->h, th->p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, 4,
                    CUDA_R_64F, buf, 4, CUDA_R_64F, buf + 16, CUDA_R_64F, &dw, &hw, 1) !=
          CUSOLVER_STATUS_SUCCESS)
        continue;
      if (!dws) cudaMalloc(&dws, dw > 0 ? dw * 4 : 256);
      th->host_ws.resize(hw);
      cudaMemcpyAsync(buf, eye, sizeof(eye), cudaMemcpyHostToDevice, st);
      c.set_stream(th->h, st);
      c.syev(th->h, th->p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, 4, CUDA_R_64F, buf,
             4, CUDA_R_64F, buf + 16, CUDA_R_64F, dws, dw > 0 ? dw * 4 : 256,
             th->host_ws.data(), hw, info, 1);
    }
    cudaStreamSynchronize(st);
    cudaFree(buf);
    cudaFree(info);
    cudaFree(dws);
    cudaStreamDestroy(st);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (Handle *th : made) g_pool.push_back(th);
  });
}

struct Lease {
  Handle *th = nullptr;
  Lease() {
    prewarm_pool();
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      if (!g_pool.empty()) {
        th = g_pool.back();
        g_pool.pop_back();
      }
    }
    if (!th) th = new_handle();
  }
  ~Lease() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(th);
  }
};

bool use_cusolver() {
  const char *e = getenv("SAP_EIG");
  return !(e && strcmp(e, "jacobi") == 0) && cusolver().ok;
}

size_t cusolver_ws(Handle &th, int r, int count, size_t *host) {
  size_t dws = 0, hws = 0;
  if (!th.h || cusolver().bufsize(th.h, th.p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r,
                                   CUDA_R_64F, nullptr, r, CUDA_R_64F, nullptr, CUDA_R_64F, &dws,
                                   &hws, count) != CUSOLVER_STATUS_SUCCESS)
    return 0;
  if (host) *host = hws;
  return dws;
}

}  // namespace jac
}  // namespace sap

using namespace sap;

extern "C" {

size_t sap_sym_eig_workspace(int r, int count) {
  if (r <= 0 || count <= 0) return 0;
  const size_t mats = size_t(count) * r * r * 8, vals = size_t(count) * r * 8;
  if (jac::use_cusolver()) {  // the matrices (column-major copy), eigenvalues, cuSOLVER's buffer
    jac::Lease lease;
    return (mats + 255) / 256 * 256 + (vals + 255) / 256 * 256 +
           jac::cusolver_ws(*lease.th, r, count, nullptr);
  }
  const int n = r + (r & 1);
  const size_t bytes = size_t(2) * n * (n + 1) * 8;
  return bytes <= 200 * 1024 ? 0 : bytes * size_t(count);
}

int sap_sym_eig_batch(double *A, int64_t strideA, int lda, int r, int count, double *evals,
                      double *V, int64_t strideV, int ldv, int max_sweeps, int *sweeps, void *ws,
                      size_t ws_bytes, void *stream) {
  if (r <= 0 || r > 2 * jac::kMaxPairs || count <= 0 || lda < r || ldv < r || !A || !evals || !V)
    return fail(SAP_ERR_CONTRACT, "sym_eig_batch: bad shape r=%d count=%d", r, count);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (jac::use_cusolver()) {
    // cuSOLVER's batched syev (SAP_EIG=jacobi selects the Jacobi kernel)
    if (!sweeps) return fail(SAP_ERR_CONTRACT, "sym_eig_batch: sweeps (status) array required");
    jac::Lease lease;
    jac::Handle &th = *lease.th;
    size_t hws = 0;
    const size_t dws = jac::cusolver_ws(th, r, count, &hws);
    const size_t mats = size_t(count) * r * r * 8, vals = size_t(count) * r * 8;
    const size_t need = (mats + 255) / 256 * 256 + (vals + 255) / 256 * 256 + dws;
    if (!th.h || !ws || ws_bytes < need)
      return fail(SAP_ERR_CONTRACT, "sym_eig_batch: workspace %zu < %zu bytes", ws_bytes, need);
    char *w = static_cast<char *>(ws);
    double *Acm = reinterpret_cast<double *>(w);
    double *wv = reinterpret_cast<double *>(w + (mats + 255) / 256 * 256);
    void *dbuf = w + (mats + 255) / 256 * 256 + (vals + 255) / 256 * 256;
    // the matrices densely packed (cuSOLVER's batch layout); symmetric, so
    // row-major in is column-major in
    if (lda == r && strideA == int64_t(r) * r) {
      cudaMemcpyAsync(Acm, A, mats, cudaMemcpyDeviceToDevice, st);
    } else {
      for (int q = 0; q < count; ++q)
        cudaMemcpy2DAsync(Acm + size_t(q) * r * r, size_t(r) * 8, A + q * strideA,
                          size_t(lda) * 8, size_t(r) * 8, size_t(r), cudaMemcpyDeviceToDevice, st);
    }
    if (th.host_ws.size() < hws) th.host_ws.resize(hws);
    jac::cusolver().set_stream(th.h, st);
    int *info = sweeps;  // info per matrix (0 = converged)
    const cusolverStatus_t cs = jac::cusolver().syev(
        th.h, th.p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r, CUDA_R_64F, Acm, r,
        CUDA_R_64F, wv, CUDA_R_64F, dbuf, dws, th.host_ws.data(), hws, info, count);
    if (cs != CUSOLVER_STATUS_SUCCESS)
      return fail(SAP_ERR_DEVICE, "sym_eig_batch: cusolverDnXsyevBatched status %d", int(cs));
    dim3 grid(unsigned((int64_t(r) * r + 255) / 256), unsigned(count));
    jac::reorder_kernel<<<grid, 256, 0, st>>>(Acm, int64_t(r) * r, r, wv, r, evals, V, strideV,
                                              ldv, info);
    return check_launch("eig_reorder_kernel");
  }
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
  jac::jacobi_kernel<<<count, jac::kThreads, smem, st>>>(a);
  return check_launch("jacobi_kernel");
}

}  // extern "C"
