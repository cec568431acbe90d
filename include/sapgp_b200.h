/*
 * sapgp_b200.h -- C ABI of the B200-native ADASAP hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as void*; none allocates device memory (callers pass workspace)
 * and none synchronises the stream. Return value: SAP_OK or an error code;
 * sap_last_error() returns a thread-local message for the last failure.
 *
 * Status codes map onto the reference exception types (errors.py:4-29):
 *   SAP_ERR_CONTRACT  -> ContractError   (shape/index/precondition)
 *   SAP_ERR_NUMERICAL -> NumericalError
 *   SAP_ERR_DEVICE    -> WorkerError     (CUDA launch/runtime failure)
 *
 * Reference interfaces replaced (paths relative to pkg/src/sapgp/):
 *   sap_prepare_points  <- KernelOracle.__init__ / _scale      kernels.py:45-53, :100-112
 *   sap_gather_points   <- self._scaled[rows], self._row_sq[rows] kernels.py:123-125
 *   sap_krows_times     <- col_dist_matmul (ColDistMatMat)      dist.py:108-127
 *                          row_dist_matmul (RowDistMatMat)      dist.py:130-147
 *                          KernelOracle.tile + family values    kernels.py:56-66, :118-127
 *                          KernelOracle.cross_matmul            kernels.py:161-176
 *                          KernelOracle.matmul                  kernels.py:145-159
 *   sap_ktile(64)       <- KernelOracle.tile / .block / .dense   kernels.py:118-143
 *   sap_grad_gather     <- grad = K[B,:]Z + lam Z[B] - Y[B]     solvers.py:376-377
 *   sap_pq_update       <- nesterov_update on the block rows    solvers.py:76-85, :397-401
 *   sap_woodbury_apply  <- apply_inv (Nystrom-Woodbury)         randnla.py:109-134
 *   sap_block_step      <- Phases I(tail)-IV of adasap_step     solvers.py:376-401
 *   sap_sym_eig_batch   <- the SVD / eigh of rand_nystrom        randnla.py:52-94
 *   sap_combine         <- materialising W (or Z) from the lazy
 *                          two-array Nesterov state
 *   sap_sdd_update      <- sdd_solve's momentum/averaging step  solvers.py:487-493
 *   sap_normal_fill     <- substream(seed, "omega", t).standard_normal  solvers.py:384,
 *                          rng.py:14-24 (numpy PCG64 + ziggurat, bit-exact)
 *   sap_krows_tc (+ sap_tc_points, sap_tc_gather_rows, sap_tc_gather_cols, sap_z_operand)
 *                       <- the same col_dist_matmul product on the 5th-gen
 *                          tensor cores (the solver's Phase I, solvers.py:377)
 *
 * Layouts (all row/column strides in elements):
 *   point set   Xs[j*ldx + k] float32, scaled by 1/lengthscale, zero padded
 *               to ldx (multiple of 4); sqn[j] = |Xs_j|^2 (computed in fp64)
 *   RHS / state column-major n x m: element (row j, column c) at A[c*lda + j]
 *   outputs     row-major b x m: out[i*ldo + c]
 */
#ifndef SAPGP_B200_H
#define SAPGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAP_ABI_VERSION 1

enum { SAP_OK = 0, SAP_ERR_CONTRACT = 1, SAP_ERR_NUMERICAL = 2, SAP_ERR_DEVICE = 3 };
enum { SAP_RBF = 0, SAP_MATERN32 = 1, SAP_MATERN52 = 2 };
/* "family" of the random-feature prior product (gp.py:49-114): the kernel
 * value is cos(x . F_k + p_k) instead of k(x, y); sap_krows_tc only */
enum { SAP_COSINE = 3 };
#define SAP_TC_KA_F16 48
#define SAP_TC_KA_F16X64 96

int sap_abi_version(void);
const char *sap_last_error(void);

/* Number of kernels this library has launched in the process (diagnostics). */
long long sap_launch_count(void);

/* FP32 FFMA throughput probe: 148*4 CTAs x 256 threads x 8 chains x iters FFMA. */
int sap_ffma_peak(float *out, int iters, void *stream);

/* Xs = X / ls (fp64 math, fp32 store, zero padding up to ldx), sqn = |Xs|^2. */
int sap_prepare_points(const double *X, int64_t n, int d, const double *inv_ls,
                       float *Xs, int ldx, float *sqn, void *stream);

/* Rs[i] = Xs[idx[i] - base], rsqn[i] = sqn[idx[i] - base]. */
int sap_gather_points(const float *Xs, const float *sqn, int ldx, const int64_t *idx,
                      int64_t b, int64_t base, float *Rs, float *rsqn, void *stream);

/* Workspace bytes sap_krows_times needs for (b rows, m columns, ncols points). */
size_t sap_krows_workspace(int64_t b, int m, int64_t ncols);

/*
 * out[i, c] (=, or += if accumulate) variance * sum_j k(r_i, x_j) * R[j, c]
 * with R = ca*A + cb*Bm (Bm may be NULL), k the family's unit-variance kernel
 * on scaled points, distances in expansion form clamped at 0 (kernels.py:125).
 * Diagonal rule (kernels.py:126): when row_ids != NULL, entries whose global
 * row id equals the global column id (col_ids[j] if col_ids != NULL else
 * col_base + j) use squared distance exactly 0. Reduction order over the
 * column dimension is fixed for given (b, m, ncols): results are
 * run-to-run deterministic.
 */
int sap_krows_times(const float *Xs, const float *sqn, int ldx, int64_t ncols,
                    const int64_t *col_ids, int64_t col_base,
                    const float *Rs, const float *rsqn, const int64_t *row_ids, int64_t b,
                    int d, const float *A, const float *Bm, int64_t lda, int m,
                    double ca, double cb, int family, double variance,
                    float *out, int64_t ldo, int accumulate,
                    void *ws, size_t ws_bytes, void *stream);

/*
 * Dense tile out[i, j] = variance * k(a_i, c_j) (fp64 out, kernels.py:118-127).
 * When row_ids and col_ids are both non-NULL, entries with equal ids are
 * exactly `variance` (kernels.py:126, :135). With a == c and equal id arrays
 * the result is bitwise symmetric: K[B,B] of kernels.py:129-136.
 */
int sap_ktile(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
              const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc,
              int ldx, int d, int family, double variance, double *out, int64_t ldo,
              void *stream);

/*
 * Dense K[row_ids, col_ids] in the reference's fp64 arithmetic from the fp64
 * points X (n x d row-major) and 1/lengthscale (d): the dense-access API
 * (KernelOracle.tile/block/dense, kernels.py:118-143); bitwise symmetric.
 */
int sap_ktile64(const double *X, const double *inv_ls, int d, const int64_t *row_ids, int64_t na,
                const int64_t *col_ids, int64_t nc, int family, double variance, double *out,
                int64_t ldo, void *stream);

/* sap_ktile with fp32 output (the same fp32-computed values, half the bytes). */
int sap_ktile_f32(const float *Ra, const float *rasqn, const int64_t *row_ids, int64_t na,
                  const float *Rc, const float *rcsqn, const int64_t *col_ids, int64_t nc,
                  int ldx, int d, int family, double variance, float *out, int64_t ldo,
                  void *stream);

/*
 * K_BB of `count` blocks in one launch (the lookahead's power-iteration
 * input; replaces count x oracle.block, kernels.py:129-136): block q's scaled
 * points X + q*strideX ([b][ldx] fp32, sap_gather_points' layout) and squared
 * norms xsq + q*strideSq against themselves into out + q*strideOut ([b][ldo]
 * fp32, ldo and strideOut multiples of 4, 16-byte aligned), variance on the
 * diagonal. The values of sap_ktile_f32 with row_ids = col_ids = the block's
 * (unique) ids, bit for bit. d <= 64.
 */
int sap_ktile_f32_batch(const float *X, int64_t strideX, const float *xsq, int64_t strideSq,
                        int b, int count, int ldx, int d, int family, double variance, float *out,
                        int64_t ldo, int64_t strideOut, void *stream);
/* The same, and K / variance split into fp16 hi + lo ([count] x [b][ldh]
 * each, outh/outl + q*strideH): the operands of the lookahead's three-pass
 * tensor-core sketch K_BB Omega (replaces the fp32 row_dist_matmul of
 * dist.py:130-147). outh = NULL: sap_ktile_f32_batch. */
int sap_ktile_f32_batch_split(const float *X, int64_t strideX, const float *xsq,
                              int64_t strideSq, int b, int count, int ldx, int d, int family,
                              double variance, float *out, int64_t ldo, int64_t strideOut,
                              void *outh, void *outl, int64_t ldh, int64_t strideH, void *stream);

/*
 * Batched preconditioned power-iteration stepsize (replaces randnla.py:165-196
 * rand_power_stepsize, called at solvers.py:389-396), for `count` independent
 * problems q: H_q = P^{-1/2}(K_q + lam I)P^{-1/2} with
 * P^{-1/2} x = x/sqrt(rho_q) + U_q diag(E_q) U_q^T x; `iters` steps from the
 * unit vector v0_q; eta[q] = 1 / (v . H v) of the last step, bad[q] |= 1 when
 * an iterate collapses or the estimate is not positive. K_q: fp32 [b][ldk] at
 * Kbb + q*strideK; U_q: fp64 [b][r] at U + q*strideU; E: [count][r];
 * rho, eta: [count]; v0: [count][b]. r may be 0 (U, E unused).
 */
int sap_power_stepsize(const float *Kbb, int64_t ldk, int64_t strideK, const double *U,
                       int64_t strideU, int r, const double *E, const double *rho,
                       const double *v0, int b, int count, double lam, int iters, double *eta,
                       int *bad, void *stream);

/*
 * g[i, c] = G[i, c] + (own(i) ? lam * Z[j, c] - Y[j, c] : 0), j = loc[i],
 * Z = zp*P + zq*Q; rows with loc[i] < 0 belong to another shard.
 */
int sap_grad_gather(const float *G, int64_t ldg, const float *P, const float *Q,
                    const float *Y, int64_t ldp, double zp, double zq,
                    const int64_t *loc, int64_t b, int m, double lam,
                    double *g, int64_t ldgo, void *stream);

/*
 * Block-row Nesterov step in the lazy basis: for owned rows
 *   WB[i, c] = Z[j, c] - eta * D[i, c]          (Z = zp*P + zq*Q, old basis)
 *   P[j, c] += e0 * eta * D[i, c];  Q[j, c] += e1 * eta * D[i, c]
 * eta is read from device memory (eta_dev[0]). Pb/Qb (nullable) are per-column
 * magnitude bounds, raised (atomicMax) to cover the updated values.
 */
int sap_pq_update(float *P, float *Q, int64_t ldp, const int64_t *loc, int64_t b, int m,
                  const double *D, int64_t ldd, const double *eta_dev,
                  double zp, double zq, double e0, double e1,
                  float *WB, int64_t ldwb, float *Pb, float *Qb, void *stream);

/* out = a*P + b*Q (column-major n x m, ld ldp); Q may be NULL (b ignored). */
int sap_combine(float *out, int64_t ldo, const float *P, const float *Q, int64_t ldp,
                int64_t n, int m, double a, double b, void *stream);

/* ---- tensor-core path (krows_tc.cu) ------------------------------------ */

/*
 * Augmented features for the 3-term tf32 distance GEMM (ka = 32 for d <= 9,
 * 64 for d <= 20): row form RA[j*ka..] and/or column form CA[j*ka..]
 * (either may be NULL), scaled by sqrt(c_family)/lengthscale.
 */
int sap_tc_points(const double *X, int64_t n, int d, const double *inv_ls, int family, int ka,
                  float *RA, float *CA, void *stream);

/* out[i*ka..] = RA[idx[i]*ka..] for i < b, zero rows for b <= i < bpad. */
int sap_tc_gather_rows(const float *RA, int ka, const int64_t *idx, int64_t b, int64_t bpad,
                       float *out, void *stream);

/* Column-form features (CA layout) of the points idx[0..b), rebuilt exactly
 * from their row form RA; rows b..bpad-1 are zero. */
int sap_tc_gather_cols(const float *RA, int ka, int d, int family, const int64_t *idx, int64_t b,
                       int64_t bpad, float *out, void *stream);

/*
 * Z operand of the tensor-core product: Zhi/Zlo (fp16, [nz][ldz]) = split of
 * scale_c * (zp*P + zq*Q) with scale_c a power of two from the bounds Pb/Qb
 * (zscale[c] receives it), for rows c < m. Rows m..nz-1 (MMA padding) are
 * not written: the caller zeroes them once. Q/Qb may be NULL.
 */
int sap_z_operand(const float *P, const float *Q, int64_t ldp, int64_t n, int m, double zp,
                  double zq, const float *Pb, const float *Qb, int nz, int64_t ldz, void *Zhi,
                  void *Zlo, float *zscale, void *stream);

/* out[c] = max_j |A[c*lda + j]| (bounds for RHS that are not solver state). */
int sap_colabsmax(const float *A, int64_t lda, int64_t n, int m, float *out, void *stream);

size_t sap_krows_tc_workspace(int64_t b, int m, int64_t ncols);

/* 1 if (d features, m right-hand sides) fits the tensor-core path, else 0. */
int sap_tc_supported(int d, int m);

/*
 * Tensor-core block-row product (tcgen05 + TMEM + TMA, sm_100a):
 * out[i, c] (=, or +=) variance * sum_j k(row_i, col_j) Z[j, c] with rows
 * RAg ([bpad][ka], bpad a multiple of 128), columns CA ([ncols][ka]) and Z
 * (features fp32 for ka = 32 or 64; ka = SAP_TC_KA_F16 / SAP_TC_KA_F16X64
 * means 32 / 64 fp16 features per point -- the same tf32-rounded values,
 * exact in fp16 -- and needs bpad a multiple of 256; the distance GEMM then
 * runs kind::f16)
 * given by sap_z_operand. Diagonal rule as sap_krows_times (row_ids vs
 * col_base + j). nz <= 128.
 */
int sap_krows_tc(const void *CA, int64_t ncols, int ka, const void *RAg, int64_t bpad,
                 const int64_t *row_ids, int64_t b, int64_t col_base, const void *Zhi,
                 const void *Zlo, int nz, int64_t ldz, const float *zscale, int m, int family,
                 double variance, float *out, int64_t ldo, int accumulate, void *ws,
                 size_t ws_bytes, void *stream);

/*
 * Augmented features of the random-feature prior product (gp.py:49-114):
 * rows (points X, n x d fp64) RA[n][32] = [xh, xh, xl, 1, 1, 0...] and columns
 * (frequencies F, q x d fp64, phases p) CA[q][32] = [Fh, Fl, Fh, ph, pl, 0...]
 * (tf32-rounded splits), so the tensor-core GEMM gives x.F_k + p_k to ~2^-21
 * relative. Either output may be NULL; d <= 9.
 * sap_krows_tc(..., family = SAP_COSINE, variance = sqrt(2 var / q), ...) then
 * computes out = variance * cos(X F^T + p) Z, Z = theta (q x s) -- phi(X) theta
 * without materialising phi.
 */
int sap_cos_features(const double *X, int64_t n, int d, const double *F, const double *phase,
                     int64_t q, float *RA, float *CA, void *stream);

/*
 * SDD step (solvers.py:463-516, the stochastic-dual-descent baseline on the
 * same block product): with V, W, E column-major (ldv >= rows),
 *   V[j] = momentum*V[j] - eta*g[i] for owned block rows j = loc[i] >= 0,
 *   V[j] = momentum*V[j] elsewhere;  W += V;  E += avg*(W - E).
 * VB (b x m fp32) and pos (rows ints, all -1 on entry and on return) are
 * caller workspace; rows and ldv are multiples of 4 (pad rows are zero).
 */
int sap_sdd_update(float *V, float *W, float *E, int64_t ldv, int64_t rows, int m,
                   const int64_t *loc, int64_t b, const double *g, int64_t ldg, double eta,
                   double momentum, double avg, float *VB, int *pos, void *stream);

/*
 * Device-side numpy Generator.standard_normal (replaces the host draw of the
 * Nystrom test matrix, substream(seed, "omega", t).standard_normal((b, r)),
 * solvers.py:384 via rng.py:14-24). states: device array [nstreams][4] of
 * u64 = PCG64 (state_hi, state_lo, inc_hi, inc_lo) as numpy's
 * bit_generator.state reports them for a fresh generator. Writes the first
 * `count` normals of stream s to out[s*ldo + i] (fp64), the same values
 * numpy draws (csrc/rng.cu). count <= 2^20. *sap_normal_status(ws) (a device
 * int the caller zeroes with the workspace) is sticky: 0 while every fill on
 * this workspace succeeded, nonzero once one ran out of raw words or had too
 * many rejection draws.
 */
size_t sap_normal_workspace(int64_t count, int nstreams);
int sap_normal_fill(const uint64_t *states, int nstreams, int64_t count, double *out, int64_t ldo,
                    void *ws, size_t ws_bytes, void *stream);
int *sap_normal_status(void *ws);
/* Device int64: the raw 64-bit words the last fill of MORE than 2^20 normals
 * consumed from its stream (one stream): PCG64.advance(words) continues the
 * stream exactly, so a long draw can be produced in chunks. */
long long *sap_normal_words(void *ws);

/*
 * Host-side draws of iterations t0 .. t0+count-1 (no GPU involved; replaces
 * the per-iteration numpy draws of the reference, solvers.py:260-262 block,
 * :250-251 crc, :384 Nystrom test-matrix stream, :395 power start vector,
 * via rng.py:14-24 substreams). Per iteration i:
 *   blocks[i*b .. i*b+b)   sorted substream(seed,"block",t).choice(n,b,replace=False)
 *   crcs[i]                zlib.crc32 of those int64 bytes
 *   omega_states[4*i ..]   PCG64 words of substream(seed,"omega",t) (NULL: skip)
 *   v0[i*b .. i*b+b)       substream(seed,"power",t).standard_normal(b) / its norm
 *                          (NULL: skip; SAP_ERR_NUMERICAL if zero twice)
 * Bit-exact with numpy except v0's normalisation (sum-of-squares order).
 * Runs on nthreads host threads without the Python GIL.
 */
int sap_host_draws(uint64_t seed, int64_t t0, int count, int64_t n, int64_t b, int64_t *blocks,
                   uint32_t *crcs, int64_t *omega_states, double *v0, int nthreads);

/* ---- Phase IV in one launch (phase4.cu) -------------------------------- */

/*
 * Arguments of sap_block_step: one ADASAP iteration after the block-row
 * product (solvers.py:376-401). All arrays are device memory.
 */
typedef struct sap_step_args {
  /* gradient source: the tensor-core partials [splits][m][b] left in the
   * sap_krows_tc_next workspace (reduce = 0; scaled by 2^14 zscale[c]), or,
   * with part == NULL, a reduced product G (b x m fp32, row-major, ldg) */
  const float *part;
  int splits;
  float variance;
  const float *zscale;
  const float *G;
  int64_t ldg;
  /* lam Z[B] - Y[B] with Z = zp*P + zq*Q (column-major m x ldp, Q nullable) */
  const float *P, *Q, *Y;
  int64_t ldp;
  double zp, zq, lam;
  const int64_t *loc; /* block row i -> local row, or -1 (owned by another rank) */
  int64_t b;
  int m;
  double *g;          /* gradient, b x m fp64 row-major (ldgo): out (GRAD) / in (APPLY only) */
  int64_t ldgo;
  /* Woodbury: D = g - UMc (U^T g), U and UMc = U Mc b x r fp64 row-major (ldu);
   * Mc = (rho S^-1 + U^T U)^-1 (randnla.py:109-134); r = 0: D = g */
  const double *U, *UMc;
  int64_t ldu;
  int r;
  /* lazy Nesterov update of the owned block rows (sap_pq_update semantics;
   * eta_dev[0] is eta/rho); Pw == NULL skips the update */
  float *Pw, *Qw;
  const double *eta_dev;
  double e0, e1;
  float *WB;
  int64_t ldwb;
  float *Pb, *Qb;
  /* optional D output, D * (1 / dscale_dev[0]) (dscale_dev nullable) */
  double *D;
  int64_t ldd;
  const double *dscale_dev;
  /* optional next tensor-core operand (the buffer sap_krows_tc_next filled):
   * the updated block rows' Z_{t+1} = zp1*P + zq1*Q are written into it; if
   * one leaves its column's scale, the whole buffer is rebuilt in the same
   * launch. zflag: two device ints, zero-initialised; flag_idx alternates
   * 0/1 per call */
  void *Zhi_next, *Zlo_next;
  int64_t ldz;
  float *zscale_next;
  double zp1, zq1;
  int *zflag;
  int flag_idx;
  int64_t n_local;
} sap_step_args;

enum { SAP_STEP_GRAD = 1, SAP_STEP_APPLY = 2 };

/* 1 if sap_block_step handles these shapes (m <= 128 and the staged tiles fit
 * shared memory), else 0 (callers use the unfused kernels). */
int sap_block_step_supported(int64_t b, int r, int m);

/* Workspace bytes of sap_block_step / sap_woodbury_apply; the first 256
 * bytes (grid barrier) must be zeroed once before the first call. */
size_t sap_block_step_workspace(int64_t b, int r, int m);

/*
 * mode GRAD: g = K[B,:]Z + lam Z[B] - Y[B] (solvers.py:376-377) -- the
 *   per-rank part before the all-reduce of g;
 * mode APPLY: D = g - UMc U^T g, then the update / D output / next operand;
 * GRAD|APPLY: both in one cooperative launch (one GPU).
 * Replaces sap_grad_gather + apply_inv (randnla.py:109-134) + sap_pq_update.
 */
int sap_block_step(const sap_step_args *args, int mode, void *ws, size_t ws_bytes,
                   void *stream);

/*
 * D = (g - UMc (U^T g)) / rho_dev[0]: the Nystrom-preconditioned block
 * direction of apply_inv (randnla.py:109-134) for b x m fp64 g, with
 * UMc = U (rho S^-1 + U^T U)^-1 precomputed (the Cholesky solve of the
 * reference folded into the r x r core). Workspace: sap_block_step_workspace.
 */
int sap_woodbury_apply(const double *U, const double *UMc, int64_t ldu, int64_t b, int r,
                       const double *g, int64_t ldg, int m, const double *rho_dev, double *D,
                       int64_t ldd, void *ws, size_t ws_bytes, void *stream);

/*
 * sap_krows_tc plus two options for the solver:
 *  - reduce = 0 leaves the unreduced partials in ws ([splits][m][b], for
 *    sap_block_step) and stores the split count in *splits_out;
 *  - Zhi_next != NULL also fills the NEXT iterate's operand
 *    Z_{t+1} = zp*P + zq*Q (scale from the bounds Pb/Qb) into Zhi_next /
 *    Zlo_next / zscale_next: inside the block-row kernel by its otherwise idle
 *    control warps (the CTA-pair kernel), else by a separate sap_z_operand pass.
 */
int sap_krows_tc_next(const void *CA, int64_t ncols, int ka, const void *RAg, int64_t bpad,
                      const int64_t *row_ids, int64_t b, int64_t col_base, const void *Zhi,
                      const void *Zlo, int nz, int64_t ldz, const float *zscale, int m,
                      int family, double variance, float *out, int64_t ldo, int accumulate,
                      void *ws, size_t ws_bytes, int reduce, int *splits_out, const float *P,
                      const float *Q, int64_t ldp, double zp, double zq, const float *Pb,
                      const float *Qb, void *Zhi_next, void *Zlo_next, float *zscale_next,
                      void *stream);

/* ---- batched symmetric eigensolver (jacobi.cu) ------------------------- */

/*
 * Eigen-decomposition of `count` symmetric r x r fp64 matrices (A[q] at
 * A + q*strideA, row stride lda): evals[q*r + k] descending and the
 * matching eigenvectors as columns of V[q] (V + q*strideV, row stride ldv).
 * Backend: cuSOLVER's batched syev (cusolverDnXsyevBatched, loaded at run
 * time) by default; SAP_EIG=jacobi selects the cyclic two-sided Jacobi
 * kernel (one CTA per matrix; A symmetrised, then destroyed). sweeps[q] =
 * Jacobi sweeps used (cuSOLVER: 0), -1 if not converged; required with
 * cuSOLVER (its info array).
 * Replaces np.linalg.eigh on the Nystrom Gram matrices (the Gram route of
 * rand_nystrom, randnla.py:52-94). Workspace: sap_sym_eig_workspace (for
 * the backend selected at call time).
 */
size_t sap_sym_eig_workspace(int r, int count);
int sap_sym_eig_batch(double *A, int64_t strideA, int lda, int r, int count, double *evals,
                      double *V, int64_t strideV, int ldv, int max_sweeps, int *sweeps,
                      void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SAPGP_B200_H */
