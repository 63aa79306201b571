/*
 * ngd.h -- C-ABI of the B200-native NystromNGD inner solve (libngd_b200.so).
 *
 * The reference (nystromngd, pure Python/numpy) has no FFI: its boundary is a
 * duck-typed Python protocol.  Each entry point below backs one
 * piece of that protocol; the Python host layer (paper_2505_11638_b200/*.py)
 * binds them with ctypes exactly as INTEGRATION.md shows.
 *
 * Conventions
 *   - every pointer argument named d_* is a DEVICE pointer (fp64 unless noted);
 *     h_* are host pointers.  Work is stream-ordered on the context's stream.
 *   - p x ell matrices crossing the ABI are COLUMN-major (each column a
 *     contiguous p-vector) unless the name says _rowmajor.
 *   - parameter vectors use the reference's flat layout: per layer W (n_out x n_in)
 *     row-major, then b (model.py:41-51).
 *   - return value: NGD_OK or one of the NGD_E_* codes; ngd_last_error() gives text.
 *     Python maps NGD_E_SHAPE -> ValueError, NGD_E_NONFINITE -> NonFiniteError,
 *     NGD_E_CHOL -> retry / SketchFailure, NGD_E_CUDA/NCCL -> RuntimeError.
 */
#ifndef NGD_B200_H_
#define NGD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGD_OK 0
#define NGD_E_SHAPE 1
#define NGD_E_NONFINITE 2
#define NGD_E_CHOL 3
#define NGD_E_CUDA 4
#define NGD_E_NCCL 5
#define NGD_E_STATE 6

typedef struct ngd_ctx ngd_ctx;

/* SolveReport (krylov.py:12-21) */
typedef struct ngd_solve_report {
  int32_t iterations;
  int32_t matvecs;
  int32_t converged;
  int32_t breakdown;
  double relative_residual;
} ngd_solve_report;

const char* ngd_last_error(void);
int ngd_version(void);

/* ---- context: MlpTopology (model.py:12-51) + device workspace ---------- */
int ngd_ctx_create(const int32_t* widths, int32_t n_widths, int32_t device, ngd_ctx** out);
int ngd_ctx_destroy(ngd_ctx* ctx);
int ngd_ctx_set_stream(ngd_ctx* ctx, void* cuda_stream);
int64_t ngd_param_count(const ngd_ctx* ctx);

/* ---- multi-GPU: point shards + NCCL all-reduce -------------- */
int ngd_nccl_unique_id(uint8_t* h_id_out /* 128 bytes */);
int ngd_ctx_set_comm(ngd_ctx* ctx, const uint8_t* h_id /* 128 bytes */, int32_t rank, int32_t nranks);

/* ---- quadrature: QuadratureSet + data offsets (problems.py:34-48,161-177)
 * x_* row-major (n, d); w_* quadrature weights; off_* residual offsets
 * (source f on interior points, -g on boundary points) so that
 * residual = metric + off.  Device pointers, copied into the context. */
int ngd_set_points(ngd_ctx* ctx, int64_t n_int, const double* d_x_int, const double* d_w_int,
                   const double* d_off_int, int64_t n_bnd, const double* d_x_bnd, const double* d_w_bnd,
                   const double* d_off_bnd);
/* General row set (heat1p1d's metric and residual stacks differ, problems.py:294-311):
 * "head" rows at the interior points and "value" rows (F = u) at the second point set,
 * each with a METRIC weight wm (Gramian) and a RESIDUAL weight wr (loss / gradient);
 * a row absent from one stack carries weight 0 there.  ngd_set_points(...) ==
 * ngd_set_rows(..., w_int, w_int, ..., w_bnd, w_bnd, ...). */
int ngd_set_rows(ngd_ctx* ctx, int64_t n_int, const double* d_x_int, const double* d_wm_int,
                 const double* d_wr_int, const double* d_off_int, int64_t n_val, const double* d_x_val,
                 const double* d_wm_val, const double* d_wr_val, const double* d_off_val);
/* Output head of the interior rows.  coef: C = d+2 coefficients over the
 * output channels (value, d_1 u .. d_d u, Lambda), Lambda = sum_{i in lap_mask} d_ii u;
 * metric row  F = coef.o + 3 kappa ubar^2 u   (ubar = u at theta_bar, frozen),
 * residual    R = coef.o + kappa u^3 + off.
 * poisson*: coef = e_Lambda, kappa 0, mask all; heat1p1d: coef = e_{d_t} - e_Lambda,
 * mask {x}; nlpoisson2d: coef = e_Lambda, kappa = -1 (problems.py:161-385).
 * Default: the Poisson head. */
int ngd_set_head(ngd_ctx* ctx, const double* h_coef, int32_t n_coef, double kappa, uint32_t lap_mask);

/* ---- loss (PdeProblem.loss_value, problems.py:92-99); all-reduced ------- */
int ngd_loss(ngd_ctx* ctx, const double* d_theta, double* h_loss);
/* relative H1 error at the interior points (PdeProblem.h1_relative_error, problems.py:104-119):
 * d_exact = per interior point [u*, grad u*] ((n_int, d+1) row-major); weights = interior metric weights */
int ngd_h1_error(ngd_ctx* ctx, const double* d_theta, const double* d_exact, double* h_err);
/* loss at theta - alpha * dir (backtracking_linesearch candidate, optim.py:137) */
int ngd_loss_at(ngd_ctx* ctx, const double* d_theta, double alpha, const double* d_dir, double* h_loss);

/* ---- linearisation (GramianOperator.from_problem, gramian.py:33-41) -----
 * caches jets + adjoints at theta; also returns the loss (may be NULL) and,
 * if d_metric != NULL, the metric stack values [Lap u]_int ++ [u]_bnd. */
int ngd_linearize(ngd_ctx* ctx, const double* d_theta, double* h_loss, double* d_metric);
/* as ngd_linearize, with the metric coefficient frozen at d_theta_bar (NULL: theta; the
 * metric_stack(theta, freeze(theta_bar)) of problems.py:364-373) and, if d_resid != NULL,
 * the residual rows.  After a theta_bar != theta linearisation ngd_loss_grad is refused. */
int ngd_linearize_ex(ngd_ctx* ctx, const double* d_theta, const double* d_theta_bar, double* h_loss,
                     double* d_metric, double* d_resid);
/* gradient J^T (w o r) at the current linearisation (PdeProblem.loss_grad, problems.py:101-102) */
int ngd_loss_grad(ngd_ctx* ctx, double* d_grad);
/* metric-stack JVP / VJP at the current linearisation (LinearizedMap.jvp/vjp, autodiff.py:605-609) */
int ngd_jvp(ngd_ctx* ctx, const double* d_v, double* d_out /* n_int + n_bnd */);
int ngd_vjp(ngd_ctx* ctx, const double* d_cot /* n_int + n_bnd */, double* d_out /* p */);

/* ---- Gramian (GramianOperator.matvec/matmat, ShiftedOperator; gramian.py:48-61,123-135) */
int ngd_gram_matvec(ngd_ctx* ctx, const double* d_v, double mu, double* d_out);
int ngd_gram_matmat(ngd_ctx* ctx, const double* d_V, int64_t ell, int64_t ldv, double* d_Y, int64_t ldy);
/* dense G = J^T diag(w) J (p x p column-major, ldg >= p), one DSYRK per Jacobian-row chunk
 * (assemble_dense, gramian.py:138-145; the spectrum of harness.py:237-266) */
int ngd_gram_dense(ngd_ctx* ctx, double* d_G, int64_t ldg);

/* ---- randomized Nystrom (nystrom_approximate, sketch.py:58-90) ----------
 * prepare: orthonormalise Omega in place (p x ell, col-major).
 * finish : given Y = G Omega, produce U (p x ell, column-major) and eigenvalues
 *          (descending, >= 0); returns NGD_E_CHOL when Omega^T Y_nu is not PD. */
int ngd_fill_gaussian(ngd_ctx* ctx, uint64_t seed, double* d_out, int64_t n);
int ngd_nystrom_prepare(ngd_ctx* ctx, double* d_omega, int64_t p, int32_t ell);
int ngd_nystrom_finish(ngd_ctx* ctx, const double* d_omega, double* d_Y, int64_t p, int32_t ell,
                       double* d_U, double* d_eig, double* h_shift);
/* small dense SVD A = U diag(sigma) V^T of an ell x ell column-major matrix (the step of
 * sketch.py:85 after B = QR); method 3 = block-exchange cluster Jacobi (FP64),
 * 4 = FP32 pre-sweeps + FP64 block Jacobi (the library's choice for ell <= 512; V in global memory
 * above ~310), 1 = cuSOLVER polar SVD (the library's choice above 512).  h_sweeps receives the
 * Jacobi sweep count (negative if not converged; method 4: 1000 * FP32 sweeps + FP64 sweeps). */
int ngd_small_svd(ngd_ctx* ctx, const double* d_A, int32_t ell, double* d_U, double* d_sigma, int32_t method,
                  int32_t* h_sweeps);
/* dense operator helper (DenseOperator.matmat, gramian.py:101-120): Y = G V */
int ngd_dense_matmat(ngd_ctx* ctx, const double* d_G, int64_t p, const double* d_V, int64_t ell, double* d_Y);
/* the in-house FP64 DMMA GEMM behind every dense product of the sketch / factorisation (test hook):
 * C = alpha op(A) op(B) + beta C, column-major, op = transpose when trans_* != 0 */
int ngd_gemm(ngd_ctx* ctx, int32_t trans_a, int32_t trans_b, int32_t M, int32_t N, int32_t K, double alpha,
             const double* d_A, int64_t lda, const double* d_B, int64_t ldb, double beta, double* d_C, int64_t ldc);

/* the FP64-exact GEMM on the INT8 tensor cores (Ozaki scheme II: 16 moduli, tcgen05 kind::i8,
 * CRT) behind the large sketches' S = J_c Omega and Y += J_c^T S (gramian.py:55-61; test hook):
 * C = alpha A B + beta C with K-major A(m, k) = d_A[m lda + k], B(k, n) = d_B[n ldb + k],
 * C column-major.  Option "sketch_gemm" selects the sketch engine (0 DMMA, 1 INT8, 2 auto). */
int ngd_gemm_ozaki(ngd_ctx* ctx, int32_t M, int32_t N, int32_t K, double alpha, const double* d_A, int64_t lda,
                   const double* d_B, int64_t ldb, double beta, double* d_C, int64_t ldc);

/* ---- preconditioner (NystromPreconditioner.apply, sketch.py:101-112) ---- */
int ngd_precond_apply(ngd_ctx* ctx, const double* d_U, const double* d_eig, int32_t ell, double mu,
                      const double* d_v, double* d_out, int64_t p);

/* ---- PCG (krylov.py:24-88) on (G + mu I) at the current linearisation, or on
 * a dense SPD matrix d_dense (p x p) when non-NULL.  U/eig may be NULL (no precond). */
int ngd_pcg(ngd_ctx* ctx, const double* d_dense, int64_t p, const double* d_b, double mu,
            const double* d_U, const double* d_eig, int32_t ell, double precond_mu, double rel_tol,
            int32_t maxit, int32_t recompute_every, double* d_x, ngd_solve_report* h_report);

/* upper Cholesky A = U^T U in place (A n x n column-major, upper triangle read/written), the
 * factorisation inside ngd_nystrom_* exposed for testing: method 0 = the library's choice (one CTA,
 * cluster, blocked with DMMA updates above 512), 1 one-CTA (n <= 160), 2 8-CTA cluster (n <= 512);
 * *h_info = 0 or the first failing pivot + 1 (LAPACK potrf semantics) */
int ngd_small_cholesky(ngd_ctx* ctx, double* d_A, int32_t n, int32_t method, int32_t* h_info);

/* ---- knobs: "svd" = 3 (FP32 pre-sweeps + FP64 block Jacobi for ell <= 512, cuSOLVER polar SVD above;
 *      default) | 1 (polar SVD at every ell);  "graphs" = 1 (replay PCG iterations as a CUDA graph,
 *      default) | 0;  "pdl" = 1 (programmatic dependent launch along the PCG kernel chain, default;
 *      process-wide) | 0;  "l2window" / "l2u" = 1 (L2 persisting windows over the jets / the
 *      preconditioner basis during PCG, default) | 0;  "force_comm" = 1 (build an NCCL communicator
 *      even for one rank: tests of the multi-rank paths) */
int ngd_set_option(ngd_ctx* ctx, const char* key, int64_t value);
/* diagnostics: "jacobi_sweeps" (FP64 sweeps of the last Nystrom factorisation), "jacobi_sweeps_f32"
 * (its FP32 pre-sweeps, svd = 3), "phase_b_splits" */
int ngd_get_stat(ngd_ctx* ctx, const char* key, int64_t* out);

/* ---- vector helpers used by the host policy ------------------------------
 * ngd_dot: h_out = x . y (deterministic reduction, synchronises);
 * ngd_axpy: out = a - alpha * b (theta update / line-search candidate, optim.py:137,252) */
int ngd_dot(ngd_ctx* ctx, const double* d_x, const double* d_y, int64_t n, double* h_out);
int ngd_axpy(ngd_ctx* ctx, const double* d_a, double alpha, const double* d_b, double* d_out, int64_t n);

/* ---- evidence for bench.py ---------------------------------------------
 * ngd_launch_count: number of this library's kernel launches so far (process-wide).
 * ngd_probe_start(kind, n): bracket the next n launches of kernel class `kind`
 *   (1 FWD jets, 2 REV jets, 3 phase A, 4 phase B, 5 J rows, 6 preconditioner,
 *   7 vector/scalar, 8 pack, 9 small SVD, 10 small Cholesky, 11 (unused), 12 cuSOLVER, 13 triangular
 *   solve, 14 DMMA GEMM, 15 INT8 tensor-core GEMM, 16 Ozaki residue conversion, 17 CRT
 *   reconstruction; 0 = every class at once, read back with ngd_probe_stop_all) with CUDA events
 *   on their launch stream;
 *   ngd_probe_stop returns the summed device time and the launch count. */
int ngd_stream_sync(ngd_ctx* ctx);
int64_t ngd_launch_count(void);
/* algorithmic FLOPs (2 M N K) of every in-house DMMA GEMM launched so far (process-wide) */
double ngd_gemm_flops(void);
/* INT8 tensor ops (2 M N K per modulus) of every Ozaki-scheme GEMM launched so far (process-wide) */
double ngd_i8_ops(void);
/* FP64 elements converted to residues (Ozaki scheme) so far (process-wide) */
double ngd_oz_conv_elems(void);
/* algorithmic FLOPs (2 P_w S each) of the phase A (kind 3) / phase B (kind 4) invocations launched
 * directly so far (process-wide; graph captures excluded, like the per-launch timing) */
double ngd_phase_flops(int32_t kind);
int ngd_probe_start(int32_t kind, int32_t max_launches);
int ngd_probe_stop(double* h_total_ms, int64_t* h_count);
int ngd_probe_stop_all(double* h_ms, int64_t* h_count, int32_t n_kinds);

#ifdef __cplusplus
}
#endif
#endif /* NGD_B200_H_ */
