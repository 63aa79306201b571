// Internal launch interface of the CUDA kernels (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ngd_common.cuh"

namespace ngd {

// kernel classes for launch accounting / probe timing (ngd_probe.cu)
enum KernelKind {
  K_FWD = 1, K_REV = 2, K_PHA = 3, K_PHB = 4, K_FORMJ = 5, K_PRECOND = 6, K_VEC = 7, K_PACK = 8, K_SVD = 9, K_CHOL = 10,
  K_BLAS = 11, K_SOLVER = 12,  // library calls (cuBLAS / cuSOLVER): timed, not counted as our launches
  K_TRSM = 13, K_GEMM = 14, K_I8GEMM = 15, K_OZCONV = 16, K_OZCRT = 17
};
void probe_before(int kind, cudaStream_t st);
void probe_after(int kind, cudaStream_t st);
void lib_probe_before(int kind, cudaStream_t st);
void lib_probe_after(int kind, cudaStream_t st);

// device-side PCG scalars (krylov.py:24-88)
struct PcgState {
  double bb, norm_b, tol, rz, rz_new, dad, alpha, rr, rel, beta;
  int iterations, matvecs, breakdown, converged, done, it;
};

// Nystrom preconditioner operands read by the kernels from device memory, so a
// captured CUDA graph can be replayed for a new factor / damping.
struct PrecondArgs {
  const double* U;  // p x ell row-major
  const double* eig;
  double mu;
};

enum JetMode { FWD = 0, REV = 1, PHA = 2 };

struct JetArgs {
  const double* A;     // packed operand, row-major [Mp][Kp] (zero padded)
  int Kp;              // padded K (multiple of 16)
  int K;               // real K (0 = use Kp); k-steps beyond K are skipped
  int M;               // real rows
  const double* B;     // [Kp rows][s_pad], zero rows beyond K
  int64_t s_pad;
  int64_t col0;        // first column of this segment (interior 0, boundary int_cols)
  int pt0;             // first padded point index of this segment
  const double* bias;  // FWD: b_k, PHA: vb_k (value channel), may be null
  double* pre_out;     // FWD: pre-activations [M][s_pad] (may be null)
  double* z_out;       // FWD: activated jets, null for the output layer
  double* dbuf;        // REV: in = pre-activations, out = adjoints
  const double* Dk;    // PHA: adjoints of this layer
  double* partA;       // PHA: [mtiles][n_pts_pad] partial (J v) per point
  int n_pts_pad;
  const int* skip;     // PCG done flag (kernel returns immediately when set)
  unsigned lap_mask;   // FWD/REV: coordinates summed into the second-derivative channel
};

// Output head of the interior ("head") rows, SURVEY 8f #3.  With o the output
// channels (value, d_1..d_d, Lambda_S):
//   metric row   F = coef . o + alpha_p u      (alpha_p = 3 kappa ubar_p^2, ubar at theta_bar)
//   residual row R = coef . o + kappa u^3 + off
// Poisson: coef = e_Lambda, kappa = 0; heat: coef = e_{d_t} - e_Lambda (S = {x});
// nonlinear Poisson: coef = e_Lambda, kappa = -1 (problems.py:161-385).
constexpr int kMaxC = 16;
struct Head {
  double coef[kMaxC];
  double kappa;
};

struct PhbArgs {
  const double* D;     // [>=M rows][s_pad]
  const double* Z;     // [>=N rows][s_pad]
  const double* cvec;  // per padded point cotangent
  int M, N;            // n_k, n_{k-1}
  int64_t s_pad;
  int64_t int_cols;    // interior columns (nib*PB*C)
  int C;               // interior channels
  int nib;
  int ktiles_total;    // s_pad / 16
  int ktiles_per_split;
  int64_t off;         // parameter offset of W_k
  double* part;        // [G][p]
  int64_t p;
  const int* skip;
};

struct FormJArgs {
  const double* const* Z;   // per layer input jets
  const double* const* D;   // per layer adjoints
  const int* n_in;
  const int* n_out;
  const int64_t* off;       // W_k offset in the parameter vector
  int64_t s_pad, int_cols;
  int C, nib, n_int;
  int blk0;                 // first point block of this chunk (padded point order)
  int blk_stride;           // CTA x takes block blk0 + x * blk_stride (0 = 1; > 1 only with no_store)
  double* Jt;               // [16 * blocks][ldj], row = padded point within the chunk
  int64_t ldj;
  // optional (INT8 sketch, ngd_ozaki.cu two-sided scaling):
  //   cmax: running maxima of |J| per parameter (column) as ordered bit patterns (RED.MAX.U64; NaN /
  //         inf order above every finite value), accumulated over all chunks in a first pass;
  //   rmax: per chunk row (point), the maximum of |J(r, k)| 2^cexp[k] as a "log-bit" pattern
  //         bits(|J|) + cexp[k] 2^52 (signed RED.MAX; LLONG_MAX = non-finite);
  //   no_store: the first pass computes the maxima only (over a strided sample of the point blocks)
  unsigned long long* cmax;
  long long* rmax;
  const int* cexp;
  int no_store;
};

// FP64 DMMA GEMM (ngd_gemm.cu): C(m, n) = alpha sum_k A(m, k) B(k, n) [* row_scale(m)] + beta C(m, n),
// C column-major (ldc).  K-major operand: A(m, k) = p[m * ld + k]; MN-major: A(m, k) = p[k * ld + m].
// TMA needs 16-byte aligned bases and even leading dimensions (gemm_operand_ok).
struct GemmOperand {
  const double* p;
  int64_t ld;
  bool kmaj;
};
struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n, kstages, splits, kps;
  double alpha, beta;
  double* C;
  int64_t ldc;
  const double* row_scale;
  double* part;  // split-K partials [splits][N][M]
};
struct GemmPlan {
  int bm, bn;  // CTA tile: 128 x 128 or 256 x 64
  int tiles_m, tiles_n, kstages, splits, kps;
  size_t work_bytes;
};
bool gemm_operand_ok(const GemmOperand& o, int MN, int K);
GemmPlan gemm_plan(int M, int N, int K);
cudaError_t dgemm(int M, int N, int K, double alpha, const GemmOperand& A, const GemmOperand& B, double beta,
                  double* C, int64_t ldc, const double* row_scale, double* work, size_t work_bytes, cudaStream_t st);
double gemm_flops_total();

// FP64-exact GEMM on the INT8 tensor cores, Ozaki scheme II (ngd_ozaki.cu): residues of the
// row / column scaled operands modulo kOzMods moduli, one tcgen05 kind::i8 GEMM per modulus,
// CRT reconstruction.  Residue blocks are [kOzMods][rows][ld] int8 (ld a multiple of 16);
// product residues [splits][kOzMods][N][ldo] (column-major).
constexpr int kOzMods = 16;
constexpr int kOzNonFinite = -0x40000000;  // exponent flag of a row / column with a NaN or inf
// "log-bit" pattern of |x| 2^g for maxima of prescaled values: (bits(|x|) >> 1) + g 2^51 -- monotone
// in |x| 2^g, no overflow for |g| <= 2000; LLONG_MAX flags NaN / inf; values below kOzLogEmpty mean
// "no entry" (the RED.MAX start value is memset to 0x80 bytes)
constexpr long long kOzLogEmpty = -(3ll << 61);
__device__ __forceinline__ long long oz_logbits(double x, int g) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(x));
  if (b >= 0x7ff0000000000000ull || g == kOzNonFinite) return 0x7fffffffffffffffll;
  if (b == 0) return kOzLogEmpty - 1;
  g = g < -2000 ? -2000 : (g > 2000 ? 2000 : g);
  return (long long)(b >> 1) + ((long long)g << 51);
}
extern int g_oz_pair;  // option "i8_pair" (process-wide): CTA-pair INT8 GEMM (1) or one CTA per tile (0)
constexpr int kOzMaxKSplit = 130944;  // K per split: 128 * 128 * K < 2^31
int oz_bits(int64_t K);               // integer width t of the scaled operands for inner length K
int oz_splits(int64_t K);
double oz_i8_ops_total();
double oz_conv_elems_total();
cudaError_t oz_exps(const unsigned long long* maxbits, int n, int t, int* exps, cudaStream_t st);
cudaError_t oz_exps_log(const long long* logmax, int n, int t, int* exps, cudaStream_t st);
// residues of A(r, k) = A[r lda + k] scaled by 2^(exps[r] + colsign colexp[k]) (colexp optional; with
// have_exps false the row exponents are computed first from the column-prescaled row maxima)
cudaError_t oz_rows(const double* A, int64_t lda, int rows, int K, int t, int8_t* out, int64_t ldo, int64_t plane,
                    int* exps, bool have_exps, cudaStream_t st, const int* colexp = nullptr, int colsign = 1);
// plane pitch of a residue block: rounded to 256 B plus an odd multiple of 256 B, so the 16 moduli
// planes written together do not alias onto the same memory channels (power-of-two plane strides
// made the residue writes 4-5x slower than the HBM write bandwidth)
inline int64_t oz_plane(int64_t rows, int64_t ld) { return (rows * ld + 255) / 256 * 256 + 37 * 256; }
// a_mn: A stored MN-major (A(m, k) = A[k lda + m] per plane), else K-major (A[m lda + k])
// a_nrb > 0: A is blocked ([row block][column block][128][128] per plane, oz_rows_blocked; pair kernel)
cudaError_t oz_i8gemm(const int8_t* A, int64_t lda, int64_t planeA, bool a_mn, int M, const int8_t* B, int64_t ldb,
                      int64_t planeB, int N, int K, int8_t* res, int64_t ldo, int64_t planeO, cudaStream_t st,
                      int a_nrb = 0, int a_ncb = 0);
// residues of J'(r, k) = rint(J 2^(rexp[r] + cexp[k])) in 128 x 128 blocks (zero past rows / K)
cudaError_t oz_rows_blocked(const double* A, int64_t lda, int rows, int K, int nrb, int ncb, const int* rexp,
                            const int* cexp, int8_t* out, int64_t plane, cudaStream_t st);
cudaError_t oz_crt(const int8_t* res, int64_t ldo, int64_t planeO, int M, int N, int splits, const int* ea,
                   const int* eb, const double* row_w, double alpha, double beta, double* C, int64_t ldc,
                   cudaStream_t st);
cudaError_t gemv_rows(const double* G, int64_t n, const double* x, double* y, const int* skip, cudaStream_t st);

constexpr int kMaxLayers = 8;
struct PhaAll {
  JetArgs L[kMaxLayers];      // per layer, interior segment settings
  int tile_start[kMaxLayers + 1];
  int mtiles[kMaxLayers];
  int n_layers, nib, nbb;
  int64_t int_cols;
};
struct PhbAll {
  PhbArgs L[kMaxLayers];          // per layer (ktiles_per_split set per layer)
  int tile_start[kMaxLayers + 1];  // flat CTA offsets: layer l owns tiles_m*tiles_n*G_l CTAs
  int tiles_n[kMaxLayers], tiles_m[kMaxLayers], G[kMaxLayers];
  int n_layers;
  int thin[kMaxLayers];  // phb2: layer whose tiles are thin (N <= 16 or M <= 16): paired with heavy work
};
// fixed-order reduction plan of the phase-B partials: param range of layer l uses G[l] splits
struct RedPlan {
  int64_t start[kMaxLayers + 1];
  int G[kMaxLayers];
  int n_layers;
};
struct PackAll {  // entries: forward W_l (+ bias row) and, for the reverse sweep, W_{l+1}^T (no bias)
  double* dst[2 * kMaxLayers];
  int Mp[2 * kMaxLayers], Kp[2 * kMaxLayers], n_out[2 * kMaxLayers], n_in[2 * kMaxLayers];
  int trans[2 * kMaxLayers];       // 1: dst = W^T (W is n_out x n_in), no bias row
  int64_t woff[2 * kMaxLayers], boff[2 * kMaxLayers];
  int64_t start[2 * kMaxLayers + 1];  // element offsets (packed matrix [+ bias row] per entry)
  int n_layers;                       // number of entries
};

cudaError_t jet_gemm(int C, int mode, const JetArgs& a, int nblocks, int mtiles, cudaStream_t st);
cudaError_t jet_gemm_both(int C, int mode, const JetArgs& a, int nib, int nbb, int64_t int_cols, int mtiles,
                          cudaStream_t st);
cudaError_t pha_all(int C, const PhaAll& a, cudaStream_t st);
// pipelined phase B (ngd_phb2.cu): TMA producer + MMA warps; tensor maps cached per context
struct Phb2Maps {
  CUtensorMap d[kMaxLayers];  // D_l: [M rows][s_pad], box 64 x 16
  CUtensorMap z[kMaxLayers];  // Zin_l: [N rows][s_pad]
};
struct Phb2Cache {  // host-side: re-encoded when a layer's buffers or shape change
  Phb2Maps maps;
  const double* kd[kMaxLayers] = {};
  const double* kz[kMaxLayers] = {};
  int km[kMaxLayers] = {}, kn[kMaxLayers] = {};
  int64_t ks[kMaxLayers] = {};
};
cudaError_t phase_b2_all_layers(const PhbAll& a, Phb2Cache& cache, cudaStream_t st);
// phase A of the wide layers on the DMMA GEMM core (ngd_phag.cu): items (layer, n-tile, m-tile),
// T = V_l Zin_l on 128 x 128 tiles (K = n_{l-1}), epilogue <D_l, T + vb_l> per column and 64-row half
struct PhagArgs {
  int n_heavy;
  int M[kMaxLayers], Kp[kMaxLayers];  // n_l, n_{l-1} padded to 16
  int tiles_m[kMaxLayers];            // 128-row m tiles of heavy layer h
  int item_start[kMaxLayers + 1];     // items of the heavy layers before h
  int slot0[kMaxLayers];              // first column-partial row of layer h (2 per m tile)
  int tiles_n;                        // 128-column tiles of s_pad
  int64_t s_pad;
  const double* vbias[kMaxLayers];    // vb_l (packed v, value channel only)
  const double* dptr[kMaxLayers];     // D_l [M rows][s_pad]
  double* colpart;                    // [slots][s_pad] per-column partials <D_l[rows], (V Zin)[rows]>
  int int_units, C;                   // interior channel runs (nib * C), channels
  const int* skip;
};
struct PhagMaps {
  CUtensorMap v[kMaxLayers];  // packed V_l [Mp rows][Kp], box 16 x 128 (K-major A)
  CUtensorMap z[kMaxLayers];  // Zin_l [Kp rows][s_pad], box 16 x 16 (MN-major B)
  CUtensorMap d[kMaxLayers];  // D_l [M rows][s_pad], box 16 x 128 (epilogue operand)
};
struct PhagCache {
  PhagMaps maps;
  const double* src_v[kMaxLayers] = {};  // set by the caller
  const double* src_z[kMaxLayers] = {};
  const double* src_d[kMaxLayers] = {};
  int mp[kMaxLayers] = {};               // packed rows of V_l
  int64_t s_pad = 0;
  const double* kv[kMaxLayers] = {};     // encoded keys
  const double* kz[kMaxLayers] = {};
  const double* kd[kMaxLayers] = {};
  int64_t ks[kMaxLayers] = {};
};
cudaError_t phase_a_gemm(const PhagArgs& a, PhagCache& cache, cudaStream_t st);
// extra phase-A terms of reduce_pha_cols: the wide layers' column partials (ngd_phag.cu) and the
// output layer from its precontracted rows G[k][pt] (out_contract)
struct PhaCols {
  const double* colpart = nullptr;  // [cslots][s_pad]
  int cslots = 0;
  const double* gout = nullptr;     // [kout][n_pts_pad], null: output layer in the partA rows
  int kout = 0;
  const double* vout = nullptr;     // v of W_L (packed row 0), vbout: v of b_L
  const double* vbout = nullptr;
  const double* dseed = nullptr;    // D_L (value channel column per point)
};
// cot[pt] = w[pt] * (sum of partA rows + column partials of the point's channel columns + output layer)
void reduce_pha_cols(const double* partA, int rows, const Geom& gm, const PhaCols& rc, const double* w, double* cot,
                     const int* done, cudaStream_t st);
// output layer (M = 1) precontracted: G[k][pt] = sum_c D_L(pt, c) Zin_L[k](pt, c), the W_L block of J_pt
void out_contract(const double* zin, const double* dseed, int K, const Geom& gm, double* G, cudaStream_t st);
// its phase B: part[g][off + k] = sum_{pt in split g} cot[pt] G[k][pt], part[g][off + K] = sum cot[pt] D_L(pt, value)
constexpr int kOutSplits = 148;
void out_phase_b(const double* G, const double* dseed, int K, const Geom& gm, const double* cot, double* part, int64_t p,
                 int64_t off, int splits, const int* done, cudaStream_t st);
// phase B of the wide layers on the DMMA GEMM core (ngd_phbg.cu): items (split, heavy layer, tile)
struct PhbgArgs {
  int n_heavy;                         // layers handled here (both sides >= 128)
  int M[kMaxLayers], N[kMaxLayers];    // n_l, n_{l-1} of heavy layer h
  int tiles_n[kMaxLayers];             // 128-wide n tiles of heavy layer h
  int item_start[kMaxLayers + 1];      // tiles of the heavy layers before h (one split)
  int64_t off[kMaxLayers];             // W_l offset in the parameter vector
  int G, kstages, kps;                 // K splits, 16-column stages, stages per split
  const double* cvec;                  // per padded point cotangent
  int int_units, C, nib;               // interior stages (nib * C), channels, interior point blocks
  double* part;                        // [G][p] partials (flat parameter layout)
  int64_t p;
  const int* skip;
};
struct PhbgMaps {
  CUtensorMap d[kMaxLayers];  // D_l [M rows][s_pad], box 16 x 128
  CUtensorMap z[kMaxLayers];  // Zin_l [N rows][s_pad]
};
struct PhbgCache {
  PhbgMaps maps;
  const double* src_d[kMaxLayers] = {};  // set by the caller: the heavy layers' operands
  const double* src_z[kMaxLayers] = {};
  int64_t s_pad = 0;
  const double* kd[kMaxLayers] = {};
  const double* kz[kMaxLayers] = {};
  int km[kMaxLayers] = {}, kn[kMaxLayers] = {};
  int64_t ks[kMaxLayers] = {};
};
bool phbg_layer_ok(int M, int N);
int phbg_splits(int tiles, int kstages);
cudaError_t phase_b_gemm(const PhbgArgs& a, PhbgCache& cache, cudaStream_t st);
int phb2_ctas_per_sm();
int phb2_thin_only_ctas();
void pack_all(const PackAll& a, const double* src, const int* skip, cudaStream_t st);
cudaError_t form_j(const FormJArgs& a, int nblocks, int n_layers, int max_nin, int max_nout, cudaStream_t st);

void pack(double* dst, int Mp, int Kp, const double* src, int64_t off, int n_out, int n_in, int trans,
          const int* skip, cudaStream_t st);
void init_point_data(double* zin1, double* dlast, Geom gm, const double* x_int, const double* x_bnd,
                     cudaStream_t st);
int nblocks_for(int64_t n);
void dot(const double* x, const double* y, int64_t n, double* partials, unsigned int* counter, double* out,
         const int* done, cudaStream_t st);
// residual / loss of the stack; when dseed != null also the metric rows F and the output
// adjoint seeds (linearisation); alpha_bar != null supplies a frozen per-point 3 kappa ubar^2
void residual_loss(const double* pre_last, Geom gm, const Head& hd, const double* w_res, const double* off,
                   const double* alpha_bar, double* F, double* R, double* cot, double* dseed, double* partials,
                   unsigned int* counter, double* loss_sum, cudaStream_t st);
void frozen_alpha(const double* pre_last, Geom gm, double kappa, double* alpha, cudaStream_t st);
void reduce_pha(const double* partA, int rows, int n_pts_pad, const double* w, double* cot, const int* done,
                cudaStream_t st);
void reduce_splits(const double* part, const RedPlan& rp, int64_t p, double mu, const double* mu_p, const double* v,
                   double* out, const int* done, cudaStream_t st);
void add_scaled(double* out, double mu, const double* mu_p, const double* v, int64_t n, const int* done,
                cudaStream_t st);
int precond_blocks(int64_t p);
// counters: two consecutive unsigned counters (utv combine, uc dot)
cudaError_t precond_apply(const PrecondArgs* pa, int64_t p, int ell, const double* v, double* out, double* part,
                          double* cprime, unsigned* counters, const int* done, PcgState* pcg, int first,
                          double* partials, cudaStream_t st);
void pcg_init(PcgState* s, double rel_tol, cudaStream_t st);
void pcg_start(const double* b, double* x, double* r, int64_t p, cudaStream_t st);
void pcg_first_dir(const double* z, double* d, int64_t p, PcgState* s, cudaStream_t st);
void pcg_ad(const double* part, const RedPlan& rp, int64_t p, const double* mu_p, const double* d, double* ad,
            PcgState* s, int ad_ready, double* partials, unsigned* counter, cudaStream_t st);
void pcg_update(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s, int recompute,
                double* partials, unsigned* counter, cudaStream_t st);
void pcg_true_res(const double* b, const double* ax, double* r, int64_t p, PcgState* s, int count, int final_pass,
                  double* partials, unsigned* counter, cudaStream_t st);
void pcg_dir_pack(const double* z, double* d, const PackAll& pk, PcgState* s, int* host_flag, cudaStream_t st);
void pcg_dir(const double* z, double* d, int64_t p, PcgState* s, int* host_flag, cudaStream_t st);
void theta_minus(const double* a, double alpha, const double* b, double* out, int64_t n, cudaStream_t st);
void scale_cols_sqrt(double* J, int64_t p, int64_t R, const double* w, cudaStream_t st);
void symmetrize_upper(double* G, int64_t n, int64_t ld, cudaStream_t st);
void add_shift(double* y, const double* omega, int64_t n, const double* fro2, double* shift_out, cudaStream_t st);
void eig_from_sv(const double* s, int ell, const double* shift, double* eig, cudaStream_t st);
void triu(double* a, int n, int lda, cudaStream_t st);
void transpose(const double* src, int64_t lds, int rows, int cols, double* dst, int64_t ldd, cudaStream_t st);
void info_combine(int* info, const int* info2, int offset, cudaStream_t st);
void shift_diag(double* w, int n, double coef, cudaStream_t st);
void fill_gaussian(double* out, int64_t n, uint64_t seed, cudaStream_t st);
int jsvd_block_supported(int ell);
// FP32 pre-sweeps + FP64 finish (V in place in global memory for ell > ~310): cluster size, 0 if unsupported
int jsvd_mixed_supported(int ell);
bool chol_supported(int n);
// X R = A in place (A p x n col-major, R n x n upper col-major); work: trsm_work(n) bytes
size_t trsm_work(int n);
bool trsm_supported(int n);
cudaError_t trsm_right_upper(double* A, int64_t lda, int64_t p, const double* R, int ldr, int n, double* work,
                             cudaStream_t st);
cudaError_t chol_upper(double* A, int n, int lda, int* info, cudaStream_t st);
// cluster Cholesky (8 CTAs), n <= 512; flag: one int of device scratch
bool chol_cluster_supported(int n);
cudaError_t chol_upper_cluster(double* A, int n, int lda, int* info, int* flag, cudaStream_t st);
cudaError_t jacobi_svd_block(const double* A, int ell, int lda, double* U, int ldu, double* sigma, int* info,
                             cudaStream_t st);
// FP64 block Jacobi on X = A^T starting from V = V0 (orthonormal): sigma / U of A^T V0 rotated
cudaError_t jacobi_svd_block_from(const double* A, int ell, int lda, double* V0, int ldv, double* U, int ldu,
                                  double* sigma, int* info, cudaStream_t st);
// FP32 pre-sweeps of the block Jacobi on A^T: V (ell x ell, unsorted, only near-orthogonal) out
cudaError_t jacobi_presweep_f32(const double* A, int ell, int lda, double* V, int ldv, double coupling, int* info,
                                cudaStream_t st);
void h1_terms(const double* pre_last, Geom gm, const double* exact, double* num, double* den, cudaStream_t st);
void gather_points(const double* padded, double* compact, Geom gm, cudaStream_t st);
void scatter_points(const double* compact, double* padded, Geom gm, cudaStream_t st);

}  // namespace ngd
