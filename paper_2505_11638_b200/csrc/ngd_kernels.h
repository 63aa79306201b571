// Internal launch interface of the CUDA kernels (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ngd_common.cuh"

namespace ngd {

// kernel classes for launch accounting / probe timing (ngd_probe.cu)
enum KernelKind { K_FWD = 1, K_REV = 2, K_PHA = 3, K_PHB = 4, K_FORMJ = 5, K_PRECOND = 6, K_VEC = 7, K_PACK = 8 };
void probe_before(int kind, cudaStream_t st);
void probe_after(int kind, cudaStream_t st);

// device-side PCG scalars (krylov.py:24-88)
struct PcgState {
  double bb, norm_b, tol, rz, rz_new, dad, alpha, rr, rel;
  int iterations, matvecs, breakdown, converged, done;
};

enum JetMode { FWD = 0, REV = 1, PHA = 2 };

struct JetArgs {
  const double* A;     // packed operand, row-major [Mp][Kp] (zero padded)
  int Kp;              // padded K (multiple of 16)
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
  int q0;                   // first real point of this chunk (interior first, then boundary)
  double* Jt;               // [R][ldj]
  int64_t ldj;
};

cudaError_t jet_gemm(int C, int mode, const JetArgs& a, int nblocks, int mtiles, cudaStream_t st);
cudaError_t phase_b(const PhbArgs& a, int splits, cudaStream_t st);
cudaError_t form_j(const FormJArgs& a, int R, int n_layers, cudaStream_t st);

void pack(double* dst, int Mp, int Kp, const double* src, int64_t off, int n_out, int n_in, int trans,
          const int* skip, cudaStream_t st);
void init_point_data(double* zin1, double* dlast, Geom gm, const double* x_int, const double* x_bnd,
                     cudaStream_t st);
int nblocks_for(int64_t n);
void dot(const double* x, const double* y, int64_t n, double* partials, unsigned int* counter, double* out,
         const int* done, cudaStream_t st);
void residual_loss(const double* pre_last, Geom gm, const double* w, const double* off, double* F, double* cot,
                   double* partials, unsigned int* counter, double* loss_sum, cudaStream_t st);
void reduce_pha(const double* partA, int rows, int n_pts_pad, const double* w, double* cot, const int* done,
                cudaStream_t st);
void reduce_splits(const double* part, int G, int64_t p, double mu, const double* v, double* out, const int* done,
                   cudaStream_t st);
void add_scaled(double* out, double mu, const double* v, int64_t n, const int* done, cudaStream_t st);
int precond_blocks(int64_t p);
cudaError_t precond_apply(const double* U, int64_t p, int ell, const double* eig, const double* mu_p, double mu_v,
                          const double* v, double* out, double* part, double* cprime, const int* done,
                          cudaStream_t st);
void pcg_init(PcgState* s, double rel_tol, cudaStream_t st);
void pcg_start(const double* b, double* x, double* r, int64_t p, cudaStream_t st);
void pcg_first_dir(const double* z, double* d, int64_t p, PcgState* s, cudaStream_t st);
void pcg_alpha(PcgState* s, int it, cudaStream_t st);
void pcg_update(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s, int recompute,
                cudaStream_t st);
void pcg_true_res(const double* b, const double* ax, double* r, int64_t p, PcgState* s, int count, int final_pass,
                  cudaStream_t st);
void pcg_check(PcgState* s, cudaStream_t st);
void pcg_dir(const double* z, double* d, int64_t p, PcgState* s, cudaStream_t st);
void pcg_final(PcgState* s, cudaStream_t st);
void theta_minus(const double* a, double alpha, const double* b, double* out, int64_t n, cudaStream_t st);
void scale_rows(double* S, int64_t R, int ell, const double* w, cudaStream_t st);
void add_shift(double* y, const double* omega, int64_t n, const double* fro2, double* shift_out, cudaStream_t st);
void eig_from_sv(const double* s, int ell, const double* shift, double* eig, cudaStream_t st);
void triu(double* a, int n, int lda, cudaStream_t st);
void shift_diag(double* w, int n, double coef, cudaStream_t st);
void fill_gaussian(double* out, int64_t n, uint64_t seed, cudaStream_t st);
void gather_points(const double* padded, double* compact, Geom gm, cudaStream_t st);
void scatter_points(const double* compact, double* padded, Geom gm, cudaStream_t st);

}  // namespace ngd
