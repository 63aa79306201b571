// HBM-bound helper kernels: packing, residual/loss, deterministic reductions,
// Nystrom preconditioner apply, fused PCG vector updates, Philox Gaussians.
// All reductions use a fixed work assignment and a fixed combination order, so
// results are bitwise reproducible run to run.
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

// ------------------------------- packing -----------------------------------
// dst[m][k] (Mp x Kp, zero padded) = W[m][k] (trans=0) or W[k][m] (trans=1),
// W = src[off ...] row-major (n_out x n_in)  (model.py:41-51 layout)
__global__ void pack_kernel(double* dst, int Mp, int Kp, const double* src, int64_t off, int n_out, int n_in,
                            int trans, const int* skip) {
  if (skip && *skip) return;
  const int64_t n = (int64_t)Mp * Kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / Kp), k = (int)(i % Kp);
    double v = 0.0;
    if (!trans) {
      if (m < n_out && k < n_in) v = src[off + (int64_t)m * n_in + k];
    } else {
      if (m < n_in && k < n_out) v = src[off + (int64_t)k * n_in + m];
    }
    dst[i] = v;
  }
}

void pack(double* dst, int Mp, int Kp, const double* src, int64_t off, int n_out, int n_in, int trans,
          const int* skip, cudaStream_t st) {
  const int64_t n = (int64_t)Mp * Kp;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  probe_before(K_PACK, st);
  pack_kernel<<<grid, 256, 0, st>>>(dst, Mp, Kp, src, off, n_out, n_in, trans, skip);
  probe_after(K_PACK, st);
}

// --------------------- input jets and output adjoint seeds ------------------
// Zin_1: value channel = x, gradient channel i = e_i, Laplacian channel = 0.
__global__ void input_jets_kernel(double* z, int64_t s_pad, Geom gm, const double* x_int, const double* x_bnd) {
  const int npts = gm.n_pts_pad();
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npts; pt += gridDim.x * blockDim.x) {
    if (pt < gm.nib * PB) {
      const bool real = pt < gm.n_int;
      for (int i = 0; i < gm.d; ++i) {
        double* row = z + (int64_t)i * s_pad;
        for (int c = 0; c < gm.C; ++c) {
          double v = 0.0;
          if (c == 0) v = real ? x_int[(int64_t)pt * gm.d + i] : 0.0;
          else if (c == 1 + i) v = 1.0;
          row[col_int(pt, c, gm.C)] = v;
        }
      }
    } else {
      const int s = pt - gm.nib * PB;
      const bool real = s < gm.n_bnd;
      for (int i = 0; i < gm.d; ++i)
        z[(int64_t)i * s_pad + gm.int_cols() + s] = real ? x_bnd[(int64_t)s * gm.d + i] : 0.0;
    }
  }
}

// D_{L+1}: dF/d(output pre-activation jets) = indicator of the metric channel
// (Laplacian channel on interior points, value channel on boundary points).
__global__ void seed_adjoint_kernel(double* d, Geom gm) {
  const int npts = gm.n_pts_pad();
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npts; pt += gridDim.x * blockDim.x) {
    if (pt < gm.nib * PB) {
      for (int c = 0; c < gm.C; ++c) d[col_int(pt, c, gm.C)] = (c == gm.C - 1) ? 1.0 : 0.0;
    } else {
      d[gm.int_cols() + (pt - gm.nib * PB)] = 1.0;
    }
  }
}

void init_point_data(double* zin1, double* dlast, Geom gm, const double* x_int, const double* x_bnd,
                     cudaStream_t st) {
  const int npts = gm.n_pts_pad();
  const int grid = std::max(1, std::min((npts + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  input_jets_kernel<<<grid, 256, 0, st>>>(zin1, gm.s_pad, gm, x_int, x_bnd);
  probe_after(K_VEC, st);
  probe_before(K_VEC, st);
  seed_adjoint_kernel<<<grid, 256, 0, st>>>(dlast, gm);
  probe_after(K_VEC, st);
}

// ----------------------- deterministic two-stage sums ------------------------
// Each launch uses grid = nblocks_for(n) blocks; block b sums a fixed strided set,
// the last block to finish sums the block partials in index order.
int nblocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 2047) / 2048, 296)); }

template <typename F>
__device__ __forceinline__ void finish_sum(double v, double* partials, unsigned int* counter, double* out, F&& post) {
  __shared__ double sh[kThreads / 32];
  __shared__ bool last;
  const double bs = block_sum(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    volatile double* vp = partials;
    for (unsigned i = 0; i < gridDim.x; ++i) s += vp[i];
    *counter = 0;
    post(s, out);
  }
}

// out[0] = sum_i x[i]*y[i]   (skip if *done)
__global__ void dot_kernel(const double* x, const double* y, int64_t n, double* partials, unsigned int* slot, double* out,
                           const int* done) {
  if (done && *done) return;
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v = fma(x[i], y[i], v);
  finish_sum(v, partials, slot, out, [](double s, double* o) { o[0] = s; });
}

void dot(const double* x, const double* y, int64_t n, double* partials, unsigned int* slot, double* out, const int* done,
         cudaStream_t st) {
  probe_before(K_VEC, st);
  dot_kernel<<<nblocks_for(n), kThreads, 0, st>>>(x, y, n, partials, slot, out, done);
  probe_after(K_VEC, st);
}

// residual / loss: F = metric channel of the output-layer pre-activations;
// R = F + off;  loss = 0.5 * sum w R R  (problems.py:92-96, 161-166); cot = w R
__global__ void residual_kernel(const double* pre_last, Geom gm, const double* w, const double* off, double* F,
                                double* cot, double* partials, unsigned int* slot, double* loss_sum) {
  const int npts = gm.n_pts_pad();
  double v = 0.0;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npts; pt += gridDim.x * blockDim.x) {
    const int64_t col = pt < gm.nib * PB ? col_int(pt, gm.C - 1, gm.C) : gm.int_cols() + (pt - gm.nib * PB);
    const double f = pre_last[col];
    const double r = f + off[pt];
    const double wr = w[pt] * r;
    if (F) F[pt] = f;
    if (cot) cot[pt] = wr;
    v = fma(wr, r, v);
  }
  finish_sum(v, partials, slot, loss_sum, [](double s, double* o) { o[0] = s; });
}

void residual_loss(const double* pre_last, Geom gm, const double* w, const double* off, double* F, double* cot,
                   double* partials, unsigned int* slot, double* loss_sum, cudaStream_t st) {
  probe_before(K_VEC, st);
  probe_before(K_VEC, st);
  residual_kernel<<<nblocks_for(gm.n_pts_pad()), kThreads, 0, st>>>(pre_last, gm, w, off, F, cot, partials, slot,
                                                                    loss_sum);
  probe_after(K_VEC, st);
  probe_after(K_VEC, st);
}

// phase A reduction: s[pt] = sum over (layer, mtile) partials in fixed order; cot = w * s
__global__ void reduce_pha_kernel(const double* partA, int rows, int n_pts_pad, const double* w, double* cot,
                                  const int* done) {
  if (done && *done) return;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < n_pts_pad; pt += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += partA[(int64_t)r * n_pts_pad + pt];
    cot[pt] = w ? w[pt] * s : s;
  }
}

void reduce_pha(const double* partA, int rows, int n_pts_pad, const double* w, double* cot, const int* done,
                cudaStream_t st) {
  const int grid = std::max(1, std::min((n_pts_pad + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  reduce_pha_kernel<<<grid, 256, 0, st>>>(partA, rows, n_pts_pad, w, cot, done);
  probe_after(K_VEC, st);
}

// phase B reduction: out[i] = sum_g part[g][i] (+ mu * v[i])
__global__ void reduce_splits_kernel(const double* part, int G, int64_t p, double mu, const double* v, double* out,
                                     const int* done) {
  if (done && *done) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += part[(int64_t)g * p + i];
    if (v) s = fma(mu, v[i], s);
    out[i] = s;
  }
}

void reduce_splits(const double* part, int G, int64_t p, double mu, const double* v, double* out, const int* done,
                   cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((p + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  reduce_splits_kernel<<<grid, 256, 0, st>>>(part, G, p, mu, v, out, done);
  probe_after(K_VEC, st);
}

// out += mu * v
__global__ void add_scaled_kernel(double* out, double mu, const double* v, int64_t n, const int* done) {
  if (done && *done) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fma(mu, v[i], out[i]);
}
void add_scaled(double* out, double mu, const double* v, int64_t n, const int* done, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  add_scaled_kernel<<<grid, 256, 0, st>>>(out, mu, v, n, done);
  probe_after(K_VEC, st);
}

// padded point order (interior blocks, then boundary blocks) <-> compact order
__global__ void gather_points_kernel(const double* padded, double* compact, Geom gm, int dir) {
  const int n = gm.n_int + gm.n_bnd;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int pt = q < gm.n_int ? q : gm.nib * PB + (q - gm.n_int);
    if (dir == 0) compact[q] = padded[pt];
    else compact[pt] = padded[q];  // scatter: 'compact' is the padded destination
  }
}
void gather_points(const double* padded, double* compact, Geom gm, cudaStream_t st) {
  const int n = gm.n_int + gm.n_bnd;
  probe_before(K_VEC, st);
  gather_points_kernel<<<std::max(1, std::min((n + 255) / 256, 1184)), 256, 0, st>>>(padded, compact, gm, 0);
  probe_after(K_VEC, st);
}
void scatter_points(const double* compact, double* padded, Geom gm, cudaStream_t st) {
  cudaMemsetAsync(padded, 0, sizeof(double) * gm.n_pts_pad(), st);
  const int n = gm.n_int + gm.n_bnd;
  probe_before(K_VEC, st);
  gather_points_kernel<<<std::max(1, std::min((n + 255) / 256, 1184)), 256, 0, st>>>(compact, padded, gm, 1);
  probe_after(K_VEC, st);
}

// ------------------------- Nystrom preconditioner ---------------------------
// P^{-1} v = U((scale*inv - 1) o (U^T v)) + v   (sketch.py:101-112, fused into 2 passes over U)
// U row-major p x ell.  Pass 1: per row-block partial U^T v.
template <int JCH>
__global__ void __launch_bounds__(kThreads) utv_kernel(const double* U, int64_t p, int ell, const double* v,
                                                       int64_t rows_per_blk, double* part, const int* done) {
  if (done && *done) return;
  __shared__ double sh[JCH * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[JCH];
#pragma unroll
  for (int j = 0; j < JCH; ++j) acc[j] = 0.0;
  const int64_t r0 = blockIdx.x * rows_per_blk, r1 = std::min<int64_t>(p, r0 + rows_per_blk);
  for (int64_t i = r0 + warp; i < r1; i += kThreads / 32) {
    const double vi = v[i];
    const double* row = U + i * ell;
#pragma unroll
    for (int j = 0; j < JCH; ++j) {
      const int col = j * 32 + lane;
      if (col < ell) acc[j] = fma(row[col], vi, acc[j]);
    }
  }
  // fixed-order cross-warp accumulation (warp 0 first)
  for (int w = 0; w < kThreads / 32; ++w) {
    if (warp == w) {
#pragma unroll
      for (int j = 0; j < JCH; ++j) sh[j * 32 + lane] = (w == 0 ? 0.0 : sh[j * 32 + lane]) + acc[j];
    }
    __syncthreads();
  }
  for (int col = threadIdx.x; col < ell; col += kThreads) part[(int64_t)blockIdx.x * ell + col] = sh[col];
}

// combine partials and scale:  c'[j] = (scale*inv[j] - 1) * sum_b part[b][j]
__global__ void utv_combine_kernel(const double* part, int nblk, int ell, const double* eig, const double* mu_p,
                                   double mu_v, double* cprime, const int* done) {
  if (done && *done) return;
  const double mu = mu_p ? *mu_p : mu_v;
  const double scale = eig[ell - 1] + mu;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ell; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * ell + j];
    cprime[j] = (scale / (eig[j] + mu) - 1.0) * s;
  }
}

// out[i] = v[i] + sum_j U[i][j] c'[j]; one warp per row.  Optionally also
// accumulates r.z for PCG (rz_out) -- fused dot.
__global__ void __launch_bounds__(kThreads) uc_kernel(const double* U, int64_t p, int ell, const double* cprime,
                                                      const double* v, double* out, const int* done) {
  if (done && *done) return;
  extern __shared__ double cs[];
  for (int j = threadIdx.x; j < ell; j += blockDim.x) cs[j] = cprime[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * (kThreads / 32) + warp; i < p; i += (int64_t)gridDim.x * (kThreads / 32)) {
    const double* row = U + i * ell;
    double s = 0.0;
    for (int j = lane; j < ell; j += 32) s = fma(row[j], cs[j], s);
    s = warp_sum(s);
    if (lane == 0) out[i] = v[i] + s;
  }
}

int precond_blocks(int64_t p) { return (int)std::max<int64_t>(1, std::min<int64_t>((p + 63) / 64, 296)); }

cudaError_t precond_apply(const double* U, int64_t p, int ell, const double* eig, const double* mu_p, double mu_v,
                          const double* v, double* out, double* part, double* cprime, const int* done,
                          cudaStream_t st) {
  const int nblk = precond_blocks(p);
  const int64_t rpb = (p + nblk - 1) / nblk;
  const int jch = (ell + 31) / 32;
#define NGD_UTV(J) (probe_before(K_PRECOND, st), utv_kernel<J><<<nblk, kThreads, 0, st>>>(U, p, ell, v, rpb, part, done), probe_after(K_PRECOND, st))
  if (jch <= 1) NGD_UTV(1);
  else if (jch <= 2) NGD_UTV(2);
  else if (jch <= 4) NGD_UTV(4);
  else if (jch <= 8) NGD_UTV(8);
  else if (jch <= 16) NGD_UTV(16);
  else if (jch <= 24) NGD_UTV(24);
  else if (jch <= 32) NGD_UTV(32);
  else return cudaErrorInvalidValue;
#undef NGD_UTV
  probe_before(K_PRECOND, st);
  utv_combine_kernel<<<(ell + 255) / 256, 256, 0, st>>>(part, nblk, ell, eig, mu_p, mu_v, cprime, done);
  probe_after(K_PRECOND, st);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((p + 7) / 8, 148 * 8));
  probe_before(K_PRECOND, st);
  uc_kernel<<<grid, kThreads, sizeof(double) * ell, st>>>(U, p, ell, cprime, v, out, done);
  probe_after(K_PRECOND, st);
  return cudaGetLastError();
}

// ------------------------------ PCG device state ----------------------------
// krylov.py:24-88, scalar logic executed by one thread on the device so the
// whole solve runs without host round trips.
__global__ void pcg_init_kernel(PcgState* s, double rel_tol) {
  s->norm_b = sqrt(s->bb);
  s->tol = rel_tol;
  s->iterations = 0;
  s->matvecs = 0;
  s->breakdown = 0;
  s->converged = 0;
  s->done = (s->norm_b == 0.0) ? 2 : 0;  // 2 = zero right-hand side
}

// x = 0, r = b, (z computed by precond afterwards), copy
__global__ void pcg_start_kernel(const double* b, double* x, double* r, int64_t p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = 0.0;
    r[i] = b[i];
  }
}

// d = z ; rz already computed into s->rz_new
__global__ void pcg_first_dir_kernel(const double* z, double* d, int64_t p, PcgState* s) {
  if (s->done) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = z[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) s->rz = s->rz_new;
}

// after A d and dad: breakdown test, alpha  (krylov.py:60-66)
__global__ void pcg_alpha_kernel(PcgState* s, int it) {
  if (s->done) return;
  s->matvecs += 1;
  if (s->dad <= 0.0) {
    s->breakdown = 1;
    s->done = 1;
    return;
  }
  s->alpha = s->rz / s->dad;
  s->iterations = it;
}

// x += alpha d ; r -= alpha Ad (unless this is a recompute iteration)
__global__ void pcg_update_kernel(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s,
                                  int recompute) {
  if (s->done) return;
  const double a = s->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = x[i] + a * d[i];
    if (!recompute) r[i] = r[i] - a * ad[i];
  }
}

// r = b - Ax (true residual recompute, krylov.py:69-71)
__global__ void pcg_true_res_kernel(const double* b, const double* ax, double* r, int64_t p, PcgState* s,
                                    int count_matvec, int final_pass) {
  if (!final_pass && s->done) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - ax[i];
  if (count_matvec && blockIdx.x == 0 && threadIdx.x == 0) s->matvecs += 1;
}

// convergence test on ||r||/||b|| (krylov.py:72-74)
__global__ void pcg_check_kernel(PcgState* s) {
  if (s->done) return;
  const double rel = sqrt(s->rr) / s->norm_b;
  s->rel = rel;
  if (rel <= s->tol) s->done = 3;  // converged by tolerance
}

// beta = r.z_new / rz ; d = z + beta d  (krylov.py:75-81)
__global__ void pcg_dir_kernel(const double* z, double* d, int64_t p, PcgState* s) {
  if (s->done) return;
  const double beta = s->rz_new / s->rz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = z[i] + beta * d[i];
}
__global__ void pcg_rz_roll_kernel(PcgState* s) {
  if (s->done) return;
  s->rz = s->rz_new;
}

// final report (krylov.py:83-88)
__global__ void pcg_final_kernel(PcgState* s) {
  if (s->done == 2) return;  // zero rhs: report stays (0 its, 0 matvecs, converged)
  s->matvecs += 1;
  s->rel = sqrt(s->rr) / s->norm_b;
  s->converged = (!s->breakdown) && (s->rel <= s->tol);
}

static int vgrid(int64_t p) { return (int)std::max<int64_t>(1, std::min<int64_t>((p + 255) / 256, 148 * 8)); }

void pcg_init(PcgState* s, double rel_tol, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_init_kernel<<<1, 1, 0, st>>>(s, rel_tol);
  probe_after(K_VEC, st);
}
void pcg_start(const double* b, double* x, double* r, int64_t p, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_start_kernel<<<vgrid(p), 256, 0, st>>>(b, x, r, p);
  probe_after(K_VEC, st);
}
void pcg_first_dir(const double* z, double* d, int64_t p, PcgState* s, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_first_dir_kernel<<<vgrid(p), 256, 0, st>>>(z, d, p, s);
  probe_after(K_VEC, st);
}
void pcg_alpha(PcgState* s, int it, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_alpha_kernel<<<1, 1, 0, st>>>(s, it);
  probe_after(K_VEC, st);
}
void pcg_update(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s, int recompute,
                cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_update_kernel<<<vgrid(p), 256, 0, st>>>(x, r, d, ad, p, s, recompute);
  probe_after(K_VEC, st);
}
void pcg_true_res(const double* b, const double* ax, double* r, int64_t p, PcgState* s, int count, int final_pass,
                  cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_true_res_kernel<<<vgrid(p), 256, 0, st>>>(b, ax, r, p, s, count, final_pass);
  probe_after(K_VEC, st);
}
void pcg_check(PcgState* s, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_check_kernel<<<1, 1, 0, st>>>(s);
  probe_after(K_VEC, st);
}
void pcg_dir(const double* z, double* d, int64_t p, PcgState* s, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_dir_kernel<<<vgrid(p), 256, 0, st>>>(z, d, p, s);
  probe_after(K_VEC, st);
  probe_before(K_VEC, st);
  pcg_rz_roll_kernel<<<1, 1, 0, st>>>(s);
  probe_after(K_VEC, st);
}
void pcg_final(PcgState* s, cudaStream_t st) {
  probe_before(K_VEC, st);
  pcg_final_kernel<<<1, 1, 0, st>>>(s);
  probe_after(K_VEC, st);
}

// ------------------------------- small maps ---------------------------------
// out = a - alpha * b  (line-search candidate, optim.py:137)
__global__ void axpy_kernel(const double* a, double alpha, const double* b, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - alpha * b[i];
}
void theta_minus(const double* a, double alpha, const double* b, double* out, int64_t n, cudaStream_t st) {
  probe_before(K_VEC, st);
  axpy_kernel<<<vgrid(n), 256, 0, st>>>(a, alpha, b, out, n);
  probe_after(K_VEC, st);
}

// S[q][j] (col-major R x ell) *= w[q]
__global__ void scale_rows_kernel(double* S, int64_t R, int ell, const double* w) {
  const int64_t n = R * ell;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    S[i] *= w[i % R];
}
void scale_rows(double* S, int64_t R, int ell, const double* w, cudaStream_t st) {
  probe_before(K_VEC, st);
  scale_rows_kernel<<<vgrid(R * ell), 256, 0, st>>>(S, R, ell, w);
  probe_after(K_VEC, st);
}

// y += shift * omega where shift = eps * sqrt(*fro2)  (sketch.py:77-78); writes shift
__global__ void shift_kernel(double* y, const double* omega, int64_t n, const double* fro2, double* shift_out) {
  const double shift = 2.220446049250313e-16 * sqrt(*fro2);
  if (blockIdx.x == 0 && threadIdx.x == 0) *shift_out = shift;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = y[i] + shift * omega[i];
}
void add_shift(double* y, const double* omega, int64_t n, const double* fro2, double* shift_out, cudaStream_t st) {
  probe_before(K_VEC, st);
  shift_kernel<<<vgrid(n), 256, 0, st>>>(y, omega, n, fro2, shift_out);
  probe_after(K_VEC, st);
}

// eig = max(s^2 - shift, 0)  (sketch.py:86)
__global__ void eig_kernel(const double* s, int ell, const double* shift, double* eig) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ell; j += gridDim.x * blockDim.x)
    eig[j] = fmax(s[j] * s[j] - *shift, 0.0);
}
void eig_from_sv(const double* s, int ell, const double* shift, double* eig, cudaStream_t st) {
  probe_before(K_VEC, st);
  eig_kernel<<<(ell + 255) / 256, 256, 0, st>>>(s, ell, shift, eig);
  probe_after(K_VEC, st);
}

// W += coef * trace(W) * I  (sCholQR3 shift, ||B||_F^2 = trace(B^T B)); one block
__global__ void shift_diag_kernel(double* w, int n, double coef) {
  __shared__ double sh[kThreads / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += w[(int64_t)i * n + i];
  const double tr = block_sum(v, sh);
  __shared__ double s;
  if (threadIdx.x == 0) s = coef * tr;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[(int64_t)i * n + i] += s;
}
void shift_diag(double* w, int n, double coef, cudaStream_t st) {
  probe_before(K_VEC, st);
  shift_diag_kernel<<<1, kThreads, 0, st>>>(w, n, coef);
  probe_after(K_VEC, st);
}

// zero the strictly-lower triangle of an n x n column-major matrix (potrf leaves garbage there)
__global__ void triu_kernel(double* a, int n, int lda) {
  const int64_t tot = (int64_t)n * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % n), c = (int)(i / n);
    if (r > c) a[(int64_t)c * lda + r] = 0.0;
  }
}
void triu(double* a, int n, int lda, cudaStream_t st) {
  probe_before(K_VEC, st);
  triu_kernel<<<vgrid((int64_t)n * n), 256, 0, st>>>(a, n, lda);
  probe_after(K_VEC, st);
}

// --------------------------- Philox4x32-10 Gaussians ------------------------
__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t (&k)[2]) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
  const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
  const uint32_t n0 = h1 ^ c[1] ^ k[0], n2 = h0 ^ c[3] ^ k[1];
  c[0] = n0; c[1] = l1; c[2] = n2; c[3] = l0;
  k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u;
}

__global__ void gaussian_kernel(double* out, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0x5EEDu, 0u};
    uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
    for (int r = 0; r < 10; ++r) philox_round(c, k);
    const uint64_t a = ((uint64_t)c[0] << 21) ^ (c[1] >> 11);
    const uint64_t b = ((uint64_t)c[2] << 21) ^ (c[3] >> 11);
    const double u1 = ((double)(a & ((1ull << 53) - 1)) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = (double)(b & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    out[2 * i] = rad * cs;
    if (2 * i + 1 < n) out[2 * i + 1] = rad * sn;
  }
}
void fill_gaussian(double* out, int64_t n, uint64_t seed, cudaStream_t st) {
  probe_before(K_VEC, st);
  gaussian_kernel<<<vgrid((n + 1) / 2), 256, 0, st>>>(out, n, seed);
  probe_after(K_VEC, st);
}

}  // namespace ngd
