// HBM-bound helper kernels: packing, residual/loss, deterministic reductions,
// Nystrom preconditioner apply, fused PCG vector updates, Philox Gaussians.
// All reductions use a fixed work assignment and a fixed combination order, so
// results are bitwise reproducible run to run.
#include <cstdlib>
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

int g_pdl = [] {  // NGD_PDL=0: plain stream-ordered launches (A/B); option "pdl" at run time
  const char* e = getenv("NGD_PDL");
  return e ? atoi(e) : 1;
}();

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

void init_point_data(double* zin1, double* dlast, Geom gm, const double* x_int, const double* x_bnd,
                     cudaStream_t st) {
  const int npts = gm.n_pts_pad();
  const int grid = std::max(1, std::min((npts + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  input_jets_kernel<<<grid, 256, 0, st>>>(zin1, gm.s_pad, gm, x_int, x_bnd);
  probe_after(K_VEC, st);
  (void)dlast;  // output adjoint seeds are written per linearisation (residual_kernel)
}

// ----------------------- deterministic two-stage sums ------------------------
// Each launch uses grid = nblocks_for(n) blocks; block b sums a fixed strided set,
// the last block to finish sums the block partials in index order.
int nblocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184)); }

template <typename T, typename F>
__device__ __forceinline__ void finish_sum(double v, double* partials, unsigned int* counter, T* out, F&& post) {
  __shared__ double sh[kThreads / 32];
  __shared__ bool last;
  const double bs = block_sum(v, sh);
#ifndef NGD_PDL_NO_TAIL_TRIGGER
  // this block's streaming work is done: once every block got here, the next kernel of the chain
  // may launch (it still waits for this grid's completion) and overlaps the last-block combine
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {  // block-uniform: the whole last block combines the partials (fixed order)
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += __ldcg(&partials[i]);
    const double tot = block_sum(s, sh);
    if (threadIdx.x == 0) {
      *counter = 0;
      post(tot, out);
    }
  }
}

// sum_{g<G} part[g*stride + i] in index order, with 8 loads in flight (latency hiding
// without changing the deterministic summation order)
template <typename P>
__device__ __forceinline__ double sum_partials(P part, int G, int64_t stride, int64_t i) {
  double s = 0.0;
  int g = 0;
  for (; g + 8 <= G; g += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(&part[(int64_t)(g + u) * stride + i]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; g < G; ++g) s += __ldcg(&part[(int64_t)g * stride + i]);
  return s;
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

// residual / loss of the stack (problems.py:92-96, 161-385).  Head rows (interior
// points, C channels o): F = coef.o + alpha u, R = coef.o + kappa u^3 + off with
// alpha = 3 kappa ubar^2 (ubar = u at theta unless alpha_bar supplies a frozen
// theta_bar value); value rows: F = u, R = u + off.  loss = 0.5 sum w_res R^2,
// cot = w_res R (gradient cotangent: the residual's Jacobian is the metric row
// frozen at theta).  When linearising, dseed receives dF/d(output jets).
__global__ void residual_kernel(const double* pre_last, Geom gm, Head hd, const double* w, const double* off,
                                const double* alpha_bar, double* F, double* R, double* cot, double* dseed,
                                double* partials, unsigned int* slot, double* loss_sum) {
  const int npts = gm.n_pts_pad();
  double v = 0.0;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npts; pt += gridDim.x * blockDim.x) {
    double f, r;
    if (pt < gm.nib * PB) {
      double lin = 0.0;
      for (int c = 0; c < gm.C; ++c) {
        const double cc = hd.coef[c];
        if (cc != 0.0) lin = fma(cc, pre_last[col_int(pt, c, gm.C)], lin);
      }
      f = lin;
      r = lin;
      double alpha = 0.0;
      if (hd.kappa != 0.0) {
        const double u = pre_last[col_int(pt, 0, gm.C)];
        alpha = alpha_bar ? alpha_bar[pt] : 3.0 * hd.kappa * u * u;
        f = fma(alpha, u, lin);
        r = fma(hd.kappa * u * u, u, lin);
      }
      if (dseed)
        for (int c = 0; c < gm.C; ++c) dseed[col_int(pt, c, gm.C)] = hd.coef[c] + (c == 0 ? alpha : 0.0);
    } else {
      const int64_t col = gm.int_cols() + (pt - gm.nib * PB);
      f = r = pre_last[col];
      if (dseed) dseed[col] = 1.0;
    }
    r += off[pt];
    const double wr = w[pt] * r;
    if (F) F[pt] = f;
    if (R) R[pt] = r;
    if (cot) cot[pt] = wr;
    v = fma(wr, r, v);
  }
  finish_sum(v, partials, slot, loss_sum, [](double s, double* o) { o[0] = s; });
}

void residual_loss(const double* pre_last, Geom gm, const Head& hd, const double* w_res, const double* off,
                   const double* alpha_bar, double* F, double* R, double* cot, double* dseed, double* partials,
                   unsigned int* slot, double* loss_sum, cudaStream_t st) {
  probe_before(K_VEC, st);
  residual_kernel<<<nblocks_for(gm.n_pts_pad()), kThreads, 0, st>>>(pre_last, gm, hd, w_res, off, alpha_bar, F, R,
                                                                    cot, dseed, partials, slot, loss_sum);
  probe_after(K_VEC, st);
}

// alpha[pt] = 3 kappa ubar^2 from a forward pass at theta_bar (problems.py:364-368: ubar frozen)
__global__ void frozen_alpha_kernel(const double* pre_last, Geom gm, double kappa, double* alpha) {
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < gm.nib * PB; pt += gridDim.x * blockDim.x) {
    const double u = pre_last[col_int(pt, 0, gm.C)];
    alpha[pt] = 3.0 * kappa * u * u;
  }
}

void frozen_alpha(const double* pre_last, Geom gm, double kappa, double* alpha, cudaStream_t st) {
  probe_before(K_VEC, st);
  frozen_alpha_kernel<<<std::max(1, std::min((gm.nib * PB + 255) / 256, 1184)), 256, 0, st>>>(pre_last, gm, kappa,
                                                                                              alpha);
  probe_after(K_VEC, st);
}

// phase A reduction: s[pt] = sum over (layer, mtile) partials in fixed order; cot = w * s
__global__ void reduce_pha_kernel(const double* partA, int rows, int n_pts_pad, const double* w, double* cot,
                                  const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < n_pts_pad; pt += gridDim.x * blockDim.x) {
    const double s = sum_partials(partA, rows, n_pts_pad, pt);
    cot[pt] = w ? w[pt] * s : s;
  }
}

void reduce_pha(const double* partA, int rows, int n_pts_pad, const double* w, double* cot, const int* done,
                cudaStream_t st) {
  const int grid = std::max(1, std::min((n_pts_pad + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  launch_pdl(reduce_pha_kernel, dim3(grid), dim3(256), 0, st, partA, rows, n_pts_pad, w, cot, done);
  probe_after(K_VEC, st);
}

// as reduce_pha, plus (PhaCols) the wide layers' per-column partials (ngd_phag.cu: the point's C
// channel columns -- one on the boundary -- of every column-partial row) and the output layer from its
// precontracted rows (out_contract), all in fixed order
__global__ void reduce_pha_cols_kernel(const double* partA, int rows, Geom gm, PhaCols rc, const double* w, double* cot,
                                       const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  const int npp = gm.n_pts_pad(), int_pts = gm.nib * PB, C = gm.C;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npp; pt += gridDim.x * blockDim.x) {
    double s = sum_partials(partA, rows, npp, pt);
    const bool interior = pt < int_pts;
    const int64_t col0 = interior ? (int64_t)(pt / PB) * PB * C + (pt % PB) : (int64_t)int_pts * C + (pt - int_pts);
    const int nch = interior ? C : 1;
    for (int q = 0; q < rc.cslots; ++q) {
      const double* row = rc.colpart + (int64_t)q * gm.s_pad + col0;
      double r = 0.0;
      for (int c = 0; c < nch; ++c) r += __ldcg(&row[(int64_t)c * PB]);
      s += r;
    }
    if (rc.gout) {  // <v_{W_L}, J_pt[W_L]> + v_{b_L} D_L(pt, value)
      double r = rc.vbout[0] * rc.dseed[col0];
      int k = 0;
#pragma unroll 1
      for (; k + 8 <= rc.kout; k += 8) {
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) g[u] = __ldcs(&rc.gout[(int64_t)(k + u) * npp + pt]);
#pragma unroll
        for (int u = 0; u < 8; ++u) r = fma(rc.vout[k + u], g[u], r);
      }
      for (; k < rc.kout; ++k) r = fma(rc.vout[k], __ldcs(&rc.gout[(int64_t)k * npp + pt]), r);
      s += r;
    }
    cot[pt] = w ? w[pt] * s : s;
  }
}

void reduce_pha_cols(const double* partA, int rows, const Geom& gm, const PhaCols& rc, const double* w, double* cot,
                     const int* done, cudaStream_t st) {
  const int npp = gm.n_pts_pad();
  const int grid = std::max(1, std::min((npp + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  launch_pdl(reduce_pha_cols_kernel, dim3(grid), dim3(256), 0, st, partA, rows, gm, rc, w, cot, done);
  probe_after(K_VEC, st);
}

// G[k][pt] = sum_c D_L(pt, c) Zin_L[k](pt, c): the W_L block of the Jacobian row of point pt (the output
// layer has one unit, so its row is K numbers instead of the C K of its input jets)
__global__ void out_contract_kernel(const double* __restrict__ zin, const double* __restrict__ dseed, Geom gm,
                                    double* __restrict__ G) {
  const int npp = gm.n_pts_pad(), int_pts = gm.nib * PB, C = gm.C;
  const int k = blockIdx.y;
  const double* zrow = zin + (int64_t)k * gm.s_pad;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < npp; pt += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (pt < int_pts) {
      const int64_t col0 = (int64_t)(pt / PB) * PB * C + (pt % PB);
      for (int c = 0; c < C; ++c) s = fma(dseed[col0 + (int64_t)c * PB], zrow[col0 + (int64_t)c * PB], s);
    } else {
      const int64_t col = (int64_t)int_pts * C + (pt - int_pts);
      s = dseed[col] * zrow[col];
    }
    G[(int64_t)k * npp + pt] = s;
  }
}

void out_contract(const double* zin, const double* dseed, int K, const Geom& gm, double* G, cudaStream_t st) {
  const int npp = gm.n_pts_pad();
  probe_before(K_PHA, st);
  out_contract_kernel<<<dim3(std::max(1, std::min((npp + 255) / 256, 64)), K), 256, 0, st>>>(zin, dseed, gm, G);
  probe_after(K_PHA, st);
}

// phase B of the output layer from G: block g sums its point range [g P, (g + 1) P) for every k (warp
// w takes rows w, w + 8, ..; lanes 32 consecutive points; fixed xor tree), plus the bias entry
__global__ void __launch_bounds__(256) out_phase_b_kernel(const double* __restrict__ G, const double* __restrict__ dseed,
                                                          int K, Geom gm, const double* __restrict__ cot, double* part,
                                                          int64_t p, int64_t off, int per, const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  const int npp = gm.n_pts_pad(), int_pts = gm.nib * PB, C = gm.C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pt0 = blockIdx.x * per, pt1 = min(npp, pt0 + per);
  double* out = part + (int64_t)blockIdx.x * p + off;
  for (int k0 = 0; k0 < K; k0 += 256) {
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
    double bacc = 0.0;
    for (int pt = pt0 + lane; pt < pt1; pt += 32) {
      const double cv = cot[pt];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = k0 + warp + 8 * i;
        if (k < K) acc[i] = fma(cv, __ldcs(&G[(int64_t)k * npp + pt]), acc[i]);
      }
      if (k0 == 0 && warp == 0) {
        const int64_t col0 = pt < int_pts ? (int64_t)(pt / PB) * PB * C + (pt % PB) : (int64_t)int_pts * C + (pt - int_pts);
        bacc = fma(cv, dseed[col0], bacc);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double v = acc[i];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int k = k0 + warp + 8 * i;
      if (lane == 0 && k < K) out[k] = v;
    }
    if (k0 == 0 && warp == 0) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) bacc += __shfl_xor_sync(0xffffffffu, bacc, o);
      if (lane == 0) out[K] = bacc;
    }
  }
}

void out_phase_b(const double* G, const double* dseed, int K, const Geom& gm, const double* cot, double* part, int64_t p,
                 int64_t off, int splits, const int* done, cudaStream_t st) {
  const int npp = gm.n_pts_pad();
  const int per = ((npp + splits - 1) / splits + 31) & ~31;
  probe_before(K_PHB, st);
  launch_pdl(out_phase_b_kernel, dim3(splits), dim3(256), 0, st, G, dseed, K, gm, cot, part, p, off, per, done);
  probe_after(K_PHB, st);
}

// phase B reduction: out[i] = sum_g part[g][i] (+ mu * v[i])
__device__ __forceinline__ int plan_G(const RedPlan& rp, int64_t i) {
  int l = 0;
  while (l + 1 < rp.n_layers && i >= rp.start[l + 1]) ++l;
  return rp.G[l];
}

__global__ void reduce_splits_kernel(const double* part, RedPlan rp, int64_t p, double mu, const double* mu_p,
                                     const double* v, double* out, const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  if (mu_p) mu = *mu_p;
  // four lanes per element (lane q sums g = q, q+4, ...; fixed-order combine), as pcg_ad_kernel
  const int q = threadIdx.x & 3;
  for (int64_t i0 = (int64_t)blockIdx.x * (blockDim.x / 4); i0 < p; i0 += (int64_t)gridDim.x * (blockDim.x / 4)) {
    const int64_t i = i0 + (threadIdx.x >> 2);
    double a = 0.0;
    if (i < p) {
      const int G = plan_G(rp, i);
      int g = q;
      for (; g + 12 < G; g += 16) {
        const double x0 = __ldcg(&part[(int64_t)g * p + i]), x1 = __ldcg(&part[(int64_t)(g + 4) * p + i]);
        const double x2 = __ldcg(&part[(int64_t)(g + 8) * p + i]), x3 = __ldcg(&part[(int64_t)(g + 12) * p + i]);
        a += x0;
        a += x1;
        a += x2;
        a += x3;
      }
      for (; g < G; g += 4) a += __ldcg(&part[(int64_t)g * p + i]);
    }
    const double a1 = __shfl_xor_sync(0xffffffffu, a, 1);
    const double a2 = __shfl_xor_sync(0xffffffffu, a, 2);
    const double a3 = __shfl_xor_sync(0xffffffffu, a, 3);
    if (q == 0 && i < p) {
      double s = (a + a1) + (a2 + a3);
      if (v) s = fma(mu, v[i], s);
      out[i] = s;
    }
  }
}

void reduce_splits(const double* part, const RedPlan& rp, int64_t p, double mu, const double* mu_p, const double* v,
                   double* out, const int* done, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((p + 63) / 64, 148 * 8));
  probe_before(K_VEC, st);
  launch_pdl(reduce_splits_kernel, dim3(grid), dim3(256), 0, st, part, rp, p, mu, mu_p, v, out, done);
  probe_after(K_VEC, st);
}

// out += mu * v
__global__ void add_scaled_kernel(double* out, double mu, const double* mu_p, const double* v, int64_t n,
                                  const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  if (mu_p) mu = *mu_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fma(mu, v[i], out[i]);
}
void add_scaled(double* out, double mu, const double* mu_p, const double* v, int64_t n, const int* done,
                cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  probe_before(K_VEC, st);
  launch_pdl(add_scaled_kernel, dim3(grid), dim3(256), 0, st, out, mu, mu_p, v, n, done);
  probe_after(K_VEC, st);
}

// per-point H1 error terms at the interior points (problems.py:104-119):
// num = (u - ue)^2 + |grad u - ge|^2, den = ue^2 + |ge|^2; exact = [ue, ge_1..ge_d] per point
__global__ void h1_terms_kernel(const double* pre_last, Geom gm, const double* exact, double* num, double* den) {
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < gm.nib * PB; pt += gridDim.x * blockDim.x) {
    double nu = 0.0, de = 0.0;
    if (pt < gm.n_int) {
      const double* ex = exact + (int64_t)pt * (gm.d + 1);
      const double e0 = pre_last[col_int(pt, 0, gm.C)] - ex[0];
      nu = e0 * e0;
      de = ex[0] * ex[0];
      for (int i = 0; i < gm.d; ++i) {
        const double ei = pre_last[col_int(pt, 1 + i, gm.C)] - ex[1 + i];
        nu = fma(ei, ei, nu);
        de = fma(ex[1 + i], ex[1 + i], de);
      }
    }
    num[pt] = nu;
    den[pt] = de;
  }
}
void h1_terms(const double* pre_last, Geom gm, const double* exact, double* num, double* den, cudaStream_t st) {
  probe_before(K_VEC, st);
  h1_terms_kernel<<<std::max(1, std::min((gm.nib * PB + 255) / 256, 1184)), 256, 0, st>>>(pre_last, gm, exact, num,
                                                                                         den);
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
// U column-major p x ell (each basis vector contiguous).
// Pass 1 (utv_kernel): one block per basis vector: c'_j = (scale/(lam_j+mu) - 1) * <u_j, v>.
// Pass 2 (uc_kernel): out = v + U c', optionally with the PCG dot r.z fused in.
__global__ void __launch_bounds__(kThreads) utv_kernel(const PrecondArgs* pa, int64_t p, int ell, const double* v,
                                                       double* cprime, const int* done) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  __shared__ double sh[kThreads / 32];
  const int j = blockIdx.x;
  const double* u = pa->U + (int64_t)j * p;
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t i = threadIdx.x;
  for (; i + 7 * kThreads < p; i += 8 * kThreads) {  // 16 loads in flight per thread
    double uu[8], vv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uu[q] = u[i + q * kThreads];
      vv[q] = v[i + q * kThreads];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(uu[q], vv[q], acc[q]);
  }
  for (; i < p; i += kThreads) acc[0] = fma(u[i], v[i], acc[0]);  // (a runtime acc index would go to local memory)
  const double tot =
      block_sum(((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7])), sh);
  if (threadIdx.x == 0) {
    const double mu = pa->mu;
    const double* eig = pa->eig;
    cprime[j] = ((eig[ell - 1] + mu) / (eig[j] + mu) - 1.0) * tot;
  }
}

// out[i] = v[i] + sum_j U[j p + i] c'_j.  Block = 64 rows x 4 column groups (fixed-order
// combine in shared memory).  With pcg != null the dot r.z (r = v, z = out) is finished by
// the last block: first pass rz = r.z; otherwise beta = r.z_new / rz, rz = r.z_new (krylov.py:75-78).
__global__ void __launch_bounds__(kThreads) uc_kernel(const PrecondArgs* pa, int64_t p, int ell, const double* cprime,
                                                      const double* v, double* out, const int* done, PcgState* pcg,
                                                      int first, double* partials, unsigned* counter) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (done && *done) return;
  extern __shared__ double cs[];  // [ell] c' then [8][32] partial rows
  double* part = cs + ell;
  for (int j = threadIdx.x; j < ell; j += blockDim.x) cs[j] = cprime[j];
  __syncthreads();
  constexpr int kRows = 32, kGroups = kThreads / kRows;
  const int rl = threadIdx.x & (kRows - 1), grp = threadIdx.x / kRows;
  const int64_t i = (int64_t)blockIdx.x * kRows + rl;
  double s = 0.0;
  if (i < p && ell > 0) {
    const double* U = pa->U;
    const int per = (ell + kGroups - 1) / kGroups;
    const int j0 = grp * per, j1 = min(ell, j0 + per);
    int j = j0;
    double s2 = 0.0;
    for (; j + 16 <= j1; j += 16) {  // 16 loads in flight, two interleaved chains
      double u[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) u[q] = U[(int64_t)(j + q) * p + i];
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        s = fma(u[q], cs[j + q], s);
        s2 = fma(u[q + 1], cs[j + q + 1], s2);
      }
    }
    for (; j < j1; ++j) s = fma(U[(int64_t)j * p + i], cs[j], s);
    s += s2;
  }
  part[grp * kRows + rl] = s;
  __syncthreads();
  double rz = 0.0;
  if (grp == 0 && i < p) {
    double t = 0.0;
#pragma unroll
    for (int g2 = 0; g2 < kGroups; ++g2) t += part[g2 * kRows + rl];
    const double z = v[i] + t;
    out[i] = z;
    rz = v[i] * z;
  }
  if (!pcg) return;
  finish_sum(rz, partials, counter, pcg, [first](double sum, PcgState* st) {
    st->rz_new = sum;
    if (first) {
      st->rz = sum;
    } else {
      st->beta = sum / st->rz;
      st->rz = sum;
    }
  });
}

int precond_blocks(int64_t p) { return (int)std::max<int64_t>(1, (p + 31) / 32); }

cudaError_t precond_apply(const PrecondArgs* pa, int64_t p, int ell, const double* v, double* out, double* part,
                          double* cprime, unsigned* counters, const int* done, PcgState* pcg, int first,
                          double* partials, cudaStream_t st) {
  (void)part;
  if (ell > 0) {
    probe_before(K_PRECOND, st);
    launch_pdl(utv_kernel, dim3(ell), dim3(kThreads), 0, st, pa, p, ell, v, cprime, done);
    probe_after(K_PRECOND, st);
  }
  const int grid = precond_blocks(p);
  probe_before(K_PRECOND, st);
  launch_pdl(uc_kernel, dim3(grid), dim3(kThreads), sizeof(double) * (std::max(ell, 1) + kThreads), st, pa, p, ell, cprime, v, out, done, pcg,
                                                                              first, partials, counters + 1);
  probe_after(K_PRECOND, st);
  return cudaGetLastError();
}

// ------------------------------ PCG device state ----------------------------
// krylov.py:24-88, scalar logic executed on the device (last block of the
// fused reductions) so a whole solve runs without host round trips.
__global__ void pcg_init_kernel(PcgState* s, double rel_tol) {
  s->norm_b = sqrt(s->bb);
  s->tol = rel_tol;
  s->iterations = 0;
  s->it = 0;
  s->matvecs = 0;
  s->breakdown = 0;
  s->converged = 0;
  s->beta = 0.0;
  s->done = (s->norm_b == 0.0) ? 2 : 0;  // 2 = zero right-hand side
}

// x = 0, r = b
__global__ void pcg_start_kernel(const double* b, double* x, double* r, int64_t p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = 0.0;
    r[i] = b[i];
  }
}

// d = z
__global__ void pcg_first_dir_kernel(const double* z, double* d, int64_t p, PcgState* s) {
  if (s->done) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = z[i];
}

// ad = sum_g part[g] + mu d ; dad = d.ad ; breakdown test and alpha (krylov.py:59-66).  Four lanes per
// element split the split-K partial sum (lane q takes g = q, q+4, ...; combined in fixed order), so
// the dependent L2 loads of the G partials are spread over 4x more threads.
constexpr int kAdLanes = 8;  // lanes per element: G = 74 split partials (C2) -> <= 10 loads per lane
constexpr int kAdPerBlock = kThreads / kAdLanes;
__global__ void pcg_ad_kernel(const double* part, RedPlan rp, int64_t p, const double* mu_p, const double* d,
                              double* ad, PcgState* s, int ad_ready, double* partials, unsigned* counter) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (s->done) return;
  const double mu = *mu_p;
  const int q = threadIdx.x & (kAdLanes - 1);
  double v = 0.0;
  for (int64_t i0 = (int64_t)blockIdx.x * kAdPerBlock; i0 < p; i0 += (int64_t)gridDim.x * kAdPerBlock) {
    const int64_t i = i0 + (threadIdx.x / kAdLanes);
    if (ad_ready) {
      if (q == 0 && i < p) v = fma(d[i], ad[i], v);
      continue;
    }
    double a = 0.0;
    if (i < p) {
      const int G = plan_G(rp, i);
      int g = q;
      for (; g + 3 * kAdLanes < G; g += 4 * kAdLanes) {
        const double x0 = __ldcg(&part[(int64_t)g * p + i]);
        const double x1 = __ldcg(&part[(int64_t)(g + kAdLanes) * p + i]);
        const double x2 = __ldcg(&part[(int64_t)(g + 2 * kAdLanes) * p + i]);
        const double x3 = __ldcg(&part[(int64_t)(g + 3 * kAdLanes) * p + i]);
        a += x0;
        a += x1;
        a += x2;
        a += x3;
      }
      for (; g < G; g += kAdLanes) a += __ldcg(&part[(int64_t)g * p + i]);
    }
#pragma unroll
    for (int o = 1; o < kAdLanes; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);  // fixed xor tree
    if (q == 0 && i < p) {
      const double tot = fma(mu, d[i], a);
      ad[i] = tot;
      v = fma(d[i], tot, v);
    }
  }
  finish_sum(v, partials, counter, s, [](double sum, PcgState* st) {
    st->dad = sum;
    const int it = ++st->it;
    st->matvecs += 1;
    if (sum <= 0.0) {
      st->breakdown = 1;
      st->done = 1;
      return;
    }
    st->alpha = st->rz / sum;
    st->iterations = it;
  });
}

// x += alpha d ; r -= alpha ad ; rr = r.r ; convergence test (krylov.py:66-74)
__global__ void pcg_update_kernel(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s,
                                  int recompute, double* partials, unsigned* counter) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (s->done) return;
  const double a = s->alpha;
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = x[i] + a * d[i];
    if (!recompute) {
      const double ri = r[i] - a * ad[i];
      r[i] = ri;
      v = fma(ri, ri, v);
    }
  }
  if (recompute) return;
  finish_sum(v, partials, counter, s, [](double sum, PcgState* st) {
    st->rr = sum;
    st->rel = sqrt(sum) / st->norm_b;
    if (st->rel <= st->tol) st->done = 3;
  });
}

// r = b - Ax (true residual, krylov.py:69-71 and 83-85) ; rr ; test
__global__ void pcg_true_res_kernel(const double* b, const double* ax, double* r, int64_t p, PcgState* s,
                                    int count_matvec, int final_pass, double* partials, unsigned* counter) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (!final_pass && s->done) return;
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = b[i] - ax[i];
    r[i] = ri;
    v = fma(ri, ri, v);
  }
  finish_sum(v, partials, counter, s, [count_matvec, final_pass](double sum, PcgState* st) {
    st->rr = sum;
    if (count_matvec) st->matvecs += 1;
    st->rel = sqrt(sum) / st->norm_b;
    if (final_pass) {
      if (st->done != 2) {
        st->matvecs += 1;
        st->converged = (!st->breakdown) && (st->rel <= st->tol);
      }
    } else if (st->rel <= st->tol) {
      st->done = 3;
    }
  });
}

// d = z + beta d  (krylov.py:79-81)
__global__ void pcg_dir_kernel(const double* z, double* d, int64_t p, PcgState* s, int* host_flag) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  // last kernel of an iteration: publish the done flag to pinned host memory (zero-copy, no memcpy
  // or event between graph replays)
  if (host_flag && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<volatile int*>(host_flag) = s->done;
  if (s->done) return;
  const double beta = s->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = z[i] + beta * d[i];
}

// d = z + beta d fused with the packing of d into the forward layer matrices of the next matvec
// (pack_all_kernel's index space: every parameter is read and written by exactly one thread)
__global__ void pcg_dir_pack_kernel(const double* z, double* d, PackAll a, PcgState* s, int* host_flag) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (host_flag && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<volatile int*>(host_flag) = s->done;
  if (s->done) return;
  const double beta = s->beta;
  const int64_t n = a.start[a.n_layers];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < a.n_layers && k >= a.start[l + 1]) ++l;
    const int64_t kk = k - a.start[l];
    const int64_t mat = (int64_t)a.Mp[l] * a.Kp[l];
    int64_t i = -1;
    if (kk < mat) {
      const int m = (int)(kk / a.Kp[l]), c = (int)(kk % a.Kp[l]);
      if (m < a.n_out[l] && c < a.n_in[l]) i = a.woff[l] + (int64_t)m * a.n_in[l] + c;
    } else {
      const int m = (int)(kk - mat);
      if (m < a.n_out[l]) i = a.boff[l] + m;
    }
    double v = 0.0;
    if (i >= 0) {
      v = z[i] + beta * d[i];
      d[i] = v;
    }
    a.dst[l][kk] = v;
  }
}

static int vgrid(int64_t p) { return (int)std::max<int64_t>(1, std::min<int64_t>((p + 255) / 256, 148 * 8)); }
static int rgrid(int64_t p) { return nblocks_for(p); }

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
void pcg_ad(const double* part, const RedPlan& rp, int64_t p, const double* mu_p, const double* d, double* ad,
            PcgState* s, int ad_ready, double* partials, unsigned* counter, cudaStream_t st) {
  probe_before(K_VEC, st);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((p + kAdPerBlock - 1) / kAdPerBlock, 1184));
  launch_pdl(pcg_ad_kernel, dim3(grid), dim3(kThreads), 0, st, part, rp, p, mu_p, d, ad, s, ad_ready, partials, counter);
  probe_after(K_VEC, st);
}
void pcg_update(double* x, double* r, const double* d, const double* ad, int64_t p, PcgState* s, int recompute,
                double* partials, unsigned* counter, cudaStream_t st) {
  probe_before(K_VEC, st);
  launch_pdl(pcg_update_kernel, dim3(rgrid(p)), dim3(kThreads), 0, st, x, r, d, ad, p, s, recompute, partials, counter);
  probe_after(K_VEC, st);
}
void pcg_true_res(const double* b, const double* ax, double* r, int64_t p, PcgState* s, int count, int final_pass,
                  double* partials, unsigned* counter, cudaStream_t st) {
  probe_before(K_VEC, st);
  launch_pdl(pcg_true_res_kernel, dim3(rgrid(p)), dim3(kThreads), 0, st, b, ax, r, p, s, count, final_pass, partials, counter);
  probe_after(K_VEC, st);
}
void pcg_dir_pack(const double* z, double* d, const PackAll& pk, PcgState* s, int* host_flag, cudaStream_t st) {
  const int64_t n = pk.start[pk.n_layers];
  probe_before(K_VEC, st);
  launch_pdl(pcg_dir_pack_kernel, dim3(vgrid(n)), dim3(256), 0, st, z, d, pk, s, host_flag);
  probe_after(K_VEC, st);
}
void pcg_dir(const double* z, double* d, int64_t p, PcgState* s, int* host_flag, cudaStream_t st) {
  probe_before(K_VEC, st);
  launch_pdl(pcg_dir_kernel, dim3(vgrid(p)), dim3(256), 0, st, z, d, p, s, host_flag);
  probe_after(K_VEC, st);
}

// pack all layers' weight matrices (+ bias rows) of a parameter-layout vector in one launch
__global__ void pack_all_kernel(PackAll a, const double* src, const int* skip) {
  if (skip && *skip) return;
  const int64_t n = a.start[a.n_layers];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < a.n_layers && i >= a.start[l + 1]) ++l;
    const int64_t k = i - a.start[l];
    const int64_t mat = (int64_t)a.Mp[l] * a.Kp[l];
    double v = 0.0;
    if (k < mat) {
      const int m = (int)(k / a.Kp[l]), c = (int)(k % a.Kp[l]);
      if (a.trans[l]) {
        if (m < a.n_in[l] && c < a.n_out[l]) v = src[a.woff[l] + (int64_t)c * a.n_in[l] + m];
      } else if (m < a.n_out[l] && c < a.n_in[l]) {
        v = src[a.woff[l] + (int64_t)m * a.n_in[l] + c];
      }
    } else {
      const int m = (int)(k - mat);
      if (m < a.n_out[l]) v = src[a.boff[l] + m];
    }
    a.dst[l][k] = v;
  }
}
void pack_all(const PackAll& a, const double* src, const int* skip, cudaStream_t st) {
  const int64_t n = a.start[a.n_layers];
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  probe_before(K_PACK, st);
  pack_all_kernel<<<grid, 256, 0, st>>>(a, src, skip);
  probe_after(K_PACK, st);
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

// Jt (p x R column-major, one Jacobian row per column) columns scaled by sqrt(w)
__global__ void scale_cols_sqrt_kernel(double* J, int64_t p, int64_t R, const double* w) {
  const int64_t n = p * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    J[i] *= sqrt(w[i / p]);
}
void scale_cols_sqrt(double* J, int64_t p, int64_t R, const double* w, cudaStream_t st) {
  probe_before(K_VEC, st);
  scale_cols_sqrt_kernel<<<vgrid(p * R), 256, 0, st>>>(J, p, R, w);
  probe_after(K_VEC, st);
}


// lower triangle <- upper triangle
__global__ void symmetrize_upper_kernel(double* G, int64_t n, int64_t ld) {
  const int64_t tot = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;  // element (i, j), column-major
    if (i > j) G[j * ld + i] = G[i * ld + j];
  }
}
void symmetrize_upper(double* G, int64_t n, int64_t ld, cudaStream_t st) {
  probe_before(K_VEC, st);
  symmetrize_upper_kernel<<<vgrid(n * n), 256, 0, st>>>(G, n, ld);
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

// dst(j, i) = src(i, j): rows x cols column-major (lds) -> cols x rows column-major (ldd); the
// off-diagonal panel of the blocked Cholesky (ell > 512) is solved as a right triangular system
__global__ void transpose_kernel(const double* src, int64_t lds, int rows, int cols, double* dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int i = i0 + threadIdx.x, j = j0 + y;
    if (i < rows && j < cols) tile[y][threadIdx.x] = src[(int64_t)j * lds + i];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int j = j0 + threadIdx.x, i = i0 + y;
    if (i < rows && j < cols) dst[(int64_t)i * ldd + j] = tile[threadIdx.x][y];
  }
}
void transpose(const double* src, int64_t lds, int rows, int cols, double* dst, int64_t ldd, cudaStream_t st) {
  probe_before(K_VEC, st);
  transpose_kernel<<<dim3((rows + 31) / 32, (cols + 31) / 32), dim3(32, 8), 0, st>>>(src, lds, rows, cols, dst, ldd);
  probe_after(K_VEC, st);
}

// LAPACK potrf status of a blocked factor: the first failing pivot of either diagonal block
__global__ void info_combine_kernel(int* info, const int* info2, int offset) {
  if (*info == 0 && *info2 != 0) *info = *info2 + offset;
}
void info_combine(int* info, const int* info2, int offset, cudaStream_t st) {
  probe_before(K_VEC, st);
  info_combine_kernel<<<1, 1, 0, st>>>(info, info2, offset);
  probe_after(K_VEC, st);
}

}  // namespace ngd
