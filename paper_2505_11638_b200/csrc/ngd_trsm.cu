// Tall-skinny right triangular solve  X R = A  (A: p x n column-major, R: n x n upper,
// X overwrites A) on FP64 tensor cores, for the Nystrom factorisation (n = ell <= 512).
//
// Every Cholesky-QR step of sketch.py:73-86 as restated here (Omega's orthonormalisation,
// B = Y_nu C^{-1}, the three passes of shifted Cholesky-QR3) is a p x ell right solve.
// cuBLAS DTRSM runs these shapes at ~3 TFLOP/s on B200 (tools/blas_shapes.py: 238 us
// for 8577 x 300 vs 62 us for the same-shape DGEMM).  Here:
//   1. diag_inv: the 32 x 32 diagonal blocks of R are inverted (one CTA per block,
//      column-parallel back substitution) -- the only sequential arithmetic;
//   2. trsm: one CTA per 32-row panel of A (resident in shared memory), right-looking over
//      the column blocks:  X_J = T_J inv(R_JJ)  then  T_{>J} -= X_J R[J, >J]  (DMMA); the
//      trailing tiles are independent 8-deep DMMA chains (a left-looking form measured
//      latency-bound on its single long chain per tile).
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

constexpr int TB = 32;        // block size (rows per CTA panel, columns per block)
constexpr int XS = TB + 8;    // smem column stride of the panel: (8 t + g) distinct banks for A frags
constexpr int kTrsmThreads = 256;

// Rinv: nbk blocks of TB x TB (column-major), block J = inv(R_JJ), identity-padded past n
__global__ void __launch_bounds__(TB) diag_inv_kernel(const double* R, int ldr, int n, double* Rinv) {
  __shared__ double T[TB][TB + 1];  // T[i][k] = R_JJ[i][k]
  const int J = blockIdx.x, c = threadIdx.x, c0 = J * TB;
  const int nb = min(TB, n - c0);
  for (int i = 0; i < TB; ++i)
    T[i][c] = (i < nb && c < nb) ? (i <= c ? R[(int64_t)(c0 + c) * ldr + c0 + i] : 0.0) : (i == c ? 1.0 : 0.0);
  __syncthreads();
  // column c of W = inv(T): T W = I, back substitution from row c up
  double w[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) w[i] = 0.0;
#pragma unroll
  for (int i = TB - 1; i >= 0; --i) {
    if (i <= c) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = i + 1; k < TB; ++k)
        if (k <= c) s = fma(-T[i][k], w[k], s);
      w[i] = s / T[i][i];
    }
  }
  double* out = Rinv + (int64_t)J * TB * TB + (int64_t)c * TB;
#pragma unroll
  for (int i = 0; i < TB; ++i) out[i] = w[i];
}

__global__ void __launch_bounds__(kTrsmThreads) trsm_kernel(double* A, int64_t lda, int64_t p, const double* R,
                                                             int ldr, int n, const double* Rinv) {
  extern __shared__ __align__(16) double xs[];  // [nbk * TB columns][XS]: the CTA's 32-row panel of A / X
  const int nbk = (n + TB - 1) / TB;
  const int64_t r0 = (int64_t)blockIdx.x * TB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // panel rows [r0, r0 + 32) of A into shared memory (column-major, zero padded)
  for (int e = tid; e < nbk * TB * TB; e += kTrsmThreads) {
    const int col = e >> 5, rr = e & (TB - 1);
    xs[(size_t)col * XS + rr] = (col < n && r0 + rr < p) ? A[(int64_t)col * lda + r0 + rr] : 0.0;
  }
  __syncthreads();
  // right-looking: X_J = T_J inv(R_JJ), then T_{>J} -= X_J R[J, >J]; every tile of the trailing
  // update is an independent DMMA chain (8 k-steps), so a warp keeps many in flight
  for (int J = 0; J < nbk; ++J) {
    const int c0 = J * TB;
    const double* Ri = Rinv + (size_t)J * TB * TB;
    // 1. solve the block column: warp w -> rows 8 (w & 3), columns 16 (w >> 2) .. +15
    {
      const int tr = 8 * (warp & 3), tc = 16 * (warp >> 2);
      double x[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int k = 0; k < TB; k += 4) {
        const double a = xs[(size_t)(c0 + k + t) * XS + tr + g];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          dmma884(x[h][0], x[h][1], a, __ldg(Ri + (size_t)(tc + 8 * h + g) * TB + k + t));
      }
      __syncthreads();  // every warp has read T_J before it is overwritten with X_J
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = tc + 8 * h + 2 * t + e;
          xs[(size_t)(c0 + cl) * XS + tr + g] = x[h][e];
          if (r0 + tr + g < p && c0 + cl < n) A[(int64_t)(c0 + cl) * lda + r0 + tr + g] = x[h][e];
        }
    }
    __syncthreads();
    // 2. trailing update of the later column blocks: tiles (row tile 0..3, column tile of 8)
    const int ncol = nbk * TB - (c0 + TB);
    if (ncol > 0) {
      const int nct = ncol >> 3;
      // this warp's tiles all share row tile rt = warp & 3 (tile = warp + 8 i): X_J fragments once
      const int rt = warp & 3;
      double av[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) av[u] = -xs[(size_t)(c0 + 4 * u + t) * XS + rt * 8 + g];
      // column tiles ct = (warp >> 2) + 2 i, four at a time: 32 R loads in flight before the DMMAs
      for (int ct0 = warp >> 2; ct0 < nct; ct0 += 8) {
        double bv[4][8], d[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ct = ct0 + 2 * q;
          const int col = c0 + TB + ct * 8;
          const bool on = ct < nct && col + g < n;
          const double* rb = R + (int64_t)min(col + g, n - 1) * ldr + c0 + t;
#pragma unroll
          for (int u = 0; u < 8; ++u) bv[q][u] = on ? __ldg(rb + 4 * u) : 0.0;
          const int cc = min(col, nbk * TB - 8);
          d[q][0] = xs[(size_t)(cc + 2 * t) * XS + rt * 8 + g];
          d[q][1] = xs[(size_t)(cc + 2 * t + 1) * XS + rt * 8 + g];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma884(d[q][0], d[q][1], av[u], bv[q][u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ct = ct0 + 2 * q;
          if (ct < nct) {
            const int col = c0 + TB + ct * 8;
            xs[(size_t)(col + 2 * t) * XS + rt * 8 + g] = d[q][0];
            xs[(size_t)(col + 2 * t + 1) * XS + rt * 8 + g] = d[q][1];
          }
        }
      }
    }
    __syncthreads();
  }
}

size_t trsm_work(int n) { return sizeof(double) * (size_t)((n + TB - 1) / TB) * TB * TB; }
bool trsm_supported(int n) { return n >= 1 && n <= 512; }

cudaError_t trsm_right_upper(double* A, int64_t lda, int64_t p, const double* R, int ldr, int n, double* work,
                             cudaStream_t st) {
  if (!trsm_supported(n)) return cudaErrorInvalidValue;
  if (p <= 0) return cudaSuccess;
  const int nbk = (n + TB - 1) / TB;
  probe_before(K_TRSM, st);
  diag_inv_kernel<<<nbk, TB, 0, st>>>(R, ldr, n, work);
  probe_after(K_TRSM, st);
  const size_t smem = sizeof(double) * (size_t)nbk * TB * XS;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int64_t grid = (p + TB - 1) / TB;
  probe_before(K_TRSM, st);
  trsm_kernel<<<(unsigned)grid, kTrsmThreads, smem, st>>>(A, lda, p, R, ldr, n, work);
  probe_after(K_TRSM, st);
  return cudaGetLastError();
}

}  // namespace ngd
