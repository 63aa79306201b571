// Tall-skinny right triangular solve  X R = A  (A: p x n column-major, R: n x n upper,
// X overwrites A) on FP64 tensor cores, for the Nystrom factorisation (n = ell <= 512).
//
// Every Cholesky-QR step of sketch.py:73-86 as restated here (Omega's orthonormalisation,
// B = Y_nu C^{-1}, the three passes of shifted Cholesky-QR3) is a p x ell right solve.
// cuBLAS DTRSM runs these shapes at ~3 TFLOP/s on B200 (tools/blas_shapes.py: 238 us
// for 8577 x 300 vs 62 us for the same-shape DGEMM).  Here:
//   1. diag_inv: the 32 x 32 diagonal blocks of R are inverted (one CTA per block,
//      column-parallel back substitution) -- the only sequential arithmetic;
//   2. trsm: one CTA per 32-row panel of A walks the column blocks left to right:
//        T   = A[:, J] - X[:, <J] R[<J, J]   (DMMA, K = 32 J, X from shared memory)
//        X_J = T inv(R_JJ)                   (DMMA, K = 32)
//      so all of the O(p n^2) work is DMMA.8x8x4 with the panel resident in smem.
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
  extern __shared__ __align__(16) double xs[];  // [nbk * TB columns][XS]: solved panel X (and T scratch)
  const int nbk = (n + TB - 1) / TB;
  double* Ts = xs + (size_t)nbk * TB * XS;       // [TB][XS] T of the current block (column-major)
  const int64_t r0 = (int64_t)blockIdx.x * TB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // warp tile: rows 8 * (warp & 3) .. +7, columns 16 * (warp >> 2) .. +15 (two 8 x 8 DMMA tiles)
  const int tr = 8 * (warp & 3), tc = 16 * (warp >> 2);
  const int64_t row = r0 + tr + g;
  const bool row_ok = row < p;
  for (int J = 0; J < nbk; ++J) {
    const int c0 = J * TB;
    double d[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = c0 + tc + 8 * h + 2 * t + e;
        d[h][e] = (row_ok && col < n) ? A[(int64_t)col * lda + row] : 0.0;
      }
    }
    // T = A_J - X_{<J} R_{<J,J}
    for (int k = 0; k < c0; k += 4) {
      const double a = -xs[(size_t)(k + t) * XS + tr + g];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + tc + 8 * h + g;
        const double b = col < n ? __ldg(R + (int64_t)col * ldr + k + t) : 0.0;
        dmma884(d[h][0], d[h][1], a, b);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cl = tc + 8 * h + 2 * t;
      Ts[(size_t)cl * XS + tr + g] = d[h][0];
      Ts[(size_t)(cl + 1) * XS + tr + g] = d[h][1];
    }
    __syncthreads();
    // X_J = T inv(R_JJ)
    const double* Ri = Rinv + (size_t)J * TB * TB;
    double x[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int k = 0; k < TB; k += 4) {
      const double a = Ts[(size_t)(k + t) * XS + tr + g];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = tc + 8 * h + g;
        dmma884(x[h][0], x[h][1], a, __ldg(Ri + (size_t)cl * TB + k + t));
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cl = tc + 8 * h + 2 * t + e;
        xs[(size_t)(c0 + cl) * XS + tr + g] = x[h][e];
        if (row_ok && c0 + cl < n) A[(int64_t)(c0 + cl) * lda + row] = x[h][e];
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
  const size_t smem = sizeof(double) * ((size_t)nbk * TB * XS + (size_t)TB * XS);
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
