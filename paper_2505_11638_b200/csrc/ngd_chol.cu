// Small dense Cholesky A = U^T U (upper, column-major) in one CTA.
//
// The Nystrom factorisation needs up to five ell x ell Choleskys per NGD step
// (Cholesky-QR of Omega, the sketch Cholesky of sketch.py:80, three in the
// shifted Cholesky-QR3 of B).  cuSOLVER's potrf launches ~40 small kernels for
// ell = 300 (~0.4 ms).  This is a right-looking blocked Cholesky in a single
// 1024-thread CTA: the nb x nb diagonal block is factored in shared memory, the
// block row is solved by forward substitution (one column per thread), and the
// trailing upper triangle is updated with the staged block row (warp per
// column, lanes over rows: coalesced column-major traffic, L2-resident matrix).
// Failure semantics match LAPACK potrf: info = j + 1 for the first pivot that
// is not positive (or NaN); the factorisation stops there.
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

constexpr int kCholThreads = 1024;

template <int NB>
__global__ void __launch_bounds__(kCholThreads, 1) chol_upper_kernel(double* A, int n, int lda, int* info) {
  extern __shared__ __align__(16) double sm[];
  double* Ds = sm;                 // [NB][NB+1] diagonal block, Ds[r * (NB+1) + c]
  double* Ps = sm + NB * (NB + 1); // [NB][n] block row (rows of U), Ps[t * n + c]
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kCholThreads / 32;
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int kb = min(NB, n - k0);
    // 1. diagonal block into shared memory
    for (int e = tid; e < kb * kb; e += kCholThreads) {
      const int r = e % kb, c = e / kb;
      Ds[r * (NB + 1) + c] = (r <= c) ? A[(int64_t)(k0 + c) * lda + k0 + r] : 0.0;
    }
    __syncthreads();
    // unblocked right-looking Cholesky of the block (one warp; rows of U)
    if (warp == 0) {
      for (int j = 0; j < kb; ++j) {
        const double d = Ds[j * (NB + 1) + j];
        if (!(d > 0.0)) {  // also catches NaN
          if (lane == 0 && fail == 0) fail = k0 + j + 1;
          break;
        }
        const double rj = sqrt(d);
        __syncwarp();
        for (int c = j + 1 + lane; c < kb; c += 32) Ds[j * (NB + 1) + c] /= rj;
        if (lane == 0) Ds[j * (NB + 1) + j] = rj;
        __syncwarp();
        for (int c = j + 1 + lane; c < kb; c += 32) {
          const double ujc = Ds[j * (NB + 1) + c];
          for (int i = j + 1; i <= c; ++i) Ds[i * (NB + 1) + c] -= Ds[j * (NB + 1) + i] * ujc;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (fail) break;
    for (int e = tid; e < kb * kb; e += kCholThreads) {
      const int r = e % kb, c = e / kb;
      if (r <= c) A[(int64_t)(k0 + c) * lda + k0 + r] = Ds[r * (NB + 1) + c];
    }
    // 2. block row: U[k0:k0+kb, c] = U_kk^{-T} A[k0:k0+kb, c] for c >= k0 + kb (forward substitution)
    const int m = n - k0 - kb;
    for (int cc = tid; cc < m; cc += kCholThreads) {
      const int c = k0 + kb + cc;
      double x[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) x[i] = (i < kb) ? A[(int64_t)c * lda + k0 + i] : 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (i < kb) {
          double s = x[i];
#pragma unroll
          for (int t = 0; t < i; ++t) s -= Ds[t * (NB + 1) + i] * x[t];
          x[i] = s / Ds[i * (NB + 1) + i];
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (i < kb) {
          A[(int64_t)c * lda + k0 + i] = x[i];
          Ps[(int64_t)i * n + cc] = x[i];
        }
    }
    __syncthreads();
    // 3. trailing update of the upper triangle: A[r][c] -= sum_t P[t][r] P[t][c], k0+kb <= r <= c
    for (int cc = warp; cc < m; cc += NW) {
      double pc[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) pc[t] = (t < kb) ? Ps[(int64_t)t * n + cc] : 0.0;
      double* col = A + (int64_t)(k0 + kb + cc) * lda + k0 + kb;
      for (int rr = lane; rr <= cc; rr += 32) {
        double s = col[rr];
#pragma unroll
        for (int t = 0; t < NB; ++t) s -= Ps[(int64_t)t * n + rr] * pc[t];
        col[rr] = s;
      }
    }
    __syncthreads();
  }
  if (tid == 0) info[0] = fail;
}

size_t chol_smem(int n, int nb) { return sizeof(double) * ((size_t)nb * (nb + 1) + (size_t)nb * n); }

cudaError_t chol_upper(double* A, int n, int lda, int* info, cudaStream_t st) {
  if (n < 1 || chol_smem(n, 16) > 200 * 1024) return cudaErrorInvalidValue;
  const size_t smem = chol_smem(n, 16);
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(chol_upper_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
    attr = 200 * 1024;
  }
  probe_before(K_CHOL, st);
  chol_upper_kernel<16><<<1, kCholThreads, smem, st>>>(A, n, lda, info);
  probe_after(K_CHOL, st);
  return cudaGetLastError();
}

// single-SM L2-bound trailing updates lose to cuSOLVER's multi-kernel potrf beyond ~160 (measured: C2 ell=300)
bool chol_supported(int n) { return n >= 1 && n <= 160; }

}  // namespace ngd
