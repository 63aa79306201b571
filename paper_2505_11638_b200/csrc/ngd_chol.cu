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
#include <cooperative_groups.h>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace cg = cooperative_groups;

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


// ---------------------------------------------------------------------------
// Cluster Cholesky for 160 < n <= 512 (cuSOLVER potrf takes ~300 us at n = 300 on B200;
// one SM is bound by its FP64 rate at ~70 us).  Right-looking, 32 x 32 blocks, the matrix
// in global memory (L2-resident), a cluster of 8 CTAs synchronised by cluster barriers:
//   step J:  panel   U[J, >J] = U_JJ^{-T} A[J, >J]   (all CTAs; thread per column,
//                                                     forward substitution, U_JJ in smem)
//            barrier
//            trailing A[I, K] -= U[J, I]^T U[J, K]    (DMMA 8x8x4 tiles over all warps) while
//                     CTA 0 first updates and factors the next diagonal block in shared
//                     memory (look-ahead: the sequential pivot chain overlaps the update)
//            barrier
// Failure semantics as potrf: info = first non-positive (or NaN) pivot + 1, factor stops.
// ---------------------------------------------------------------------------
#ifdef NGD_CHOL_TRACE
__device__ unsigned long long g_ctr[8];
#define CT_T(v) long long v = clock64()
#define CT_ADD(k, d) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_ctr[k] += (unsigned long long)(d); } while (0)
#else
#define CT_T(v)
#define CT_ADD(k, d)
#endif
constexpr int CB = 32;            // block size
constexpr int kClusterChol = 8;   // CTAs
constexpr int kCholCThreads = 256;
constexpr int PSS = CB + 4;       // panel column stride in shared memory: (4 i + k) distinct banks

// factor the 32 x 32 symmetric block S (upper used, S[i][k] at S[i * (CB+1) + k]) in place: S <- U
// (upper), one warp, lane k owns column k in registers; row j of U reaches the other lanes by
// shuffles (no shared-memory round trip or warp barrier on the pivot chain).  rdiag[j] = 1 / U_jj.
// Returns the failing local pivot + 1, or 0.
__device__ int factor_diag_warp(double* S, int nb, double* rdiag) {
  const int k = threadIdx.x & 31;
  double col[CB];
#pragma unroll
  for (int i = 0; i < CB; ++i) col[i] = (i <= k) ? S[i * (CB + 1) + k] : 0.0;
  __shared__ double urow[2][CB];  // row j of U, double-buffered by j parity (one warp barrier per pivot)
  int fail = 0;
  // The pivot chain runs through lane j+1 only: its next pivot col[j+1] - u^2 uses its own u, so the
  // shared-memory broadcast of row j (needed by the other columns) stays off the chain.
  double pnext = __shfl_sync(0xffffffffu, col[0], 0);
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    if (j < nb && !fail) {
      const double piv = pnext;
      if (!(piv > 0.0)) {
        fail = j + 1;
      } else {
        const double r = rsqrt(piv);  // one MUFU op on the pivot chain; U_jj = piv / sqrt(piv)
        const double u = (k == j) ? piv * r : col[j] * r;
        if (k >= j) col[j] = u;
        if (k == j) rdiag[j] = r;
        const double uk = (k > j) ? u : 0.0;
        if (j + 1 < CB) pnext = __shfl_sync(0xffffffffu, fma(-uk, uk, col[j + 1 < CB ? j + 1 : j]), j + 1 < CB ? j + 1 : 0);
        urow[j & 1][k] = uk;
        __syncwarp();
#pragma unroll
        for (int i = j + 1; i < CB; ++i) col[i] = fma(-urow[j & 1][i], uk, col[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < CB; ++i)
    if (i <= k) S[i * (CB + 1) + k] = col[i];
  __syncwarp();
  return fail;
}

// every CTA factors the same diagonal block redundantly (identical arithmetic): no broadcast of
// U_JJ, and all CTAs see the same failure at the same step
__global__ void __launch_bounds__(kCholCThreads, 1) chol_cluster_kernel(double* A, int n, int lda, int* info,
                                                                         int* unused) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int NW = kCholCThreads / 32;
  const int nbk = (n + CB - 1) / CB;
  extern __shared__ __align__(16) double Ps[];  // [n - c1][PSS] panel row U[J, c1:n] of the current step
  __shared__ double S[CB * (CB + 1)];           // U_JJ (factored locally by every CTA)
  __shared__ double rd[CB];                     // 1 / U_jj
  __shared__ int s_fail;
  (void)unused;
  // prologue: factor block 0
  {
    const int nb0 = min(CB, n);
    for (int e = tid; e < CB * CB; e += kCholCThreads) {
      const int i = e / CB, k = e % CB;
      S[i * (CB + 1) + k] = (i < nb0 && k < nb0) ? A[(int64_t)k * lda + i] : (i == k ? 1.0 : 0.0);
    }
    __syncthreads();
    if (warp == 0) {
      CT_T(f0);
      const int f = factor_diag_warp(S, nb0, rd);
      CT_T(f1);
      CT_ADD(0, f1 - f0);
      if (lane == 0) s_fail = f;
    }
    __syncthreads();
    if (q == 0) {
      for (int e = tid; e < CB * CB; e += kCholCThreads) {
        const int i = e / CB, k = e % CB;
        if (i <= k && k < nb0) A[(int64_t)k * lda + i] = S[i * (CB + 1) + k];
      }
      if (tid == 0) info[0] = s_fail;
    }
  }
  CT_T(k0);
  for (int J = 0; J < nbk; ++J) {
    if (s_fail) break;
    CT_T(j0);
    const int c0 = J * CB, c1 = c0 + CB;
    const int np = n - c1;  // panel columns
    // panel: U[J, c] = U_JJ^{-T} A[J, c] for c >= c1 (forward substitution, lane per column); the
    // result goes to global (final U) and into every CTA's Ps (the trailing update's operand)
    for (int cc = (warp * kClusterChol + q) * 32 + lane; cc - lane < np; cc += kClusterChol * kCholCThreads) {
      if (cc >= np) continue;
      double* colp = A + (int64_t)(c1 + cc) * lda + c0;
      double x[CB];
#pragma unroll
      for (int i = 0; i < CB; ++i) x[i] = colp[i];
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        x[i] *= rd[i];
#pragma unroll
        for (int m = i + 1; m < CB; ++m) x[m] = fma(-S[i * (CB + 1) + m], x[i], x[m]);
      }
#pragma unroll
      for (int i = 0; i < CB; ++i) colp[i] = x[i];
    }
    CT_T(j1);
    CT_ADD(2, j1 - j0);
    cl.sync();
    CT_T(j2);
    CT_ADD(3, j2 - j1);
    if (J == nbk - 1) break;
    const int m = nbk - J - 1;  // trailing blocks
    const int nb1 = min(CB, n - c1);
    // stage the panel row U[J, c1:n] (32 contiguous doubles per column) with cp.async
    for (int e = tid; e < np * (CB / 2); e += kCholCThreads) {
      const int cc = e >> 4, k2 = (e & 15) * 2;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Ps + (size_t)cc * PSS + k2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(A + (int64_t)(c1 + cc) * lda + c0 + k2));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // next diagonal block S <- A[J+1, J+1] - U[J, J+1]^T U[J, J+1] (10 upper 8x8 tiles, DMMA), every CTA
    for (int tile = warp; tile < 16; tile += NW) {
      const int ti = tile >> 2, tk = tile & 3;
      if (ti > tk) continue;
      const int ri = ti * 8 + g, ck = tk * 8 + 2 * t, cb = tk * 8 + g;
      double d0 = (ri < nb1 && ck < nb1) ? A[(int64_t)(c1 + ck) * lda + c1 + ri] : 0.0;
      double d1 = (ri < nb1 && ck + 1 < nb1) ? A[(int64_t)(c1 + ck + 1) * lda + c1 + ri] : 0.0;
#pragma unroll
      for (int k0 = 0; k0 < CB; k0 += 4) {
        const double a = (ri < nb1) ? -Ps[(size_t)ri * PSS + k0 + t] : 0.0;
        const double b = (cb < nb1) ? Ps[(size_t)cb * PSS + k0 + t] : 0.0;
        dmma884(d0, d1, a, b);
      }
      S[ri * (CB + 1) + ck] = d0;
      S[ri * (CB + 1) + ck + 1] = d1;
    }
    __syncthreads();
    CT_T(j3);
    CT_ADD(4, j3 - j2);
    if (warp == 0) {
      for (int i = 0; i < CB; ++i)  // identity padding past n
        if (i >= nb1 && lane >= nb1) S[i * (CB + 1) + lane] = (i == lane) ? 1.0 : 0.0;
      __syncwarp();
      CT_T(f0);
      const int f = factor_diag_warp(S, nb1, rd);
      CT_T(f1);
      CT_ADD(0, f1 - f0);
      if (lane == 0) s_fail = f;
      if (q == 0) {
        if (lane == 0 && f) info[0] = c1 + f;
        for (int e = lane; e < CB * CB; e += 32) {
          const int i = e >> 5, k = e & (CB - 1);
          if (i <= k && k < nb1) A[(int64_t)(c1 + k) * lda + c1 + i] = S[i * (CB + 1) + k];
        }
      }
    } else {
      // the rest of the trailing update: 8x8 tiles of blocks (I, K), J < I <= K, except (J+1, J+1),
      // over warps 1..7 of every CTA
      const int units = m * (m + 1) / 2 * 16;
      const int pool = kClusterChol * (NW - 1);
      for (int u = q * (NW - 1) + warp - 1; u < units; u += pool) {
        const int pr = u >> 4, tile = u & 15;
        int I = 0, rem = pr;  // pair index -> (I, K), 0 <= I <= K < m, row-major upper triangle
        while (rem >= m - I) {
          rem -= m - I;
          ++I;
        }
        const int K = I + rem;
        if (I == 0 && K == 0) continue;
        const int ti = tile >> 2, tk = tile & 3;
        if (I == K && ti > tk) continue;
        const int li = I * CB + ti * 8, lk = K * CB + tk * 8;  // panel-local column offsets
        if (li >= np || lk >= np) continue;
        const int ri = li + g, ck = lk + 2 * t, cb = lk + g;
        double d0 = (ri < np && ck < np) ? A[(int64_t)(c1 + ck) * lda + c1 + ri] : 0.0;
        double d1 = (ri < np && ck + 1 < np) ? A[(int64_t)(c1 + ck + 1) * lda + c1 + ri] : 0.0;
#pragma unroll
        for (int k0 = 0; k0 < CB; k0 += 4) {
          const double a = (ri < np) ? -Ps[(size_t)ri * PSS + k0 + t] : 0.0;
          const double b = (cb < np) ? Ps[(size_t)cb * PSS + k0 + t] : 0.0;
          dmma884(d0, d1, a, b);
        }
        if (ri < np && ck < np) A[(int64_t)(c1 + ck) * lda + c1 + ri] = d0;
        if (ri < np && ck + 1 < np) A[(int64_t)(c1 + ck + 1) * lda + c1 + ri] = d1;
      }
    }
    CT_T(j4);
    CT_ADD(5, j4 - j3);
    cl.sync();  // trailing updates visible; every CTA done reading Ps
    CT_T(j5);
    CT_ADD(6, j5 - j4);
  }
  CT_T(k1);
  CT_ADD(7, k1 - k0);
  if (q == 0 && tid == 0 && s_fail == 0) info[0] = 0;
}

bool chol_cluster_supported(int n) { return n > 0 && n <= 512; }

cudaError_t chol_upper_cluster(double* A, int n, int lda, int* info, int* flag, cudaStream_t st) {
  if (!chol_cluster_supported(n)) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * (size_t)n * PSS;
  static size_t smem_attr = 0;
  if (smem > smem_attr) {
    cudaError_t e = cudaFuncSetAttribute(chol_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_attr = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterChol, 1, 1);
  cfg.blockDim = dim3(kCholCThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterChol;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  probe_before(K_CHOL, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, chol_cluster_kernel, A, n, lda, info, flag);
  probe_after(K_CHOL, st);
  return e;
}

}  // namespace ngd
